"""Multi-process host logic on CPU (gloo, world_size 2): chunk sharding,
the per-step all-gather of per-site counts and the controller give every
rank the same thresholds, identical to a single-process run over the same
fixed step groups (PIN15, reading R15).  Per-chunk statistics come from the
oracle (the CUDA path is covered by -m gpu tests)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import workloads as W
from paper_2410_20790_b200.sharding import shard

STEPS, GROUP = 4, 4


def _setup():
    net = W.models.toy_encoder(20, 24)
    W.init_weights(net, 5)
    frames = {}
    for cid in range(STEPS * GROUP):
        u8 = W.gen_video(1, 6, 20, 24, 3, 1000 + cid, n_objects=3, size=(4, 8), speed=(1, 2), noise_q=0.1,
                         noise_amp=3)
        frames[cid] = W.to_float(u8)[0]
    return net, frames


def _run(rank, world, port, out):
    import torch.distributed as dist
    from paper_2410_20790_b200 import ThresholdController
    from paper_2410_20790_b200.sharding import StatsExchange
    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    net, frames = _setup()
    ns = oracle.num_sites(net)
    ctl = ThresholdController(ns, policy="ibst", T=0.6, eps=0.05, cycle=3)
    ex = StatsExchange(ns)
    thetas, taps = [], {}
    for step in range(STEPS):
        th = ctl.thresholds()
        thetas.append(th.copy())
        act = np.zeros(ns, np.int64)
        pix = np.zeros(ns, np.int64)
        for cid in shard(step, GROUP, rank, world):
            r = oracle.run_chunk(net, frames[cid], th, want_masks=False)
            act += r["counts"].sum(1)
            taps[cid] = r["taps"][3]
        shp = oracle.shapes(net)
        per_site_px = [20 * 24] + [shp[i][0] * shp[i][1] for i, l in enumerate(net.layers) if l["kind"] in W.NONLINEAR]
        pix[:] = np.array(per_site_px) * 5 * len(shard(step, GROUP, rank, world))
        sa, sp = ex.exchange(np.concatenate([act, pix]))
        ctl.observe(sa, sp)
    out[rank] = (np.array(thetas), taps)
    if world > 1:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_covers_every_chunk_once():
    for world in (1, 2, 4, 8):
        seen = []
        for step in range(3):
            for r in range(world):
                seen += shard(step, 8, r, world)
        assert sorted(seen) == list(range(24))
    with pytest.raises(ValueError):
        shard(0, 6, 0, 4)


def test_two_ranks_match_single_process():
    single = {}
    _run(0, 1, 0, single)
    th1, taps1 = single[0]
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    ps = [ctx.Process(target=_run, args=(r, 2, port, out)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(180)
        assert p.exitcode == 0
    th_a, taps_a = out[0]
    th_b, taps_b = out[1]
    assert np.array_equal(th_a, th_b) and np.array_equal(th_a, th1)
    assert len(np.unique(th1[:, 1])) > 1          # the controller actually moved
    merged = dict(taps_a)
    merged.update(taps_b)
    assert sorted(merged) == sorted(taps1)
    for cid in taps1:                                # PIN15: outputs bit-identical across G
        assert np.array_equal(merged[cid], taps1[cid])


# ---------------------------------------------------------------- StepLoop
def _run_loop(rank, world, port, out):
    """The bench's own step loop (paper_2410_20790_b200.sharding.StepLoop:
    R15 fixed groups, StatsExchange all-gather, the C++ controller) with the
    oracle standing in for the GPU encoder."""
    import torch.distributed as dist
    from paper_2410_20790_b200 import ThresholdController
    from paper_2410_20790_b200.sharding import StatsExchange, StepLoop
    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    net, frames = _setup()
    ns = oracle.num_sites(net)
    ctl = ThresholdController(ns, policy="ibst", T=0.6, eps=0.05, cycle=3)
    loop = StepLoop(GROUP, STEPS, rank, world, ctl, StatsExchange(ns))
    shp = oracle.shapes(net)
    per_site_px = np.array([20 * 24] + [shp[i][0] * shp[i][1] for i, l in enumerate(net.layers)
                                        if l["kind"] in W.NONLINEAR], np.int64)
    taps = {}

    def encode(group, ids, th):
        act = np.zeros(ns, np.int64)
        for cid in ids:
            r = oracle.run_chunk(net, frames[cid], th, want_masks=False)
            act += r["counts"].sum(1)
            taps[(len(loop.history), cid)] = r["taps"][3]
        return np.concatenate([act, per_site_px * 5 * len(ids)])

    for step in range(2 * STEPS):          # every group twice: the job wraps around
        loop.run_step(step, encode)
    out[rank] = (np.array(loop.history), taps)
    if world > 1:
        dist.destroy_process_group()


def test_step_loop_gpu_count_invariant():
    """PIN15 on the bench's step loop: G = 1, 2 and 4 ranks give identical
    threshold sequences and bit-identical per-chunk outputs."""
    ref = {}
    _run_loop(0, 1, 0, ref)
    th1, taps1 = ref[0]
    assert len(np.unique(th1[:, 1])) > 1
    ctx = mp.get_context("spawn")
    for world in (2, 4):
        mgr = ctx.Manager()
        out = mgr.dict()
        port = _free_port()
        ps = [ctx.Process(target=_run_loop, args=(r, world, port, out)) for r in range(world)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(300)
            assert p.exitcode == 0
        merged = {}
        for r in range(world):
            th, taps = out[r]
            assert np.array_equal(th, th1), (world, r)
            merged.update(taps)
        assert sorted(merged) == sorted(taps1)
        for k in taps1:
            assert np.array_equal(merged[k], taps1[k])
