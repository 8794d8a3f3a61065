"""Parity at the BASELINE.json full sizes (-m gpu), on sampled chunks.

Chunks are independent (each has its own reference frame), so the
oracle computes any sampled chunk of a full-size step exactly; the GPU runs
the whole step in the launch configuration bench.py times (no debug
retention, CUDA graphs after the first sight of the input buffer)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from gpu_harness import within

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _run(net, fr_np, theta, precision, repeat=2):
    import torch
    from paper_2410_20790_b200 import Encoder
    B, L = fr_np.shape[:2]
    enc = Encoder(net, B, L, precision=precision)
    fr = torch.from_numpy(fr_np).cuda()
    for _ in range(repeat):   # second pass replays the captured graph
        enc.encode_reference(fr[:, 0])
        enc.encode_diff(fr[:, 1:], theta)
    torch.cuda.synchronize()
    return enc


def _bf16_close(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    rms = float(np.sqrt(np.mean(b * b)))
    return bool(np.all(np.abs(a - b) <= 2e-2 * np.abs(b) + 2e-2 * rms))


def _bf16_report(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    rms = float(np.sqrt(np.mean(b * b)))
    bad = np.abs(a - b) > 2e-2 * np.abs(b) + 2e-2 * rms
    rel_l2 = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
    return float(bad.mean()), rel_l2


@pytest.mark.parametrize("theta", [0.0, 0.05])
def test_cfg2_bench_config_bf16_sampled(theta):
    """The bench workload itself: 64 chunks x 32 frames, BF16 mode.

    theta = 0: elementwise within the north_star bf16 bound.  theta = 0.05
    (the bench threshold): the GPU and the oracle's BF16 contract differ
    only in tensor-core summation order, but over 31 sequential frames a
    rounding difference can flip a truncation decision (reading R23), after
    which that pixel legitimately diverges by threshold-sized amounts; the
    check is >= 99.9% of output elements within the bf16 bound, relative L2
    error <= 1e-2, and per-site counts within 0.1% of the site's pixels."""
    cfg = W.get_config(2)
    net = cfg.build_net()
    u8 = W.gen_video(cfg.chunks_per_step, cfg.L, cfg.h, cfg.w, cfg.c, cfg.video_seed(0), **cfg.video)
    fr = W.to_float(u8)
    enc = _run(net, fr, theta, "bf16")
    act, _, px = enc.get_sparsity()
    tap = enc.taps[0]
    out = enc.outputs(tap)
    N = [cfg.h * cfg.w] + [h * w for (h, w, c), l in zip(oracle.shapes(net), net.layers) if l["kind"] in W.NONLINEAR]
    for b in (0, 29, 63):
        r = oracle.run_chunk(net, fr[b], theta, want_masks=False, precision="bf16")
        got = out[b].cpu().numpy()
        if theta == 0.0:
            assert _bf16_close(got, r["taps"][tap]), (b, _bf16_report(got, r["taps"][tap]))
        else:
            bad, rel = _bf16_report(got, r["taps"][tap])
            assert bad <= 1e-3 and rel <= 1e-2, (b, bad, rel)
        assert np.array_equal(act[b][0], r["counts"][0])          # input site: identical fp32 work
        diff = np.abs(act[b] - r["counts"]).astype(np.float64)
        assert np.all(diff <= 1e-3 * np.array(N)[:, None] + 2), (b, diff.max())


def test_cfg4_resnet18_720p_fp32_sampled():
    cfg = W.get_config(4)
    net = cfg.build_net()
    u8 = W.gen_video(2, 3, cfg.h, cfg.w, cfg.c, cfg.video_seed(0), **cfg.video)
    fr = W.to_float(u8)
    enc = _run(net, fr, 0.05, "fp32")
    act, _, _ = enc.get_sparsity()
    tap = enc.taps[0]
    r = oracle.run_chunk(net, fr[1], 0.05, want_masks=False)
    assert np.array_equal(enc.outputs(tap)[1].cpu().numpy(), r["taps"][tap])
    assert np.array_equal(act[1], r["counts"])


def test_cfg5_effdet_d0_1080p_fp32_sampled():
    cfg = W.get_config(5)
    net = cfg.build_net()
    u8 = W.gen_video(1, 3, cfg.h, cfg.w, cfg.c, cfg.video_seed(0), **cfg.video)
    fr = W.to_float(u8)
    enc = _run(net, fr, 0.05, "fp32")
    act, _, _ = enc.get_sparsity()
    r = oracle.run_chunk(net, fr[0], 0.05, want_masks=False)
    for tap in enc.taps:
        assert within(enc.outputs(tap)[0].cpu().numpy(), r["taps"][tap]), tap
    N = [cfg.h * cfg.w] + [h * w for (h, w, c), l in zip(oracle.shapes(net), net.layers) if l["kind"] in W.NONLINEAR]
    assert np.all(np.abs(act[0] - r["counts"]) <= 1e-4 * np.array(N)[:, None])


@pytest.mark.parametrize("cid", [3, 4, 5])
def test_bench_config_bf16_sampled(cid):
    """cfg3 / cfg4 / cfg5 in the bench launch configuration: all chunks of a
    step x all frames, uint8 frames, BF16 mode (tcgen05 convs), CUDA graph
    replay; one sampled chunk against the oracle's BF16 contract at the
    config's fixed threshold.  Criteria as for cfg2 at theta > 0 (reading
    R23: a rounding-order difference may flip a truncation decision, after
    which that pixel diverges by threshold-sized amounts): >= 99.9 % of every
    tap's elements within the bf16 bound, relative L2 <= 1e-2, input-site
    counts identical; per site the step total of emitted pixel-frames within
    0.5 % and every frame within 3 % of the site's pixels (+2).  The
    per-frame bound is looser than cfg2's because one flipped decision in a
    mid layer is dilated by every following 3x3 conv before it reaches the
    920-pixel (ResNet-18 layer4 at 720p) sites."""
    import torch
    from paper_2410_20790_b200 import Encoder
    cfg = W.get_config(cid)
    net = cfg.build_net()
    B, L = cfg.chunks_per_step, cfg.L
    u8 = np.stack([W.gen_chunk(cfg.video_seed(c), L, cfg.h, cfg.w, cfg.c, **cfg.video) for c in range(B)])
    theta = cfg.theta_fixed
    enc = Encoder(net, B, L, precision="bf16")
    x = torch.from_numpy(u8).cuda()
    for _ in range(2):   # second pass replays the captured graph
        enc.encode_reference(x[:, 0])
        enc.encode_diff(x[:, 1:], theta)
    torch.cuda.synchronize()
    act, _, _ = enc.get_sparsity()
    b = B - 1
    fr = W.to_float(u8[b])
    del x, u8
    r = oracle.run_chunk(net, fr, theta, want_masks=False, precision="bf16")
    for tap in enc.taps:
        got = enc.outputs(tap)[b].cpu().numpy()
        bad, rel = _bf16_report(got, r["taps"][tap])
        assert bad <= 1e-3 and rel <= 1e-2, (cid, tap, bad, rel)
    assert np.array_equal(act[b][0], r["counts"][0])
    N = [cfg.h * cfg.w] + [h * w for (h, w, c), l in zip(oracle.shapes(net), net.layers) if l["kind"] in W.NONLINEAR]
    Nc = np.array(N, np.float64)
    diff = np.abs(act[b] - r["counts"]).astype(np.float64)
    assert np.all(diff <= 3e-2 * Nc[:, None] + 2), (cid, diff.max())
    tot = np.abs(act[b].sum(1) - r["counts"].sum(1)).astype(np.float64)
    assert np.all(tot <= 5e-3 * Nc * (L - 1) + 2), (cid, tot.max())
