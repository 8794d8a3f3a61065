#!/usr/bin/env python
"""SparseBatch vs vanilla vs own dense: device memory and throughput per
config (PAPER.md P:139 vs P:152, the Fig.
memory_comparison / Table 1 memory analogue on synthetic inputs).

Encoders (total device bytes = arena + fixed areas + weights, st_device_bytes):
(a) SparseBatch: one step over L-1 diff frames; row capacity first at the
    all-active bound, then re-planned from the measured occupancy
    (st_encoder_fit_capacity, --headroom);
(b) streaming continuation: the SparseBatch step with the vanilla caches
    kept, each call continuing every chunk by L-1 frames;
(c) vanilla DeltaCNN schedule: a per-frame encoder (max_frames 2, arena for
    one frame) driven reference + L-1 single-frame passes, every site's
    x_acc / y_acc cached across passes;
(d) own dense path: every frame a reference frame, one frame per call.
Plus the oracle accountant's element counts (SparseBatch evaluated on the
measured rows).  CUDA events on the launch stream, L2 flushed between
calls.  One JSON document on stdout.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,4")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--precision", default="bf16")
ap.add_argument("--headroom", type=float, default=1.25)
a = ap.parse_args()

import torch  # noqa: E402
from paper_2410_20790_b200 import Encoder  # noqa: E402
from paper_2410_20790_b200.binding import StError  # noqa: E402
import oracle  # noqa: E402  (test infrastructure: the accountant's element counts only)

dev = torch.device("cuda:0")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
doc = {}
for cid in [int(c) for c in a.configs.split(",")]:
    cfg = W.get_config(cid)
    net = cfg.build_net()
    B, L = cfg.chunks_per_step, cfg.L
    nwin = a.steps + 3   # first call + 2 warm-up continuations + timed ones, each a new window
    u8 = np.stack([W.gen_chunk(cfg.video_seed(c), 1 + nwin * (L - 1), cfg.h, cfg.w, cfg.c, **cfg.video)
                   for c in range(B)])
    x = torch.from_numpy(u8).to(dev).float().div_(255.0)
    del u8
    th = cfg.theta_fixed
    res = {"chunks": B, "frames_per_call": L - 1}

    def timed(fn, k):
        fn()
        fn()
        torch.cuda.synchronize()
        ms = 0.0
        for i in range(k):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
            e1.synchronize()
            ms += e0.elapsed_time(e1)
        return ms / k

    rows = None
    for mode in ("sparsebatch", "streaming", "vanilla", "dense"):
        # vanilla: a genuinely per-frame encoder (max_frames = 2: one diff frame
        # per call, its arena sized for one frame) whose streaming caches carry
        # every site's x_acc / y_acc from frame to frame;
        # dense: the own dense path, one frame of each chunk per call
        Lm = {"vanilla": 2, "dense": 1}.get(mode, L)
        try:
            enc = Encoder(net, B, Lm, precision=a.precision, streaming=mode in ("streaming", "vanilla"))
        except StError as err:   # SE nets: the gate schedule spans a call (R8), no streaming caches
            res[mode] = {"unsupported": str(err)}
            continue
        mem = dict(enc.memory_report(), device_bytes=enc.device_bytes())
        if mode == "sparsebatch":
            def step():
                enc.encode_reference(x[:, 0], s)
                enc.encode_diff(x[:, 1:L], th, s)
            step()
            torch.cuda.synchronize()
            cap, pk = enc.capacity()
            rows = {i: int(v) // B for i, v in enumerate(pk[:-1]) if v >= 0}
            rows[-1] = int(pk[-1]) // B
            mem["all_active_bound"] = dict(mem)
            enc.fit_capacity(a.headroom)   # row capacity from the measured occupancy (a9)
            mem.update(enc.memory_report(), device_bytes=enc.device_bytes(), headroom=a.headroom)
            ms = timed(step, a.steps)
        elif mode == "vanilla":
            def step():
                enc.encode_reference(x[:, 0], s)
                for t in range(1, L):
                    enc.encode_diff(x[:, t:t + 1], th, s)
            ms = timed(step, a.steps)
        elif mode == "dense":
            xd = x[:, :L].reshape(B, L, *x.shape[2:])

            def step():
                for t in range(L):
                    enc.encode_reference(xd[:, t], s)
                    enc.encode_diff(None, th, s)
            ms = timed(step, a.steps)
        else:
            enc.encode_reference(x[:, 0], s)
            enc.encode_diff(x[:, 1:L], th, s)
            # continuation calls walk forward through the video, L-1 new frames each
            state = {"k": 1}

            def step():
                k = state["k"]
                enc.encode_diff(x[:, 1 + k * (L - 1):1 + (k + 1) * (L - 1)], th, s)
                state["k"] += 1
            ms = timed(step, a.steps)
        nfr = B * L if mode == "dense" else B * (L - 1)
        res[mode] = {"memory": mem, "ms_per_call": ms, "fps": nfr / (ms / 1e3)}
        del enc
        torch.cuda.empty_cache()
    eb = 2 if a.precision == "bf16" else 4
    for sched in ("sparsebatch", "vanilla"):
        m = oracle.account_memory(net, sched, n_videos=B, L=L, rows=rows if sched == "sparsebatch" else None)
        res[f"accountant_{sched}_MB"] = {k: v * 4 / 1e6 for k, v in m.items() if k.endswith("values")}
    res["accountant_note"] = ("oracle/memory.py element counts x 4 bytes (fp32 states); SparseBatch evaluated on "
                              "the measured rows per tensor (rows x %d-byte deltas counted as 4)" % eb)
    doc[f"cfg{cid}"] = res
    print(json.dumps({f"cfg{cid}": res}), file=sys.stderr)
print(json.dumps(doc))
