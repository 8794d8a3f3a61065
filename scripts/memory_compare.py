#!/usr/bin/env python
"""SparseBatch vs vanilla (streaming caches) memory and throughput per config
(PAPER.md P:139 vs P:152, the Fig. memory_comparison /
Table 1 memory analogue on synthetic inputs).

For each config: st_memory_report of a SparseBatch encoder and of a
streaming encoder (the vanilla DeltaCNN schedule's persistent per-site
caches), the oracle accountant's element counts for both schedules, and the
diff-frame throughput of (a) the SparseBatch step (reference + 31 diff
frames), (b) streaming continuation calls (no reference frame, each call
continuing every chunk by L-1 frames) and (c) the vanilla DeltaCNN schedule
(reference + L-1 single-frame passes with the caches kept across passes).  CUDA events on the launch stream,
L2 flushed between calls.  One JSON document on stdout.
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
a = ap.parse_args()

import torch  # noqa: E402
from paper_2410_20790_b200 import Encoder  # noqa: E402
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

    for mode in ("sparsebatch", "streaming", "vanilla"):
        enc = Encoder(net, B, L, precision=a.precision, streaming=(mode != "sparsebatch"))
        mem = enc.memory_report()
        if mode == "sparsebatch":
            def step():
                enc.encode_reference(x[:, 0], s)
                enc.encode_diff(x[:, 1:L], th, s)
            ms = timed(step, a.steps)
        elif mode == "vanilla":
            # the vanilla DeltaCNN schedule: one pass through
            # all layers per frame index, every site's caches kept across passes
            def step():
                enc.encode_reference(x[:, 0], s)
                for t in range(1, L):
                    enc.encode_diff(x[:, t:t + 1], th, s)
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
        res[mode] = {"memory": mem, "ms_per_call": ms, "diff_fps": B * (L - 1) / (ms / 1e3)}
        del enc
        torch.cuda.empty_cache()
    for sched in ("sparsebatch", "vanilla"):
        m = oracle.account_memory(net, sched, n_videos=B, L=L)
        res[f"accountant_{sched}_MB_fp32"] = {k: v * 4 / 1e6 for k, v in m.items() if k.endswith("values")}
    doc[f"cfg{cid}"] = res
    print(json.dumps({f"cfg{cid}": res}), file=sys.stderr)
print(json.dumps(doc))
