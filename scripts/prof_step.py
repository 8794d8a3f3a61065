#!/usr/bin/env python
"""Run W warm-up steps then K steps of config c (for ncu / ST_PROF_TRACE).

    python scripts/prof_step.py --config 2 --warmup 3 --steps 1 [--profiling]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--profiling", action="store_true", help="library per-launch events (ST_PROF_TRACE lines)")
ap.add_argument("--precision", default="bf16")
a = ap.parse_args()

import torch  # noqa: E402
from paper_2410_20790_b200 import Encoder, ThresholdController  # noqa: E402

cfg = W.get_config(a.config)
net = cfg.build_net()
B, L = cfg.chunks_per_step, cfg.L
enc = Encoder(net, max_chunks=B, max_frames=L, device=0, precision=a.precision)
ctl = ThresholdController(enc.n_sites, policy=cfg.policy, T=cfg.T, eps=cfg.eps, theta_fixed=cfg.theta_fixed,
                          cycle=cfg.cycle)
u8 = np.stack([W.gen_chunk(cfg.video_seed(c), L, cfg.h, cfg.w, cfg.c, **cfg.video) for c in range(B)])
x = torch.from_numpy(W.to_float(u8)).cuda()
s = torch.cuda.current_stream()


def step():
    enc.encode_reference(x[:, 0], s)
    enc.encode_diff(x[:, 1:], ctl.thresholds(), s)
    if cfg.policy != "fixed":
        _, sa, sp = enc.get_sparsity()
        ctl.observe(sa, sp)


for _ in range(a.warmup):
    step()
torch.cuda.synchronize()
if a.profiling:
    enc.set_profiling(True)
for _ in range(a.steps):
    step()
torch.cuda.synchronize()
if a.profiling:
    enc.kernel_times(reset=True)   # folds the records: ST_PROF_TRACE lines go to stderr
print("done", file=sys.stderr)
