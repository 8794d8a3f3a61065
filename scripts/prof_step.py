#!/usr/bin/env python
"""The bench step of a config for ncu: calibrate (BST until every site is
frozen, as bench.py does), W warm-up steps, then K profiled steps between
cudaProfilerStart/Stop (run ncu with --profile-from-start off).

    python scripts/prof_step.py --config 5 --warmup 3 --steps 1 [--profiling] [--eager]

--eager: ST_NO_GRAPHS=1 (one launch per kernel instead of a graph replay).
--profiling: library per-launch events (ST_PROF_TRACE=1 lines on stderr).
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--profiling", action="store_true")
ap.add_argument("--eager", action="store_true")
ap.add_argument("--precision", default="bf16")
a = ap.parse_args()
if a.eager:
    os.environ["ST_NO_GRAPHS"] = "1"
if a.profiling:
    os.environ["ST_PROF_TRACE"] = "1"   # read at st_encoder_create

import torch  # noqa: E402
from paper_2410_20790_b200 import Encoder, ThresholdController  # noqa: E402

cfg = W.get_config(a.config)
net = cfg.build_net()
B, L = cfg.chunks_per_step, cfg.L
enc = Encoder(net, max_chunks=B, max_frames=L, device=0, precision=a.precision)
policy = "bst" if cfg.policy != "fixed" else "fixed"
ctl = ThresholdController(enc.n_sites, policy=policy, T=cfg.T, eps=cfg.eps, theta_fixed=cfg.theta_fixed,
                          cycle=cfg.cycle)
u8 = np.stack([W.gen_chunk(cfg.video_seed(c), L, cfg.h, cfg.w, cfg.c, **cfg.video) for c in range(B)])
x = torch.from_numpy(u8).cuda()
s = torch.cuda.current_stream()


def step(observe):
    enc.encode_reference(x[:, 0], s)
    enc.encode_diff(x[:, 1:], ctl.thresholds(), s)
    if observe:
        _, sa, sp = enc.get_sparsity()
        ctl.observe(sa, sp)


n = 0
while policy != "fixed" and n < 40 and not bool(np.all(ctl.state()[3])):
    step(True)
    n += 1
for _ in range(a.warmup):
    step(False)
torch.cuda.synchronize()
print(f"calibrated {n} steps, theta {np.round(ctl.thresholds(), 4).tolist()}", file=sys.stderr)
if a.profiling:
    enc.set_profiling(True)
torch.cuda.profiler.start()
for _ in range(a.steps):
    step(False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
if a.profiling:
    enc.kernel_times(reset=True)   # folds the records: ST_PROF_TRACE lines go to stderr
print(f"done: {enc.last_launch_count()} launches per step", file=sys.stderr)
