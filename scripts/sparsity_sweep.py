#!/usr/bin/env python
"""Speedup over the own dense path per sparsity level (SURVEY §8(d) item 4,
the Table 2 analogue of PAPER.md P:285-290) and the fixed-threshold vs
online-adjustment per-site sparsity comparison (SURVEY §8(f) N4, P:174,
P:211).

    python scripts/sparsity_sweep.py --config 4 --targets 0.5,0.6,0.7,0.8,0.9,0.95
    python scripts/sparsity_sweep.py --config 3 --n4

Sweep: for each target sparsity T the BST controller (reading
R16) is calibrated on untimed steps until every site is frozen, then the
thresholds stay fixed and K steps are timed exactly like bench.py (CUDA
events on the launch stream, L2 flushed between steps).  Reported per
level: diff-frames/s, mean site sparsity, the row-weighted conv-output skip
1 - sum(conv output rows) / sum(B (L-1) H_out W_out), and the speedup over
the own dense path (the same kernels with every frame as a reference frame).

N4: the same workload once with one fixed threshold at every site and once
with IBST; reports the per-site sparsity of both (the fixed threshold gives
an imbalanced profile across layers, the controller pulls every site to T).
Writes one JSON document to stdout.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--targets", default="0.5,0.6,0.7,0.8,0.9,0.95")
    ap.add_argument("--eps", type=float, default=None)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--max-calib", type=int, default=16)
    ap.add_argument("--n4", action="store_true", help="fixed theta vs IBST per-site sparsity (N4)")
    ap.add_argument("--theta-fixed", type=float, default=0.05)
    ap.add_argument("--precision", default="bf16", choices=["fp32", "bf16"])
    args = ap.parse_args()

    import torch
    from paper_2410_20790_b200 import Encoder, ThresholdController

    cfg = W.get_config(args.config)
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    B, L = cfg.chunks_per_step, cfg.L
    net = cfg.build_net()
    enc = Encoder(net, max_chunks=B, max_frames=L, device=0, precision=args.precision)
    ns = enc.n_sites
    u8 = np.stack([W.gen_chunk(cfg.video_seed(c), L, cfg.h, cfg.w, cfg.c, **cfg.video) for c in range(B)])
    x = torch.from_numpy(W.to_float(u8)).to(dev)
    del u8
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    conv_ids = [i for i, l in enumerate(net.layers) if l["kind"] == W.CONV]
    conv_dense_rows = sum(B * (L - 1) * enc.layer_shape(i)[0] * enc.layer_shape(i)[1] for i in conv_ids)

    def step(th):
        enc.encode_reference(x[:, 0], stream)
        enc.encode_diff(x[:, 1:], th, stream)

    def timed(th, k):
        step(th)
        step(th)   # second sight of the key: graph captured
        torch.cuda.synchronize(dev)
        ms = 0.0
        for i in range(k):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(th)
            e1.record(stream)
            e1.synchronize()
            ms += e0.elapsed_time(e1)
        return ms / k

    def stats():
        _, sa, sp = enc.get_sparsity()
        lc = enc.layer_counts()
        site = [round(1 - a / p, 4) if p else None for a, p in zip(sa, sp)]
        rows = int(sum(lc["rows_out"][i] for i in conv_ids))
        return site, 1.0 - rows / conv_dense_rows

    # own dense path: every frame a reference frame (same kernels)
    denc = Encoder(net, max_chunks=B * L, max_frames=1, device=0, precision=args.precision)
    xd = x.reshape(B * L, cfg.h, cfg.w, cfg.c)
    zero_th = np.zeros(ns, np.float32)
    for _ in range(2):
        denc.encode_reference(xd, stream)
        denc.encode_diff(None, zero_th, stream)
    torch.cuda.synchronize(dev)
    dms = 0.0
    for i in range(args.steps):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        denc.encode_reference(xd, stream)
        denc.encode_diff(None, zero_th, stream)
        e1.record(stream)
        e1.synchronize()
        dms += e0.elapsed_time(e1)
    del denc
    dense_fps = B * L / (dms / args.steps / 1e3)
    doc = {"config": f"cfg{cfg.cid}: {cfg.note}", "precision": args.precision, "chunks": B, "frames": L,
           "dense_fps": dense_fps, "timing": "CUDA events on the launch stream, L2 flushed between steps"}

    if args.n4:
        out = {}
        for pol in ("fixed", "ibst"):
            ctl = ThresholdController(ns, policy=pol, T=cfg.T, eps=cfg.eps, theta_fixed=args.theta_fixed,
                                      cycle=cfg.cycle)
            for _ in range(args.max_calib):
                step(ctl.thresholds())
                _, sa, sp = enc.get_sparsity()
                ctl.observe(sa, sp)
            th = ctl.thresholds()
            ms = timed(th, args.steps)
            site, skip = stats()
            out[pol] = {"diff_fps": B * (L - 1) / (ms / 1e3), "ms_per_step": ms, "site_sparsity": site,
                        "site_sparsity_std": float(np.std([s for s in site[1:] if s is not None])),
                        "conv_row_skip": skip, "theta": [float(t) for t in th]}
        doc["n4"] = out
    else:
        levels = []
        for T in [float(t) for t in args.targets.split(",")]:
            ctl = ThresholdController(ns, policy="bst", T=T, eps=args.eps if args.eps is not None else cfg.eps)
            n_cal = 0
            for n_cal in range(1, args.max_calib + 1):
                step(ctl.thresholds())
                _, sa, sp = enc.get_sparsity()
                ctl.observe(sa, sp)
                if ctl.state()[3].all():
                    break
            th = ctl.thresholds()
            ms = timed(th, args.steps)
            site, skip = stats()
            fps = B * (L - 1) / (ms / 1e3)
            levels.append({"T": T, "calibration_steps": n_cal, "frozen": bool(ctl.state()[3].all()),
                           "diff_fps": fps, "ms_per_step": ms, "speedup_vs_dense": fps / dense_fps,
                           "mean_site_sparsity": float(np.mean([s for s in site if s is not None])),
                           "input_site_sparsity": site[0], "conv_row_skip": skip,
                           "theta": [round(float(t), 6) for t in th]})
            print(json.dumps(levels[-1]), file=sys.stderr)
        doc["levels"] = levels
    print(json.dumps(doc))


if __name__ == "__main__":
    main()
