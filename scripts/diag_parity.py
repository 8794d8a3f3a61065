#!/usr/bin/env python
"""Per-layer parity diagnostics (debug retention + band-follow) of one chunk.

    python scripts/diag_parity.py --config 3 --frames 7 --precision bf16
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
import oracle  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--frames", type=int, default=7)
ap.add_argument("--precision", default="bf16")
ap.add_argument("--theta", type=float, default=0.05)
a = ap.parse_args()
import torch  # noqa: E402
from paper_2410_20790_b200 import Encoder  # noqa: E402

cfg = W.get_config(a.config)
net = cfg.build_net()
L = a.frames
fr = W.to_float(W.gen_video(1, L, cfg.h, cfg.w, cfg.c, cfg.video_seed(0), **cfg.video))
enc = Encoder(net, 1, L, precision=a.precision, debug_retain=True)
x = torch.from_numpy(fr).cuda()
enc.encode_reference(x[:, 0])
enc.encode_diff(x[:, 1:], a.theta)
torch.cuda.synchronize()
follow = {i: np.stack([enc.debug_mask(i, 0, t) for t in range(1, L)])
          for i, l in enumerate(net.layers) if l["kind"] in W.NONLINEAR}
r = oracle.run_chunk(net, fr[0], a.theta, want_deltas=True, want_dense0=True, precision=a.precision, follow=follow)
fs = r["follow_stats"]
for i, l in enumerate(net.layers):
    if l["kind"] == W.OUTPUT:
        got = enc.outputs(i)[0].cpu().numpy().astype(np.float64)
        ref = r["taps"][i].astype(np.float64)
        e = np.abs(got - ref)
        print(f"TAP {i}: max err {e.max():.4g} rms {np.sqrt(np.mean(ref**2)):.4g} per-frame max {[round(float(v),4) for v in e.reshape(L,-1).max(1)]}")
        continue
    d0g = enc.debug_dense0(i, 0).astype(np.float64)
    d0o = r["dense0"][i].astype(np.float64)
    de = np.abs(d0g - d0o).max()
    errs = []
    for t in range(1, L):
        m = enc.debug_mask(i, 0, t)
        if not np.array_equal(m, r["masks"][i][t - 1]):
            errs.append("MASK")
            continue
        idx, rows = enc.debug_rows(i, 0, t)
        exp = r["deltas"][i][t - 1].reshape(-1, rows.shape[1])[idx]
        errs.append(float(np.abs(rows - exp).max()) if rows.size else 0.0)
    print(f"{i:3d} {W.KIND_NAMES[l['kind']]:7s} src {l['src']:3d} dense0 err {de:.3g} (rms {np.sqrt(np.mean(d0o**2)):.3g}) "
          f"rows max err/frame {[e if isinstance(e, str) else round(e, 4) for e in errs]} follow {fs[i].tolist()}")
