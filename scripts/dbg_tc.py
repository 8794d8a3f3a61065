"""Debug: CRNN cfg2 small run, BF16, per-layer finite check (debug on / off)."""
import sys
import numpy as np
sys.path.insert(0, "tests")
import oracle
import workloads as W
from gpu_harness import gpu_run, make_frames

cfg = W.get_config(2)
net = cfg.build_net()
fr = make_frames(cfg, 2, L=8)
for debug in (True, False):
    enc, _ = gpu_run(net, fr, 0.0, precision="bf16", debug=debug)
    tap = enc.taps[0]
    out = enc.outputs(tap).cpu().numpy()
    print("debug", debug, "tap finite", np.isfinite(out).all(), "max", np.nanmax(np.abs(out[np.isfinite(out)])))
    if debug:
        r = oracle.run_chunk(net, fr[0], 0.0, want_deltas=True, precision="bf16")
        for i, l in enumerate(net.layers[:-1]):
            bad = 0; err = 0.0; n = 0
            for t in range(1, 8):
                idx, rows = enc.debug_rows(i, 0, t)
                fin = np.isfinite(rows).all()
                exp = r["deltas"][i][t - 1].reshape(-1, rows.shape[1])[idx] if rows.ndim == 2 else None
                if not fin: bad += 1
                if exp is not None and fin and rows.size:
                    err = max(err, float(np.max(np.abs(rows - exp)) / (np.sqrt(np.mean(exp ** 2)) + 1e-9)))
                n += rows.shape[0]
            print(f"layer {i} kind {l['kind']} nonfinite_frames {bad} rows {n} max_err/rms {err:.3e}")
