#!/usr/bin/env python
"""Calibrated synthetic weights for the EfficientNet workloads (reading R30).

    python scripts/calibrate_weights.py --config 3 [--config 5 ...]

Trained weights are out of scope, and plain He-normal weights let
SiLU / squeeze-excitation stacks fade: without BatchNorm statistics the deep
EfficientNet sites carried almost no signal.  This
fixture script does what a trained network's folded BatchNorm does: for every
convolution, in topological order, it measures the per-channel mean and
standard deviation of the pre-activation on a calibration frame (frame 0 of
the config's chunk 0) and folds them into the weights, so every channel's
pre-activation has mean 0 and the layer's pre-activation has standard
deviation 1 on that frame; every SE
excitation is rescaled so its gate logits have mean 0.6 and standard
deviation 0.7 over channels (gates mostly inside [0.3, 0.85]).  The deviation is one per
layer (the per-channel means are removed): per-channel scaling would amplify
near-constant channels and make the random network chaotic.

It runs once, in fp64 with torch CPU library routines (F.conv2d etc.), and
writes only the per-channel fold factors -- w' = w * scale[c_out],
b' = b * scale + shift -- to workloads/calib/cfg<N>.npz (a few tens of KB),
which workloads.configs applies when it builds the config's network.  The
runtime path of workloads/ holds no arithmetic of the method; this script is
not imported by anything.  It also writes the per-site RMS table of the
calibrated network (dense, calibration frame) and the frame 0 -> 1 delta at
every tap to profiles/r02_calibration_cfg<N>.json.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from workloads import CONV, RELU, SILU, MAXPOOL, ADD, SE, OUTPUT  # noqa: E402

SE_LOGIT_STD = 0.7
SE_LOGIT_MEAN = 0.6


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64))


def _layer(l, a, b2=None):
    k = l["kind"]
    if k == CONV:
        return F.conv2d(a, _t(l["w"]), _t(l["b"]), stride=(l["s_h"], l["s_w"]), padding=(l["p_h"], l["p_w"]),
                        groups=l["groups"])
    if k == RELU:
        return torch.relu(a)
    if k == SILU:
        return a * torch.sigmoid(a)
    if k == MAXPOOL:
        return F.max_pool2d(a, (l["k_h"], l["k_w"]), (l["s_h"], l["s_w"]), (l["p_h"], l["p_w"]))
    if k == ADD:
        return a + b2
    if k == SE:
        return a * torch.sigmoid(_se_logits(l, a)).view(1, -1, 1, 1)
    return a


def _se_logits(l, a):
    m = a.mean(dim=(2, 3)).squeeze(0)
    h = _t(l["w"]) @ m + _t(l["b"])
    h = h * torch.sigmoid(h)
    return _t(l["w2"]) @ h + _t(l["b2"])


def _last_use(net):
    """Index of the last layer reading each layer's output (OUTPUT taps and
    sites are kept: the report reads them)."""
    last = {}
    for i, l in enumerate(net.layers):
        for s in (l["src"], l["src2"] if l["kind"] == ADD else -1):
            if s >= 0:
                last[s] = i
    return last


def _drop(net, outs, i, last, keep_sites):
    # free tensors whose last reader has run (B4-B6 at 1024-1280 px in fp64
    # would otherwise hold tens of GB); sites and taps are kept for the report
    for s in (net.layers[i]["src"], net.layers[i]["src2"] if net.layers[i]["kind"] == ADD else -1):
        if s >= 0 and last.get(s) == i and not (keep_sites and net.layers[s]["kind"] in W.NONLINEAR + (OUTPUT,)):
            outs[s] = None


def forward(net, frame):
    x = _t(frame).permute(2, 0, 1).unsqueeze(0)
    outs = []
    last = _last_use(net)
    for i, l in enumerate(net.layers):
        a = x if l["src"] < 0 else outs[l["src"]]
        b2 = None
        if l["kind"] == ADD:
            b2 = x if l["src2"] < 0 else outs[l["src2"]]
        outs.append(_layer(l, a, b2))
        _drop(net, outs, i, last, True)
    return outs


def calibrate(net, frame):
    """Fold per-channel statistics into the weights, layer by layer (fp64)."""
    x = _t(frame).permute(2, 0, 1).unsqueeze(0)
    outs = []
    fold = {}
    last = _last_use(net)
    for i, l in enumerate(net.layers):
        a = x if l["src"] < 0 else outs[l["src"]]
        if l["kind"] == CONV:
            y = _layer(l, a)
            mu = y.mean(dim=(0, 2, 3))
            # one scale per layer (LSUV-style), not per channel: dividing each
            # channel by its own deviation amplifies near-constant channels and
            # makes the random network chaotic -- frame-to-frame noise then
            # decorrelates the deep features, which a trained network does not do
            sd = float((y - mu.view(1, -1, 1, 1)).pow(2).mean().sqrt().clamp_min(1e-3))
            scale = np.full(mu.shape[0], 1.0 / sd)
            shift = (-mu / sd).numpy()
            # w' = w * scale, b' = b * scale + shift  ->  y' = (y - mu_c) / sd
            l["w"] = (l["w"].astype(np.float64) * scale[:, None, None, None]).astype(np.float32)
            l["b"] = (l["b"].astype(np.float64) * scale + shift).astype(np.float32)
            fold[f"s{i}"] = scale.astype(np.float64)
            fold[f"t{i}"] = shift.astype(np.float64)
        elif l["kind"] == SE:
            z = _se_logits(l, a)
            mu, sd = float(z.mean()), max(float(z.std()), 1e-3)
            scale = np.full(l["w2"].shape[0], SE_LOGIT_STD / sd)
            shift = np.full(l["w2"].shape[0], SE_LOGIT_MEAN - SE_LOGIT_STD * mu / sd)
            l["w2"] = (l["w2"].astype(np.float64) * scale[:, None]).astype(np.float32)
            l["b2"] = (l["b2"].astype(np.float64) * scale + shift).astype(np.float32)
            fold[f"s{i}"] = scale
            fold[f"t{i}"] = shift
        b2 = None
        if l["kind"] == ADD:
            b2 = x if l["src2"] < 0 else outs[l["src2"]]
        outs.append(_layer(l, a, b2))
        _drop(net, outs, i, last, False)
    return fold


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, action="append", required=True)
    args = ap.parse_args()
    torch.set_num_threads(os.cpu_count() or 1)
    os.makedirs(os.path.join(ROOT, "workloads", "calib"), exist_ok=True)
    for cid in args.config:
        cfg = W.get_config(cid)
        net = cfg.build_net(calibrated=False)
        u8 = W.gen_chunk(cfg.video_seed(0), 2, cfg.h, cfg.w, cfg.c, **cfg.video)
        fr = W.to_float(u8)
        fold = calibrate(net, fr[0])
        path = os.path.join(ROOT, "workloads", "calib", f"cfg{cid}.npz")
        np.savez_compressed(path, **{k: v.astype(np.float32) for k, v in fold.items()})
        # report: the network as workloads builds it from the saved factors
        net = cfg.build_net()
        o0, o1 = forward(net, fr[0]), forward(net, fr[1])
        sites = []
        for i, l in enumerate(net.layers):
            if l["kind"] in W.NONLINEAR:
                sites.append(dict(layer=i, kind=W.KIND_NAMES[l["kind"]], rms=float(o0[i].pow(2).mean().sqrt()),
                                  shape=list(o0[i].shape[1:])))
        taps = []
        for i, l in enumerate(net.layers):
            if l["kind"] == OUTPUT:
                d = (o1[i] - o0[i]).abs()
                pix = d.amax(dim=1)   # max over channels per pixel
                taps.append(dict(layer=i, rms=float(o0[i].pow(2).mean().sqrt()), delta_max=float(d.max()),
                                 delta_rms=float(d.pow(2).mean().sqrt()),
                                 pixels_over_0_05=float((pix > 0.05).double().mean())))
        rms = [s["rms"] for s in sites]
        rep = dict(config=cid, note=cfg.note, file=os.path.relpath(path, ROOT), se_logit_std=SE_LOGIT_STD,
                   site_rms_min=min(rms), site_rms_max=max(rms), sites=sites, taps=taps,
                   how="scripts/calibrate_weights.py: BN fold (per-channel mean, per-layer deviation) on frame 0 of chunk 0 (torch fp64)")
        out = os.path.join(ROOT, "profiles", f"r02_calibration_cfg{cid}.json")
        with open(out, "w") as f:
            json.dump(rep, f, indent=1)
        print(f"cfg{cid}: {len(fold) // 2} folded layers -> {path}; site rms [{min(rms):.3f}, {max(rms):.3f}]; "
              f"taps {[(t['layer'], round(t['rms'], 3), round(t['delta_max'], 4)) for t in taps]}")


if __name__ == "__main__":
    main()
