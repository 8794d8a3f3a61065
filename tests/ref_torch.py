"""Independent fp64 dense reference built from library routines (torch CPU).

Used only to PIN the oracle (tests -m "not gpu"): Eq.(1) convolution is
``torch.nn.functional.conv2d`` (cross-correlation, zero padding, groups --
exactly Eq.(1) of PAPER.md P:119-122), max pooling is
``torch.nn.functional.max_pool2d`` (-inf padding), SiLU/sigmoid from torch.
Nothing here is shared with the oracle or the CUDA path.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from workloads import CONV, RELU, SILU, MAXPOOL, ADD, SE, OUTPUT


def _nchw(x):  # [H][W][C] -> [1][C][H][W] float64
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).permute(2, 0, 1).unsqueeze(0)


def _hwc(t):
    return t.squeeze(0).permute(1, 2, 0).contiguous().numpy()


def dense_forward64(net, frame):
    """fp64 dense forward of one frame [H][W][C]; list of per-layer [H][W][C]."""
    x = _nchw(frame)
    outs = []
    for l in net.layers:
        a = x if l["src"] < 0 else outs[l["src"]]
        k = l["kind"]
        if k == CONV:
            w = torch.from_numpy(l["w"].astype(np.float64))
            b = torch.from_numpy(l["b"].astype(np.float64))
            y = F.conv2d(a, w, b, stride=(l["s_h"], l["s_w"]), padding=(l["p_h"], l["p_w"]),
                         groups=l["groups"])
        elif k == RELU:
            y = torch.relu(a)
        elif k == SILU:
            y = a * torch.sigmoid(a)
        elif k == MAXPOOL:
            y = F.max_pool2d(a, (l["k_h"], l["k_w"]), (l["s_h"], l["s_w"]), (l["p_h"], l["p_w"]))
        elif k == ADD:
            b2 = x if l["src2"] < 0 else outs[l["src2"]]
            y = a + b2
        elif k == SE:
            m = a.mean(dim=(2, 3)).squeeze(0)
            h = torch.from_numpy(l["w"].astype(np.float64)) @ m + torch.from_numpy(l["b"].astype(np.float64))
            h = h * torch.sigmoid(h)
            z = torch.from_numpy(l["w2"].astype(np.float64)) @ h + torch.from_numpy(l["b2"].astype(np.float64))
            y = a * torch.sigmoid(z).view(1, -1, 1, 1)
        elif k == OUTPUT:
            y = a
        else:
            raise ValueError(k)
        outs.append(y)
    return [_hwc(o) for o in outs]


def close(a, b, rel=1e-4, abs_=1e-5):
    """Elementwise |a-b| <= abs + rel*|b| (reading R29)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return bool(np.all(np.abs(a - b) <= abs_ + rel * np.abs(b)))


def max_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / (1e-5 + 1e-4 * np.abs(b)))) if a.size else 0.0
