"""Network topologies as layer-spec lists, plus seeded weights.

A layer is a dict whose integer fields mirror ``st_layer_spec`` in
``include/sparsetem.h``:

    kind, src, src2, c_out, groups, k_h, k_w, s_h, s_w, p_h, p_w, se_hidden
    w, b, w2, b2   (numpy float32 arrays; None when unused)

``src`` is the producer layer index (-1 = network input).  Kinds:

* CONV    -- Eq.(1) convolution, PAPER.md P:119-122 (zero padding, groups,
             weights OIHW ``[c_out][c_in/groups][k_h][k_w]``, bias ``[c_out]``);
             BatchNorm is folded into w/b.
* RELU, SILU -- pointwise non-linearities.
* MAXPOOL -- window max, -inf padding (reading R11).
* ADD     -- residual join of ``src`` and ``src2`` (linear).
* SE      -- squeeze-excitation x * sigmoid(W2 silu(W1 mean(x) + b1) + b2)
             (EfficientNet block; reading R8).
* OUTPUT  -- an output tap: the dense per-frame output is accumulated here
             (Accumulation).

Truncation sites: the network input (site 0) and then every
RELU/SILU/MAXPOOL/SE layer in spec order.
"""
from __future__ import annotations

import math

import numpy as np

CONV, RELU, SILU, MAXPOOL, ADD, SE, OUTPUT = range(7)
KIND_NAMES = {CONV: "conv", RELU: "relu", SILU: "silu", MAXPOOL: "maxpool",
              ADD: "add", SE: "se", OUTPUT: "output"}
NONLINEAR = (RELU, SILU, MAXPOOL, SE)


def _out_dim(n, k, s, p):
    # geometry of SPEC S:59: floor((h + 2p - k)/s) + 1
    return (n + 2 * p - k) // s + 1


class Net:
    """Tiny topology builder.  Produces a list of layer dicts (no weights)."""

    def __init__(self, in_c, in_h, in_w, name="net"):
        self.in_c, self.in_h, self.in_w = in_c, in_h, in_w
        self.name = name
        self.layers: list[dict] = []

    def _add(self, **kw):
        base = dict(kind=None, src=-1, src2=-1, c_out=0, groups=1, k_h=1, k_w=1,
                    s_h=1, s_w=1, p_h=0, p_w=0, se_hidden=0,
                    w=None, b=None, w2=None, b2=None, act_gain=2.0, smooth=0.0)
        base.update(kw)
        self.layers.append(base)
        return len(self.layers) - 1

    def conv(self, src, c_out, k, s=1, p=None, groups=1, act_gain=2.0, smooth=0.0):
        kh, kw = (k, k) if isinstance(k, int) else k
        sh, sw = (s, s) if isinstance(s, int) else s
        if p is None:
            p = (kh // 2, kw // 2)
        ph, pw = (p, p) if isinstance(p, int) else p
        return self._add(kind=CONV, src=src, c_out=c_out, groups=groups, k_h=kh, k_w=kw,
                         s_h=sh, s_w=sw, p_h=ph, p_w=pw, act_gain=act_gain, smooth=smooth)

    def relu(self, src):
        return self._add(kind=RELU, src=src)

    def silu(self, src):
        return self._add(kind=SILU, src=src)

    def maxpool(self, src, k, s, p=0):
        kh, kw = (k, k) if isinstance(k, int) else k
        sh, sw = (s, s) if isinstance(s, int) else s
        ph, pw = (p, p) if isinstance(p, int) else p
        return self._add(kind=MAXPOOL, src=src, k_h=kh, k_w=kw, s_h=sh, s_w=sw, p_h=ph, p_w=pw)

    def add(self, a, b):
        return self._add(kind=ADD, src=a, src2=b)

    def se(self, src, hidden):
        return self._add(kind=SE, src=src, se_hidden=hidden)

    def output(self, src):
        return self._add(kind=OUTPUT, src=src)


def infer_shapes(net: Net):
    """(h, w, c) of every layer's output.  Plumbing for buffer allocation."""
    shapes = []
    for l in net.layers:
        def sh(i):
            return (net.in_h, net.in_w, net.in_c) if i < 0 else shapes[i]
        h, w, c = sh(l["src"])
        k = l["kind"]
        if k == CONV:
            shapes.append((_out_dim(h, l["k_h"], l["s_h"], l["p_h"]),
                           _out_dim(w, l["k_w"], l["s_w"], l["p_w"]), l["c_out"]))
        elif k == MAXPOOL:
            shapes.append((_out_dim(h, l["k_h"], l["s_h"], l["p_h"]),
                           _out_dim(w, l["k_w"], l["s_w"], l["p_w"]), c))
        elif k == ADD:
            assert sh(l["src2"]) == (h, w, c), "ADD operands differ in shape"
            shapes.append((h, w, c))
        else:
            shapes.append((h, w, c))
    return shapes


def site_layers(net: Net):
    """Layer index of every truncation site; entry 0 (-1) is the network input."""
    return [-1] + [i for i, l in enumerate(net.layers) if l["kind"] in NONLINEAR]


def init_weights(net: Net, seed: int):
    """Seeded synthetic weights (trained weights are out of scope).

    CONV: He-normal, std = sqrt(gain / fan_in), fan_in = (c_in/groups)*k_h*k_w,
    so activations stay O(1) through ReLU/SiLU stacks (DESIGN.md input recipe);
    bias ~ U(-0.1, 0.1) (BatchNorm folded).  A spatial conv with
    ``smooth`` = s > 0 (reading R30) mixes in a smooth component: every
    (c_out, c_in) kernel becomes s * a * G * |w| + (1 - s) * w, with G a
    Gaussian blob of unit sum (sigma = k/4), a ~ N(0, 1) and |w| the He
    kernel's norm (so the smooth part's gain on flat content is O(1)) --
    trained low-level filters pass smooth image content; pure white-noise
    kernels act as high-pass filters, and once a BatchNorm fold rescales their
    output they amplify frame noise and rounding layer after layer.
    SE: FC1 [hidden][C] std 1/sqrt(C), FC2 [C][hidden] std 1/sqrt(hidden),
    biases small, so gates sit mid-range.
    Returns the same Net with w/b filled (float32, C-contiguous).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    shapes = infer_shapes(net)
    for i, l in enumerate(net.layers):
        src_c = net.in_c if l["src"] < 0 else shapes[l["src"]][2]
        if l["kind"] == CONV:
            cin_g = src_c // l["groups"]
            fan_in = cin_g * l["k_h"] * l["k_w"]
            std = math.sqrt(l["act_gain"] / fan_in)
            w = rng.standard_normal((l["c_out"], cin_g, l["k_h"], l["k_w"])) * std
            l["b"] = rng.uniform(-0.1, 0.1, l["c_out"]).astype(np.float32)
            sm = float(l.get("smooth", 0.0))
            if sm > 0 and l["k_h"] * l["k_w"] > 1:
                ay = np.arange(l["k_h"]) - l["k_h"] // 2
                ax = np.arange(l["k_w"]) - l["k_w"] // 2
                G = np.exp(-(ay[:, None] ** 2 / (2 * (l["k_h"] / 4) ** 2) + ax[None, :] ** 2 / (2 * (l["k_w"] / 4) ** 2)))
                G /= G.sum()
                a = rng.standard_normal((l["c_out"], cin_g))[:, :, None, None]
                nrm = np.sqrt((w * w).sum(axis=(2, 3), keepdims=True))
                w = sm * a * G * nrm + (1 - sm) * w
            l["w"] = w.astype(np.float32)
        elif l["kind"] == SE:
            c, hd = src_c, l["se_hidden"]
            l["w"] = (rng.standard_normal((hd, c)) / math.sqrt(c)).astype(np.float32)
            l["b"] = rng.uniform(-0.1, 0.1, hd).astype(np.float32)
            l["w2"] = (rng.standard_normal((c, hd)) / math.sqrt(hd)).astype(np.float32)
            l["b2"] = rng.uniform(-0.5, 0.5, c).astype(np.float32)
    return net


def apply_fold(net: Net, path: str):
    """Apply committed per-channel fold factors (reading R30): for CONV layer
    i, w' = w * s_i[c_out], b' = b * s_i + t_i; for SE layer i the excitation
    FC2, w2' = w2 * s_i[c], b2' = b2 * s_i + t_i.  Weight construction only
    (the factors come from scripts/calibrate_weights.py)."""
    f = np.load(path)
    for i, l in enumerate(net.layers):
        if f"s{i}" not in f:
            continue
        s = f[f"s{i}"].astype(np.float64)
        t = f[f"t{i}"].astype(np.float64)
        if l["kind"] == CONV:
            l["w"] = (l["w"].astype(np.float64) * s[:, None, None, None]).astype(np.float32)
            l["b"] = (l["b"].astype(np.float64) * s + t).astype(np.float32)
        elif l["kind"] == SE:
            l["w2"] = (l["w2"].astype(np.float64) * s[:, None]).astype(np.float32)
            l["b2"] = (l["b2"].astype(np.float64) * s + t).astype(np.float32)
    return net


# ----------------------------------------------------------------------------
# The five BASELINE.json topologies
# ----------------------------------------------------------------------------

def toy_encoder(h=64, w=64):
    """cfg1: 3x3 conv 3->16 + ReLU + 1x1 conv 16->8 (BASELINE.json configs[0])."""
    n = Net(3, h, w, "toy")
    c1 = n.conv(-1, 16, 3)
    r1 = n.relu(c1)
    c2 = n.conv(r1, 8, 1, act_gain=1.0)
    n.output(c2)
    return n


def crnn_vgg7(h=32, w=128):
    """cfg2: CRNN conv encoder, VGG-style, 7 convs (SURVEY reading R27).

    Conv64-P2-Conv128-P2-Conv256-Conv256-P((2,2),(2,1),(0,1))-Conv512-Conv512-
    P(same)-Conv512 2x2 valid; every conv followed by ReLU; output 512x1x33.
    """
    n = Net(1, h, w, "crnn_vgg7")
    x = n.relu(n.conv(-1, 64, 3))
    x = n.maxpool(x, 2, 2)
    x = n.relu(n.conv(x, 128, 3))
    x = n.maxpool(x, 2, 2)
    x = n.relu(n.conv(x, 256, 3))
    x = n.relu(n.conv(x, 256, 3))
    x = n.maxpool(x, (2, 2), (2, 1), (0, 1))
    x = n.relu(n.conv(x, 512, 3))
    x = n.relu(n.conv(x, 512, 3))
    x = n.maxpool(x, (2, 2), (2, 1), (0, 1))
    x = n.relu(n.conv(x, 512, 2, 1, 0))
    n.output(x)
    return n


def resnet18(h=720, w=1280):
    """cfg4: torchvision ResNet-18 topology without avgpool/fc (reading R28)."""
    n = Net(3, h, w, "resnet18")
    x = n.relu(n.conv(-1, 64, 7, 2, 3))
    x = n.maxpool(x, 3, 2, 1)
    c = 64
    for stage, (co, s) in enumerate([(64, 1), (128, 2), (256, 2), (512, 2)]):
        for blk in range(2):
            stride = s if blk == 0 else 1
            y = n.relu(n.conv(x, co, 3, stride, 1))
            y = n.conv(y, co, 3, 1, 1, act_gain=1.0)
            if stride != 1 or c != co:
                sc = n.conv(x, co, 1, stride, 0, act_gain=1.0)
            else:
                sc = x
            x = n.relu(n.add(y, sc))
            c = co
    n.output(x)
    return n


def resnet152(h=320, w=320):
    """ResNet-152, the paper's CRNN backbone for action
    recognition (224/320/420 inputs, chunk 28, batch 3);
    torchvision topology (bottleneck blocks [3, 8, 36, 3], stride on the 3x3)
    without avgpool/fc, output layer4 (2048 channels).  The last 1x1 conv of
    each residual branch uses gain 0.25 so 50 residual additions keep the
    synthetic activations O(1) (reading R30: data-independent weights)."""
    n = Net(3, h, w, "resnet152")
    x = n.relu(n.conv(-1, 64, 7, 2, 3))
    x = n.maxpool(x, 3, 2, 1)
    c = 64
    for width, blocks, s in [(64, 3, 1), (128, 8, 2), (256, 36, 2), (512, 3, 2)]:
        co = 4 * width
        for blk in range(blocks):
            stride = s if blk == 0 else 1
            y = n.relu(n.conv(x, width, 1, 1, 0))
            y = n.relu(n.conv(y, width, 3, stride, 1))
            y = n.conv(y, co, 1, 1, 0, act_gain=0.25)
            if stride != 1 or c != co:
                sc = n.conv(x, co, 1, stride, 0, act_gain=1.0)
            else:
                sc = x
            x = n.relu(n.add(y, sc))
            c = co
    n.output(x)
    return n


SPATIAL_SMOOTH = 0.7   # EfficientNet spatial kernels (stem, depthwise), reading R30


# EfficientNet compound scaling (width, depth) of the backbones of
# EfficientDet-D0 (B0) and of the paper's Table 1 detectors d4 / d5 / d6
# (B4 / B5 / B6)
EFFNET_SCALE = {"b0": (1.0, 1.0), "b4": (1.4, 1.8), "b5": (1.6, 2.2), "b6": (1.8, 2.6)}


def _round_filters(c, width):
    """Channels scaled by width, rounded to a multiple of 8 (never below 90%)."""
    if width == 1.0:
        return c
    v = c * width
    r = max(8, int(v + 4) // 8 * 8)
    return r + 8 if r < 0.9 * v else r


def efficientnet_b0(h=512, w=512):
    """cfg3/cfg5: EfficientNet-B0 backbone (EfficientDet-D0), taps P3/P4/P5."""
    return efficientnet(h, w, "b0")


def efficientnet(h=512, w=512, variant="b0"):
    """EfficientNet-B<v> backbone, taps P3/P4/P5.

    MBConv: [1x1 expand -> SiLU] -> kxk depthwise -> SiLU -> SE -> 1x1 project
    (+ residual when stride 1 and c_in == c_out).  Symmetric k//2 padding
    (reading R11).  Taps = outputs of stages 3/5/7 (reading R13).  B4-B6 scale
    every stage's channels by the width factor (multiples of 8) and its
    repeats by ceil(depth * repeats); the SE width is a quarter of the block's
    input channels, as in B0.
    """
    width, depth = EFFNET_SCALE[variant]
    n = Net(3, h, w, f"efficientnet_{variant}")
    c = _round_filters(32, width)
    x = n.silu(n.conv(-1, c, 3, 2, 1, smooth=SPATIAL_SMOOTH))
    stages = [  # expand, k, stride, c_out, repeats
        (1, 3, 1, 16, 1), (6, 3, 2, 24, 2), (6, 5, 2, 40, 2), (6, 3, 2, 80, 3),
        (6, 5, 1, 112, 3), (6, 5, 2, 192, 4), (6, 3, 1, 320, 1)]
    for si, (e, k, s, co, rep) in enumerate(stages):
        co = _round_filters(co, width)
        rep = int(math.ceil(depth * rep))
        for r in range(rep):
            stride = s if r == 0 else 1
            inp = x
            ce = c * e
            y = x
            if e != 1:
                y = n.silu(n.conv(y, ce, 1, 1, 0))
            y = n.silu(n.conv(y, ce, k, stride, k // 2, groups=ce, smooth=SPATIAL_SMOOTH))
            y = n.se(y, max(1, c // 4))
            y = n.conv(y, co, 1, 1, 0, act_gain=1.0)
            if stride == 1 and c == co:
                y = n.add(y, inp)
            x = y
            c = co
        if si in (2, 4, 6):
            n.output(x)
    return n
