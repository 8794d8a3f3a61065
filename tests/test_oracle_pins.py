"""Pins of the CPU oracle against what the paper and mathematics fix.

Every test here runs without a GPU (-m "not gpu").  Each checks the oracle
against something other than itself: torch fp64 library routines
(ref_torch.py), closed forms implied by Eq.(2), brute force, the paper's
printed example (tests/golden/nine_pixels.json), or SPEC worked
examples (tests/golden/spec_examples.json).  PIN numbers follow SURVEY §8(c).
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import workloads as W
from workloads import Net, init_weights, CONV, RELU, SILU, MAXPOOL, ADD, SE, OUTPUT
from ref_torch import dense_forward64, close, max_err
from netgen import random_net, random_frames

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _single(kind_fn, in_c, h, w, seed=0):
    n = Net(in_c, h, w)
    x = kind_fn(n)
    n.output(x)
    init_weights(n, seed)
    return n


# ------------------------------------------------------------------ dense
@pytest.mark.parametrize("seed", range(40))
def test_dense_matches_torch_fp64(oracle_lib, seed):
    """Oracle dense forward (Eq.1 etc.) == torch fp64 routines within R29."""
    net = random_net(seed)
    x = np.random.default_rng(seed).random((net.in_h, net.in_w, net.in_c)).astype(np.float32)
    ours = oracle.dense_forward(net, x)
    ref = dense_forward64(net, x)
    for i, (a, b) in enumerate(zip(ours, ref)):
        assert a.shape == b.shape, (i, a.shape, b.shape)
        assert close(a, b), (seed, i, W.KIND_NAMES[net.layers[i]["kind"]], max_err(a, b))


def test_dense_models_match_torch(oracle_lib):
    """cfg1 and a reduced-resolution CRNN / ResNet-18 / EfficientNet-B0 /
    ResNet-152 (N3, 2048-channel stages)."""
    for net in (W.models.toy_encoder(16, 16), W.models.crnn_vgg7(32, 64),
                W.models.resnet18(64, 64), W.models.efficientnet_b0(64, 64), W.models.resnet152(64, 64)):
        init_weights(net, 5)
        x = np.random.default_rng(1).random((net.in_h, net.in_w, net.in_c)).astype(np.float32)
        ours = oracle.dense_forward(net, x)
        ref = dense_forward64(net, x)
        # fp32 (oracle) vs fp64 rounding differences accumulate with depth: the
        # 155-conv ResNet-152 gets a 10x wider bound (still orders of magnitude
        # below the O(1) error of a dropped term or a wrong index)
        k = 10.0 if net.name == "resnet152" else 1.0
        for i, (a, b) in enumerate(zip(ours, ref)):
            assert close(a, b, rel=3e-4 * k, abs_=3e-5 * k), (net.name, i, max_err(a, b))


def test_dense_spec_scalars(oracle_lib):
    g = _gold("spec_examples.json")
    e = g["dense_scalar_conv"]
    n = Net(1, 1, 1)
    c = n.conv(-1, 1, 1, 1, 0)
    n.output(c)
    n.layers[c]["w"] = np.array([[[[e["w"]]]]], np.float32)
    n.layers[c]["b"] = np.array([e["b"]], np.float32)
    y = oracle.dense_forward(n, np.array([[[e["x"]]]], np.float32))
    assert y[-1][0, 0, 0] == e["expect"]
    n = Net(1, 3, 3)
    c = n.conv(-1, 1, 3, 1, 0)
    n.output(c)
    n.layers[c]["w"] = np.ones((1, 1, 3, 3), np.float32)
    n.layers[c]["b"] = np.zeros(1, np.float32)
    y = oracle.dense_forward(n, np.ones((3, 3, 1), np.float32))
    assert y[-1].shape == (1, 1, 1) and y[-1][0, 0, 0] == g["dense_window_sum"]["expect"]


# ------------------------------------------------------- PIN1 theta = 0
@pytest.mark.parametrize("seed", range(24))
@pytest.mark.parametrize("order", [0, 1])
def test_pin1_zero_threshold_equals_dense(oracle_lib, seed, order):
    """theta = 0 everywhere => per-frame diff output == dense output
    (Eq.2 linearity + Eq.3 correction), against torch fp64."""
    net = random_net(100 + seed)
    L = 8
    fr = random_frames(seed, L, net.in_h, net.in_w, net.in_c)
    r = oracle.run_chunk(net, fr, 0.0, layer_outer=bool(order))
    tap = [i for i, l in enumerate(net.layers) if l["kind"] == OUTPUT][0]
    for t in range(L):
        ref = dense_forward64(net, fr[t])[tap]
        assert close(r["taps"][tap][t], ref, rel=2e-4, abs_=2e-5), (seed, t, max_err(r["taps"][tap][t], ref))


def test_pin1_models_zero_threshold(oracle_lib):
    for net in (W.models.toy_encoder(24, 24), W.models.crnn_vgg7(32, 48), W.models.resnet18(48, 48),
                W.models.efficientnet_b0(64, 64), W.models.resnet152(40, 40)):
        init_weights(net, 3)
        fr = random_frames(7, 4, net.in_h, net.in_w, net.in_c, p_change=0.2, scale=0.2)
        r = oracle.run_chunk(net, fr, 0.0, want_masks=False)
        k = 10.0 if net.name == "resnet152" else 1.0   # depth-accumulated fp32 rounding, as above
        for tap, O in r["taps"].items():
            for t in range(4):
                ref = dense_forward64(net, fr[t])[tap]
                assert close(O[t], ref, rel=5e-4 * k, abs_=5e-5 * k), (net.name, tap, t, max_err(O[t], ref))


# ---------------------------------------------- PIN2 input-only threshold
@pytest.mark.parametrize("seed", range(10))
def test_pin2_input_threshold_only(oracle_lib, seed):
    """theta_0 > 0, all other theta = 0  =>  output_t = dense(S_t), S_t the
    propagated Subtraction buffer (closed form of Eq.2 + Eq.3 at theta=0)."""
    net = random_net(300 + seed)
    L, th0 = 8, 0.15
    fr = random_frames(seed + 50, L, net.in_h, net.in_w, net.in_c, p_change=0.5, scale=0.2)
    ns = oracle.num_sites(net)
    th = np.zeros(ns, np.float32)
    th[0] = th0
    r = oracle.run_chunk(net, fr, th)
    # S_t by the buffer rule (R3), written out independently here
    S = fr[0].copy()
    tap = [i for i, l in enumerate(net.layers) if l["kind"] == OUTPUT][0]
    for t in range(1, L):
        raw = fr[t] - S
        act = np.abs(raw).max(axis=2) > np.float32(th0)
        S = np.where(act[..., None], S + raw, S).astype(np.float32)
        ref = dense_forward64(net, S)[tap]
        assert close(r["taps"][tap][t], ref, rel=2e-4, abs_=2e-5), (seed, t)


# ---------------------------------------------------- PIN3 identical frames
def test_pin3_identical_frames(oracle_lib):
    net = random_net(7)
    fr = np.repeat(random_frames(1, 1, net.in_h, net.in_w, net.in_c), 6, axis=0)
    r = oracle.run_chunk(net, fr, 0.0)
    assert all(m.sum() == 0 for m in r["masks"].values())
    assert r["counts"].sum() == 0
    for O in r["taps"].values():
        for t in range(1, 6):
            assert np.array_equal(O[t], O[0])


# ------------------------------------------------ PIN4 nine pixels
def test_pin4_nine_pixels(oracle_lib):
    g = _gold("nine_pixels.json")
    H, Wd = g["map_hw"]
    for case in g["cases"]:
        n = Net(1, H, Wd)
        c = n.conv(-1, 2, tuple(g["kernel"]), tuple(g["stride"]), tuple(g["pad"]))
        n.output(c)
        init_weights(n, 0)
        fr = np.zeros((2, H, Wd, 1), np.float32)
        fr[1, case["pixel"][0], case["pixel"][1], 0] = 1.0
        r = oracle.run_chunk(n, fr, 0.0)
        m = r["masks"][c][0]
        assert m.sum() == case["active_out"]
        r0, r1 = case["block_rows"]
        c0, c1 = case["block_cols"]
        assert m[r0:r1 + 1, c0:c1 + 1].all()


def test_pin4_conv_bias_absent(oracle_lib):
    e = _gold("spec_examples.json")["conv_bias_absent"]
    H, Wd = e["map_hw"]
    n = Net(1, H, Wd)
    c = n.conv(-1, 1, 3, 1, 1)
    n.output(c)
    n.layers[c]["w"] = np.full((1, 1, 3, 3), e["kernel_value"], np.float32)
    n.layers[c]["b"] = np.array([e["bias"]], np.float32)
    fr = np.zeros((2, H, Wd, 1), np.float32)
    fr[1, e["pixel"][0], e["pixel"][1], 0] = e["delta"]
    r = oracle.run_chunk(n, fr, 0.0, want_deltas=True)
    m, d = r["masks"][c][0], r["deltas"][c][0]
    assert m.sum() == e["expect_active"]
    assert np.all(d[m.astype(bool)] == e["expect_value"])
    assert np.all(d[~m.astype(bool)] == 0)


# ------------------------------------------- PIN5 accumulation identity
@pytest.mark.parametrize("seed", range(8))
def test_pin5_accumulation(oracle_lib, seed):
    """O_t = O_0 + sum_{t'<=t} delta_tap(t'), checked in fp64, and
    pixels outside the tap mask are bit-identical to frame t-1."""
    net = random_net(500 + seed)
    L = 7
    fr = random_frames(seed, L, net.in_h, net.in_w, net.in_c)
    r = oracle.run_chunk(net, fr, 0.05, want_deltas=True)
    tap = [i for i, l in enumerate(net.layers) if l["kind"] == OUTPUT][0]
    O = r["taps"][tap].astype(np.float64)
    D = r["deltas"][tap].astype(np.float64)
    M = r["masks"][tap]
    for t in range(1, L):
        np.testing.assert_allclose(O[t], O[0] + D[:t].sum(0), rtol=1e-5, atol=1e-5)
        off = ~M[t - 1].astype(bool)
        assert np.array_equal(r["taps"][tap][t][off], r["taps"][tap][t - 1][off])


# -------------------------------------- PIN6 truncation rule / conservation
@pytest.mark.parametrize("seed", range(20))
def test_pin6_input_truncation(oracle_lib, seed):
    """Site 0: emitted = raw at masked pixels, residual = raw elsewhere,
    emitted + residual == raw bit-exact, max|raw| > theta iff masked (P:143,
    R1/R2)."""
    rng = np.random.default_rng(seed)
    net = _single(lambda n: n.relu(-1), 2, 6, 7, seed)
    L = 9
    fr = random_frames(seed, L, 6, 7, 2, p_change=0.6, scale=0.1)
    th = float(rng.uniform(0.01, 0.2))
    r = oracle.run_chunk(net, fr, [th, 0.0], want_deltas=True)
    D = r["deltas"][0]   # relu layer delta is not the input delta -> recompute input deltas
    S = fr[0].copy()
    for t in range(1, L):
        raw = (fr[t] - S).astype(np.float32)
        mx = np.abs(raw).max(axis=2)
        act = mx > np.float32(th)
        emitted = np.where(act[..., None], raw, 0).astype(np.float32)
        residual = np.where(act[..., None], 0, raw).astype(np.float32)
        assert np.array_equal(emitted + residual, raw)
        assert not np.any(act & (mx <= th))
        assert int(act.sum()) == r["counts"][0][t - 1]
        S = (S + emitted).astype(np.float32)
    assert D.shape[0] == L - 1


@pytest.mark.parametrize("case", ["subtract_one_pixel", "truncate_all_below", "truncate_pixel_granular"])
def test_pin6_spec_truncation_examples(oracle_lib, case):
    e = _gold("spec_examples.json")[case]
    net = _single(lambda n: n.relu(-1), 2, 1, 1)
    ref = np.array(e.get("ref", [0.0, 0.0]), np.float32)
    new = np.array(e.get("new", e.get("delta")), np.float32) + ref
    fr = np.stack([ref, new]).reshape(2, 1, 1, 2)
    r = oracle.run_chunk(net, fr, [e["theta"], 0.0])
    assert bool(r["counts"][0][0]) == e["expect_emitted"]


# ------------------------------------------------ PIN7 bounded residual
@pytest.mark.parametrize("seed", range(10))
def test_pin7_bounded_residual(oracle_lib, seed):
    """max_c |f(x_acc) - y_acc| <= theta at every pixel after truncation
    (SPEC S:250): x_acc = x0 + sum input deltas, y_acc = y0 + sum
    emitted, rebuilt here from the oracle's outputs with fp32 adds."""
    net = Net(2, 9, 9)
    c = net.conv(-1, 6, 3)
    a = net.relu(c)
    c2 = net.conv(a, 4, 3)
    s2 = net.silu(c2)
    net.output(s2)
    init_weights(net, seed)
    L, th = 8, 0.07
    fr = random_frames(seed, L, 9, 9, 2, p_change=0.5, scale=0.3)
    r = oracle.run_chunk(net, fr, th, want_deltas=True, want_dense0=True)
    for src, site, f in ((c, a, lambda x: np.maximum(x, 0)),
                         (c2, s2, lambda x: x / (1 + np.exp(-x.astype(np.float64))))):
        xa = r["dense0"][src].copy()
        ya = r["dense0"][site].copy()
        for t in range(L - 1):
            xa = (xa + r["deltas"][src][t]).astype(np.float32)
            ya = (ya + r["deltas"][site][t]).astype(np.float32)
            res = np.abs(f(xa) - ya).max(axis=2)
            assert res.max() <= th + 1e-6, (seed, t, res.max())


# ------------------------------------------------ PIN8 brute force deltas
@pytest.mark.parametrize("seed", range(12))
def test_pin8_conv_delta_bruteforce(oracle_lib, seed):
    """Eq.(2): delta_out = conv(X_t) - conv(X_{t-1}) exactly in fp64 where the
    input delta is exact (theta = 0), bias absent; off-mask exactly 0."""
    rng = np.random.default_rng(seed)
    k = int(rng.choice([1, 2, 3]))
    s = int(rng.choice([1, 2]))
    p = int(rng.integers(0, k // 2 + 1))
    cin, cout = int(rng.integers(1, 3)), int(rng.integers(1, 4))
    n = Net(cin, 8, 9)
    c = n.conv(-1, cout, k, s, p)
    n.output(c)
    init_weights(n, seed)
    fr = random_frames(seed, 4, 8, 9, cin, p_change=0.25)
    r = oracle.run_chunk(n, fr, 0.0, want_deltas=True)
    for t in range(1, 4):
        a = dense_forward64(n, fr[t])[c]
        b = dense_forward64(n, fr[t - 1])[c]
        assert close(r["deltas"][c][t - 1], a - b, rel=1e-4, abs_=1e-5)
        m = r["masks"][c][t - 1].astype(bool)
        assert np.all(r["deltas"][c][t - 1][~m] == 0)


@pytest.mark.parametrize("case", ["relu_dead_zone", "relu_cross_zero"])
def test_pin8_relu_spec(oracle_lib, case):
    e = _gold("spec_examples.json")[case]
    net = _single(lambda n: n.relu(-1), 1, 1, 1)
    fr = np.array([e["x_ref"], e["x_new"]], np.float32).reshape(2, 1, 1, 1)
    r = oracle.run_chunk(net, fr, [0.0, e["theta"]], want_deltas=True)
    assert bool(r["masks"][0][0, 0, 0]) == e["expect_emitted"]
    assert r["deltas"][0][0, 0, 0, 0] == e["expect_value"]


def test_pin8_maxpool_spec(oracle_lib):
    e = _gold("spec_examples.json")["maxpool_window"]
    net = _single(lambda n: n.maxpool(-1, 2, 2), 1, 2, 2)
    fr = np.array([e["window_ref"], e["window_new"]], np.float32).reshape(2, 2, 2, 1)
    r = oracle.run_chunk(net, fr, [0.0, e["theta"]], want_deltas=True)
    assert r["deltas"][0][0, 0, 0, 0] == e["expect_value"]


@pytest.mark.parametrize("seed", range(10))
def test_pin8_nonlinear_bruteforce(oracle_lib, seed):
    """At theta = 0 every non-linear delta equals f(x_t) - f(x_{t-1}) (fp64)."""
    for mk in (lambda n: n.relu(-1), lambda n: n.silu(-1), lambda n: n.maxpool(-1, 3, 2, 1),
               lambda n: n.se(-1, 2)):
        net = _single(mk, 3, 7, 6, seed)
        fr = random_frames(seed, 5, 7, 6, 3, p_change=0.3)
        r = oracle.run_chunk(net, fr, 0.0, want_deltas=True)
        for t in range(1, 5):
            a = dense_forward64(net, fr[t])[0]
            b = dense_forward64(net, fr[t - 1])[0]
            assert close(r["deltas"][0][t - 1], a - b, rel=1e-4, abs_=2e-6), (seed, t)


# --------------------------------------------------------- PIN9 drift
def test_pin9_drift(oracle_lib):
    e = _gold("spec_examples.json")["drift"]
    net = _single(lambda n: n.relu(-1), 1, 1, 1)
    fr = (np.arange(e["frames"], dtype=np.float32) * np.float32(e["per_frame"])).reshape(-1, 1, 1, 1)
    r = oracle.run_chunk(net, fr, [e["theta"], 0.0], want_deltas=True)
    emit_frames = [t + 1 for t in range(e["frames"] - 1) if r["counts"][0][t]]
    assert emit_frames == e["expect_emit_frames"]
    # input delta at frame 3 flows through relu of a positive ramp unchanged
    assert abs(r["deltas"][0][2, 0, 0, 0] - e["expect_value_frame3"]) <= e["value_tol"]


# ----------------------------------------------------- PIN10 dilation
def test_pin10_dilation_vs_indicator_conv(oracle_lib):
    """Dilation == (indicator map conv ones-kernel) > 0 on 200 random
    geometries, and monotone."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        H, Wd = int(rng.integers(1, 20)), int(rng.integers(1, 20))
        kh, kw = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        sh, sw = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        ph, pw = int(rng.integers(0, kh // 2 + 1)), int(rng.integers(0, kw // 2 + 1))
        Ho, Wo = (H + 2 * ph - kh) // sh + 1, (Wd + 2 * pw - kw) // sw + 1
        if Ho < 1 or Wo < 1:
            continue
        m = (rng.random((H, Wd)) < rng.uniform(0, 0.3)).astype(np.uint8)
        got = oracle.dilate(m, (kh, kw), (sh, sw), (ph, pw), (Ho, Wo))
        ind = F.conv2d(torch.from_numpy(m.astype(np.float64))[None, None], torch.ones(1, 1, kh, kw, dtype=torch.float64),
                       stride=(sh, sw), padding=(ph, pw))[0, 0].numpy() > 0
        assert np.array_equal(got.astype(bool), ind)
        m2 = m | (rng.random((H, Wd)) < 0.1).astype(np.uint8)
        got2 = oracle.dilate(m2, (kh, kw), (sh, sw), (ph, pw), (Ho, Wo))
        assert np.all(got2 >= got)


# -------------------------------------------- PIN12 schedule equivalence
@pytest.mark.parametrize("seed", range(12))
def test_pin12_frame_outer_equals_layer_outer(oracle_lib, seed):
    """SparseBatch ('N' order) == vanilla frame order, bit-exact."""
    net = random_net(700 + seed)
    fr = random_frames(seed, 7, net.in_h, net.in_w, net.in_c)
    a = oracle.run_chunk(net, fr, 0.06, layer_outer=False, want_deltas=True)
    b = oracle.run_chunk(net, fr, 0.06, layer_outer=True, want_deltas=True)
    for i in a["masks"]:
        assert np.array_equal(a["masks"][i], b["masks"][i])
        assert np.array_equal(a["deltas"][i], b["deltas"][i])
    for i in a["taps"]:
        assert np.array_equal(a["taps"][i], b["taps"][i])
    assert np.array_equal(a["counts"], b["counts"])


# ------------------------------------------------ PIN13 memory accountant
def test_pin13_memory_separation(oracle_lib):
    """SparseBatch persistent is independent of the number of non-linear
    layers; vanilla grows with it (P:139 vs P:152)."""
    rows = []
    for nl in (1, 4, 16, 32):
        n = Net(64, 56, 56)
        x = -1
        for _ in range(nl):
            x = n.relu(n.conv(x, 64, 3))
        n.output(x)
        sb = oracle.account_memory(n, "sparsebatch")
        va = oracle.account_memory(n, "vanilla", L=4)
        rows.append((nl, sb["persistent_values"], va["persistent_values"]))
        assert sb["persistent_values"] == 2 * 64 * 56 * 56
        assert sb["pass_count"] == 1 and va["pass_count"] == 4
    assert len({r[1] for r in rows}) == 1
    inc = [rows[i + 1][2] - rows[i][2] for i in range(3)]
    per = [(rows[i + 1][0] - rows[i][0]) for i in range(3)]
    assert all(d % p == 0 and d // p == inc[0] // per[0] for d, p in zip(inc, per))  # affine in N
    n16 = [r for r in rows if r[0] == 16][0]
    assert n16[2] >= 10 * n16[1]


def test_pin13b_memory_rows_worked_example(oracle_lib):
    """The accountant's SparseBatch transient = the live set of (dense x0 +
    delta rows) tensors per layer step ("N" order).  Hand-worked on
    a 2-ch 6x7 input (N = 42), conv3x3 2->3, ReLU, conv1x1 3->4, tap, L = 5:
      input rows 4*42*2 = 336        live steps 0-1
      conv0  126 + 4*42*3 = 630      live 1-2
      relu   126 + 504    = 630      live 2-3
      conv1  168 + 4*42*4 = 840      live 3-4 (the tap)
    peak = step 3: 630 + 840 = 1470; persistent = 84 + 5*168 = 924.
    Vanilla: persistent 84 + 168 + (126 + 126) = 504, one frame's tensors
    peak at step 3: 252 + 336 = 588."""
    n = Net(2, 6, 7)
    x = n.relu(n.conv(-1, 3, 3))
    n.output(n.conv(x, 4, 1, 1, 0))
    sb = oracle.account_memory(n, "sparsebatch", L=5)
    va = oracle.account_memory(n, "vanilla", L=5)
    assert (sb["persistent_values"], sb["peak_transient_values"]) == (924, 1470)
    assert (va["persistent_values"], va["peak_transient_values"]) == (504, 588)
    # measured rows replace the all-active bound: 10 active input pixel-frames,
    # 30 conv0 rows, 12 emitted ReLU rows, 12 conv1 rows
    r = {-1: 10, 0: 30, 1: 12, 2: 12}
    sbr = oracle.account_memory(n, "sparsebatch", L=5, rows=r)
    # steps: 1: 20 + (126 + 90) = 236; 2: 216 + (126 + 36) = 378; 3: 162 + (168 + 48) = 378
    assert sbr["peak_transient_values"] == 378


def test_pin13c_memory_rows_from_oracle_run(oracle_lib):
    """rows_from_run counts the oracle's masks; identical frames give no
    rows (PIN3), so the transient falls to the dense reference activations,
    and more active rows never lower the peak."""
    n = Net(2, 9, 9)
    x = n.relu(n.conv(-1, 4, 3))
    n.output(n.conv(x, 4, 3))
    init_weights(n, 3)
    still = np.repeat(random_frames(1, 1, 9, 9, 2), 5, axis=0)
    r0 = oracle.rows_from_run(oracle.run_chunk(n, still, 0.0), n)
    assert all(v == 0 for v in r0.values())
    dense_only = oracle.account_memory(n, "sparsebatch", L=5, rows=r0)["peak_transient_values"]
    assert dense_only == 2 * 9 * 9 * 4   # conv0 x0 + relu y0 (step 2), or relu + conv1 (step 3)
    moving = random_frames(2, 5, 9, 9, 2, p_change=0.3)
    rm = oracle.rows_from_run(oracle.run_chunk(n, moving, 0.0), n)
    assert rm[-1] > 0 and rm[0] >= rm[-1]   # dilation: a 3x3 conv never has fewer rows
    assert oracle.account_memory(n, "sparsebatch", L=5, rows=rm)["peak_transient_values"] > dense_only
    assert oracle.account_memory(n, "sparsebatch", L=5)["peak_transient_values"] >= \
        oracle.account_memory(n, "sparsebatch", L=5, rows=rm)["peak_transient_values"]


# -------------------------------------------------------- PIN16 SE exact
def test_pin16_se_zero_threshold(oracle_lib):
    net = _single(lambda n: n.se(-1, 3), 6, 5, 5, 2)
    fr = random_frames(4, 6, 5, 5, 6, p_change=0.4)
    r = oracle.run_chunk(net, fr, 0.0)
    for t in range(6):
        assert close(r["taps"][1][t], dense_forward64(net, fr[t])[0], rel=1e-5, abs_=1e-6)


# ------------------------------------------------ BF16-mode conv contract
def _rb(a):
    """bf16 round-to-nearest-even of fp32 values (torch's cast: a library routine)."""
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).to(torch.float64)


@pytest.mark.parametrize("cin,cout,k,s,groups", [
    (64, 16, 3, 1, 1), (128, 32, 3, 2, 1), (24, 40, 1, 1, 1), (12, 16, 3, 1, 1), (16, 12, 3, 1, 1),
    (3, 32, 3, 2, 1), (3, 64, 7, 2, 1), (1, 64, 3, 1, 1), (6, 5, 2, 1, 1),
    (32, 32, 3, 1, 32), (40, 40, 5, 2, 40), (8, 8, 7, 1, 8)])
def test_bf16_mode_conv_matches_rounded_fp64(oracle_lib, cin, cout, k, s, groups):
    """BF16 mode (R22-BF16) is one contract for EVERY convolution -- any
    channel count, kernel size, stride or groups (stems, depthwise, 1x1):
    the dense conv equals the fp64 convolution of bf16-rounded weights and
    inputs (torch bfloat16 casts, F.conv2d); it differs from FP32 mode."""
    n = Net(cin, 11, 9)
    c = n.conv(-1, cout, k, s, k // 2, groups=groups)
    n.output(c)
    init_weights(n, cin + k)
    x = np.random.default_rng(cin).standard_normal((11, 9, cin)).astype(np.float32)
    got = oracle.dense_forward(n, x, precision="bf16")[c]
    xw = _rb(x).permute(2, 0, 1).unsqueeze(0)
    ref = F.conv2d(xw, _rb(n.layers[c]["w"]), torch.from_numpy(n.layers[c]["b"].astype(np.float64)),
                   stride=s, padding=k // 2, groups=groups)[0].permute(1, 2, 0).numpy()
    assert close(got, ref, rel=1e-4, abs_=1e-5), max_err(got, ref)
    assert not np.array_equal(got, oracle.dense_forward(n, x)[c])


@pytest.mark.parametrize("seed", range(8))
def test_bf16_mode_stored_deltas_are_bf16(oracle_lib, seed):
    """R22-BF16: every stored delta (Subtraction, conv, add, every site) is a
    bf16 value: its fp32 bit pattern has zero low 16 bits."""
    net = random_net(900 + seed)
    fr = random_frames(seed, 6, net.in_h, net.in_w, net.in_c)
    r = oracle.run_chunk(net, fr, 0.03, want_deltas=True, precision="bf16")
    for i, d in list(r["deltas"].items()) + [(-1, r["in_delta"])]:
        assert np.all((d.view(np.uint32) & 0xFFFF) == 0), (seed, i)
    assert np.any(r["in_delta"] != 0)


@pytest.mark.parametrize("seed", range(6))
def test_bf16_mode_subtraction_rounding(oracle_lib, seed):
    """BF16 Subtraction: the decision is taken on the fp32 raw difference
    (R1/R2), the emitted delta is RNE-bf16(raw) (torch cast) and S
    advances by the emitted value (R3), so S_t = X_0 + sum of emitted."""
    net = _single(lambda n: n.relu(-1), 3, 7, 8, seed)
    fr = random_frames(seed, 8, 7, 8, 3, p_change=0.5, scale=0.05)
    th = 0.02
    r = oracle.run_chunk(net, fr, [th, 0.0], want_deltas=True, precision="bf16")
    S = fr[0].copy()
    for t in range(1, 8):
        raw = (fr[t] - S).astype(np.float32)
        act = np.abs(raw).max(axis=2) > np.float32(th)
        assert np.array_equal(r["in_mask"][t - 1].astype(bool), act)
        e = np.where(act[..., None], _rb(raw).numpy(), 0.0).astype(np.float32)
        assert np.array_equal(r["in_delta"][t - 1], e)
        S = (S + e).astype(np.float32)


@pytest.mark.parametrize("seed", range(6))
def test_bf16_mode_site_rounding(oracle_lib, seed):
    """BF16 ReLU site: c = relu(x_acc) - y_acc on the touched pixels, emit iff
    max_c |c| > theta on the fp32 value, the stored delta is RNE-bf16(c) and
    y_acc advances by it -- rebuilt from the oracle's own outputs (x_acc =
    x0 + sum conv deltas, y_acc = y0 + sum emitted, fp32 adds) and torch's
    bf16 cast."""
    net = Net(2, 8, 8)
    c = net.conv(-1, 8, 3)
    a = net.relu(c)
    net.output(a)
    init_weights(net, seed)
    fr = random_frames(seed, 7, 8, 8, 2, p_change=0.5, scale=0.3)
    th = 0.05
    r = oracle.run_chunk(net, fr, [0.0, th], want_deltas=True, want_dense0=True, precision="bf16")
    xa, ya = r["dense0"][c].copy(), r["dense0"][a].copy()
    n_emit = 0
    for t in range(6):
        tm = r["masks"][c][t].astype(bool)
        xa = (xa + r["deltas"][c][t]).astype(np.float32)
        cand = (np.maximum(xa, 0) - ya).astype(np.float32)
        keep = tm & (np.abs(cand).max(axis=2) > np.float32(th))
        assert np.array_equal(r["masks"][a][t].astype(bool), keep), (seed, t)
        e = np.where(keep[..., None], _rb(cand).numpy(), 0.0).astype(np.float32)
        assert np.array_equal(r["deltas"][a][t], e), (seed, t)
        ya = (ya + e).astype(np.float32)
        n_emit += int(keep.sum())
    assert n_emit > 0


# ------------------------------------------------- SE site at theta > 0 (R8)
def test_se_refresh_worked_example(oracle_lib):
    """Hand-worked 1-pixel / 2-channel SE example (tests/golden/se_refresh.json,
    reading R8): gate refresh on frame 2 only; the candidate uses the EMITTED
    gate s_emit, not the current s_t (frames 1, 5 and 6 tell them apart)."""
    g = _gold("se_refresh.json")
    n = Net(2, 1, 1)
    x = n.se(-1, 1)
    n.output(x)
    n.layers[x]["w"] = np.array(g["w1"], np.float32)
    n.layers[x]["b"] = np.array(g["b1"], np.float32)
    n.layers[x]["w2"] = np.array(g["w2"], np.float32)
    n.layers[x]["b2"] = np.array(g["b2"], np.float32)
    fr = np.array(g["frames"], np.float32).reshape(-1, 1, 1, 2)
    r = oracle.run_chunk(n, fr, [g["theta_input"], g["theta_se"]], want_deltas=True)
    assert list(r["counts"][1]) == g["expect_emitted"]
    np.testing.assert_allclose(r["deltas"][x].reshape(-1, 2), np.array(g["expect_delta"]), atol=g["tol"], rtol=0)
    np.testing.assert_allclose(r["taps"][1].reshape(-1, 2), np.array(g["expect_output"]), atol=g["tol"], rtol=0)


@pytest.mark.parametrize("seed", range(6))
def test_se_drift_bound_r21(oracle_lib, seed):
    """R21 drift bound at theta > 0: with x_acc = x0 + sum of the SE input's
    deltas, y_acc = y0 + sum of the SE's emitted deltas and s_t = gate(x_acc)
    (torch fp64), every pixel and channel obeys |x_acc*s_t - y_acc| <= theta +
    |x_acc|*theta_gate after every frame (theta_gate = theta_site): the
    residual of the last touch is <= theta and the gate moved by <= theta_gate
    since the last refresh."""
    net = Net(3, 6, 7)
    c = net.conv(-1, 6, 3)
    x = net.se(c, 2)
    net.output(x)
    init_weights(net, 40 + seed)
    L, th = 9, 0.04
    fr = random_frames(seed, L, 6, 7, 3, p_change=0.35, scale=0.25)
    r = oracle.run_chunk(net, fr, [0.01, th], want_deltas=True, want_dense0=True)
    xa = r["dense0"][c].astype(np.float64)
    ya = r["dense0"][x].astype(np.float64)
    l = net.layers[x]
    w1, b1, w2, b2 = (torch.from_numpy(l[k].astype(np.float64)) for k in ("w", "b", "w2", "b2"))
    for t in range(L - 1):
        xa = xa + r["deltas"][c][t]
        ya = ya + r["deltas"][x][t]
        m = torch.from_numpy(xa).mean(dim=(0, 1))
        h = w1 @ m + b1
        s_t = torch.sigmoid(w2 @ (h * torch.sigmoid(h)) + b2).numpy()
        bound = th + np.abs(xa) * th + 1e-5
        assert np.all(np.abs(xa * s_t - ya) <= bound), (seed, t)
    assert r["counts"][1].sum() > 0


# ------------------------------------------------ O12 band-follow mode
def _follow_net(seed):
    net = Net(2, 8, 9)
    c = net.conv(-1, 6, 3)
    a = net.silu(c)
    c2 = net.conv(a, 4, 3)
    m = net.maxpool(net.relu(c2), 2, 2)
    net.output(m)
    init_weights(net, seed)
    return net, [a, m - 1, m]


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_follow_own_masks_is_identity(oracle_lib, precision):
    """Following the oracle's own decisions changes nothing: bit-identical
    outputs, zero adoptions, zero violations."""
    net, sites = _follow_net(3)
    fr = random_frames(3, 7, 8, 9, 2, p_change=0.4, scale=0.3)
    a = oracle.run_chunk(net, fr, 0.05, want_deltas=True, precision=precision)
    b = oracle.run_chunk(net, fr, 0.05, want_deltas=True, precision=precision,
                         follow={i: a["masks"][i] for i in sites})
    for i in a["masks"]:
        assert np.array_equal(a["masks"][i], b["masks"][i]) and np.array_equal(a["deltas"][i], b["deltas"][i])
    fs = b["follow_stats"]
    assert fs[:, 2].sum() == 0 and fs[:, 3].sum() == 0 and fs[sites, 0].sum() > 0


def test_follow_adopts_only_inside_band(oracle_lib):
    """A flipped decision far from theta is a violation and is NOT adopted; a
    flipped decision inside the band (tau widened to cover it) is adopted,
    and the run continues from the GPU's decision (reading R23)."""
    net, sites = _follow_net(5)
    fr = random_frames(5, 6, 8, 9, 2, p_change=0.4, scale=0.3)
    th = 0.05
    a = oracle.run_chunk(net, fr, th, want_deltas=True, precision="fp32")
    site = sites[0]
    m = a["masks"][site].copy()
    t, y, x = map(int, np.argwhere(m == 1)[0])
    m[t, y, x] = 0                                   # the "GPU" truncated an emitted pixel
    # tight band: the flip is outside it -> violation, own decision kept
    b = oracle.run_chunk(net, fr, th, want_deltas=True, follow={site: m}, tau=(1e-4, 0.0, 1e-5))
    assert b["follow_stats"][site, 3] >= 1 and b["follow_stats"][site, 2] == 0
    assert np.array_equal(b["masks"][site], a["masks"][site])
    # band wide enough to contain that pixel's value -> adopted
    c = oracle.run_chunk(net, fr, th, want_deltas=True, follow={site: m}, tau=(0.0, 0.0, 10.0))
    assert c["follow_stats"][site, 2] == 1 and c["follow_stats"][site, 3] == 0
    assert c["masks"][site][t, y, x] == 0 and np.all(c["deltas"][site][t, y, x] == 0)
    assert c["counts"][sites.index(site) + 1][t] == a["counts"][sites.index(site) + 1][t] - 1
