"""BF16 mode (tcgen05 tensor-core convolution) parity (-m gpu).

Contract (R22-BF16): convolutions with c_in, c_out % 8 == 0 multiply
bf16-rounded operands with fp32 accumulation; the oracle's BF16 mode applies
the same rounding with its sequential fmaf chain, so the two differ only in
the fp32 summation order inside the tensor core.  Checks:
  * kernel unit: a tensor-core conv's rows (sparse, every frame) and its dense
    reference output agree with the oracle to summation-order rounding
    (|a-b| <= 1e-4 * (|b| + rms)), masks exact (dilation is integer work);
  * end to end at theta = 0 (no threshold decision can flip by more than a
    rounding-sized value): tap outputs within the north_star bf16 bound
    2e-2 |b| + 2e-2 rms, masks exact except pixels whose value is ~0;
  * end to end at theta > 0: masks agree on >= 99.9% of pixel-frames per
    layer, tap outputs within 2e-2 |b| + 2e-2 rms (reading R23/R29).
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from workloads import Net, init_weights
from gpu_harness import gpu_run, make_frames
from netgen import random_frames

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _rel_ok(a, b, rel, rms_frac):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    rms = float(np.sqrt(np.mean(b * b))) if b.size else 0.0
    err = np.abs(a - b)
    return bool(np.all(err <= rel * np.abs(b) + rms_frac * rms + 1e-6)), float(err.max() if err.size else 0)


def _tc_net(cin, cout, k, s=1, h=20, w=28, seed=0):
    # upstream convs stay on the exact CUDA-core path (c_out = 12 and c_in = 12
    # are not tensor-core shapes), so the conv under test receives
    # bit-identical input deltas on both sides
    n = Net(3, h, w)
    x = n.relu(n.conv(-1, 12, 3))
    x = n.relu(n.conv(x, cin, 3))
    y = n.conv(x, cout, k, s, k // 2)
    n.output(y)
    init_weights(n, seed)
    return n, y


@pytest.mark.parametrize("cin,cout,k,s", [(64, 64, 3, 1), (64, 128, 3, 1), (128, 256, 3, 2), (64, 512, 1, 1),
                                          (192, 96, 3, 1), (64, 32, 3, 1),
                                          # channel-padded k-blocks (c_in % 64 != 0), ragged c_out tiles
                                          (16, 96, 1, 1), (24, 40, 1, 1), (40, 24, 3, 1), (144, 24, 1, 1),
                                          (8, 16, 3, 2), (112, 672, 1, 1)])
def test_tc_conv_kernel_unit(cin, cout, k, s):
    net, conv = _tc_net(cin, cout, k, s, seed=cin + cout)
    B, L = 3, 6
    fr = np.stack([random_frames(b + 1, L, net.in_h, net.in_w, 3, p_change=0.3) for b in range(B)])
    th = np.zeros(oracle.num_sites(net), np.float32)
    th[0] = 0.02
    enc, _ = gpu_run(net, fr, th, precision="bf16")
    for b in range(B):
        r = oracle.run_chunk(net, fr[b], th, want_deltas=True, want_dense0=True, precision="bf16")
        d0 = enc.debug_dense0(conv, b)
        ok, e = _rel_ok(d0, r["dense0"][conv], 1e-4, 1e-4)
        assert ok, f"dense tc conv err {e}"
        for t in range(1, L):
            m = enc.debug_mask(conv, b, t)
            assert np.array_equal(m, r["masks"][conv][t - 1])
            idx, rows = enc.debug_rows(conv, b, t)
            exp = r["deltas"][conv][t - 1].reshape(-1, cout)[idx]
            # both sides store bf16(fp32 accumulator); the accumulators differ
            # only in summation order, so the stored values differ by at most
            # one bf16 ulp (<= 2^-7 relative) where a rounding boundary is crossed
            ok, e = _rel_ok(rows, exp, 2.0 ** -7, 1e-4)
            assert ok, f"sparse tc conv rows err {e} (chunk {b} frame {t})"


@pytest.mark.parametrize("cin,cout,k,s", [(3, 64, 7, 2), (1, 64, 3, 1), (3, 32, 3, 2), (3, 48, 5, 1)])
def test_tc_stem_kernel_unit(cin, cout, k, s):
    """Tensor-core stem (network input, c_in <= 4): sparse rows from the
    4-channel-padded dense input delta, dense reference from the fp32 frames."""
    n = Net(cin, 30, 38)
    conv = n.conv(-1, cout, k, s, k // 2)
    n.output(conv)
    init_weights(n, cin * 7 + k)
    B, L = 2, 6
    fr = np.stack([random_frames(b + 11, L, 30, 38, cin, p_change=0.3) for b in range(B)])
    th = np.array([0.02], np.float32)
    enc, _ = gpu_run(n, fr, th, precision="bf16")
    for b in range(B):
        r = oracle.run_chunk(n, fr[b], th, want_deltas=True, want_dense0=True, precision="bf16")
        ok, e = _rel_ok(enc.debug_dense0(conv, b), r["dense0"][conv], 1e-4, 1e-4)
        assert ok, f"dense stem err {e}"
        for t in range(1, L):
            assert np.array_equal(enc.debug_mask(conv, b, t), r["masks"][conv][t - 1])
            idx, rows = enc.debug_rows(conv, b, t)
            ok, e = _rel_ok(rows, r["deltas"][conv][t - 1].reshape(-1, cout)[idx], 2.0 ** -7, 1e-4)
            assert ok, f"sparse stem rows err {e} (chunk {b} frame {t})"


def test_crnn_bf16_theta0():
    cfg = W.get_config(2)
    net = cfg.build_net()
    fr = make_frames(cfg, 2, L=8)
    enc, _ = gpu_run(net, fr, 0.0, precision="bf16", debug=False)
    tap = enc.taps[0]
    out = enc.outputs(tap).cpu().numpy()
    for b in range(2):
        r = oracle.run_chunk(net, fr[b], 0.0, want_masks=False, precision="bf16")
        # summation-order differences are amplified by later bf16 roundings of
        # the deltas (one bf16 ulp = 2^-8 relative), so the bound is the
        # north_star bf16 one, not fp32's
        ok, e = _rel_ok(out[b], r["taps"][tap], 2e-2, 2e-2)
        assert ok, e


def test_crnn_bf16_threshold():
    cfg = W.get_config(2)
    net = cfg.build_net()
    fr = make_frames(cfg, 2, L=10)
    enc, _ = gpu_run(net, fr, cfg.theta_fixed, precision="bf16")
    tap = enc.taps[0]
    for b in range(2):
        r = oracle.run_chunk(net, fr[b], cfg.theta_fixed, precision="bf16")
        for i in range(len(net.layers)):
            agree, total = 0, 0
            for t in range(1, 10):
                m = enc.debug_mask(i, b, t)
                agree += int((m == r["masks"][i][t - 1]).sum())
                total += m.size
            assert agree >= 0.999 * total, (i, agree, total)
        got = enc.outputs(tap)[b].cpu().numpy()
        ok, e = _rel_ok(got, r["taps"][tap], 2e-2, 2e-2)
        assert ok, e
