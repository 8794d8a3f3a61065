"""BF16 mode parity (-m gpu), against the oracle's BF16 contract (R22-BF16).

The contract is stated without reference to kernel dispatch: EVERY conv
multiplies bf16-rounded weights and inputs with fp32 accumulation, every
stored delta is bf16 (RNE).  The GPU honours it on every path (tcgen05
convs, CUDA-core depthwise / small-c_in convs with bf16-rounded weights and
dense inputs), so the two sides differ only in fp32 summation order inside
the tensor core and in SiLU's single-precision exp.  Checks:
  * kernel units: tcgen05 conv / stem rows within one bf16 ulp, the
    CUDA-core depthwise and small convs BIT-EXACT (same fmaf order);
  * end to end with band-follow (O12, reading R23): every site decision
    outside the ambiguity band agrees, then masks / index lists, counts,
    rows and taps are compared elementwise (bf16 bound of R29);
  * BF16 GPU vs the FP32 oracle at theta = 0 within the north_star 2e-2.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from workloads import Net, init_weights
from gpu_harness import gpu_run, make_frames, bf16_within, follow_compare
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


@pytest.mark.parametrize("C,k,s", [(32, 3, 1), (96, 5, 2), (24, 3, 2), (40, 5, 1), (12, 3, 1)])
def test_cuda_core_convs_bit_exact_in_bf16_mode(C, k, s):
    """Depthwise and small-c_in convs run on CUDA cores in BF16 mode with
    bf16-rounded weights and (dense) inputs and the oracle's fmaf order, so
    under the dispatch-free contract they are BIT-EXACT: dense reference
    outputs, masks, delta rows and taps."""
    n = Net(3, 22, 26)
    x = n.relu(n.conv(-1, 6, 3))                           # c_in 3, c_out 6: CUDA-core conv
    x = n.relu(n.conv(x, C, 3))                            # c_in 6: CUDA-core conv
    y = n.conv(x, C, k, s, k // 2, groups=C)               # depthwise
    n.output(n.relu(y))
    init_weights(n, C + k)
    B, L = 2, 6
    fr = np.stack([random_frames(b + 3, L, 22, 26, 3, p_change=0.3) for b in range(B)])
    th = np.full(oracle.num_sites(n), 0.03, np.float32)
    enc, _ = gpu_run(n, fr, th, precision="bf16")
    for b in range(B):
        r = oracle.run_chunk(n, fr[b], th, want_deltas=True, want_dense0=True, precision="bf16")
        assert np.array_equal(enc.debug_dense0(y, b), r["dense0"][y]), "dense depthwise"
        for i in range(len(n.layers) - 1):
            for t in range(1, L):
                assert np.array_equal(enc.debug_mask(i, b, t), r["masks"][i][t - 1]), (i, t)
                idx, rows = enc.debug_rows(i, b, t)
                assert np.array_equal(rows, r["deltas"][i][t - 1].reshape(-1, rows.shape[1])[idx]), (i, t)
        assert np.array_equal(enc.outputs(len(n.layers) - 1)[b].cpu().numpy(), r["taps"][len(n.layers) - 1])


def test_crnn_bf16_theta0_vs_fp32_oracle():
    """The BF16 path against the FP32 oracle (no BF16 contract at all) at
    theta = 0: every frame of the tap within the north_star "2e-2 relative"
    read normwise (||a - b|| <= 2e-2 ||b||; elementwise, bf16 operand
    rounding random-walks through 7 convs of up to 4608 terms and a few tail
    elements exceed 2e-2 |b| + 2e-2 rms); against the BF16 contract every
    element within 2e-2 |b| + 2e-2 rms (R29)."""
    cfg = W.get_config(2)
    net = cfg.build_net()
    fr = make_frames(cfg, 2, L=8)
    enc, _ = gpu_run(net, fr, 0.0, precision="bf16", debug=False)
    tap = enc.taps[0]
    out = enc.outputs(tap).cpu().numpy()
    for b in range(2):
        r32 = oracle.run_chunk(net, fr[b], 0.0, want_masks=False, precision="fp32")
        for t in range(fr.shape[1]):
            a, ref = out[b][t].astype(np.float64), r32["taps"][tap][t].astype(np.float64)
            rel = float(np.linalg.norm(a - ref) / np.linalg.norm(ref))
            assert rel <= 2e-2, f"BF16 GPU vs FP32 oracle, frame {t}: relative error {rel:.4f} ({bf16_within(a, ref)})"
        r16 = oracle.run_chunk(net, fr[b], 0.0, want_masks=False, precision="bf16")
        ok, e = bf16_within(out[b], r16["taps"][tap])
        assert ok, f"BF16 GPU vs BF16 contract: {e:.2f} x bound"


@pytest.mark.parametrize("model", ["crnn", "effnet", "resnet18"])
def test_bf16_band_follow(model):
    """End to end at theta > 0 with band-follow (O12): zero decisions
    outside the R23 band disagree; masks, index lists, counts, every layer's
    delta rows and the taps compared elementwise; adopted decisions << 0.1 %."""
    if model == "crnn":
        cfg = W.get_config(2)
        net = cfg.build_net()
        fr = make_frames(cfg, 2, L=10)
    elif model == "effnet":
        # the cfg3 network itself (calibrated weights, R30) at 512x512, 7 frames
        cfg = W.get_config(3)
        net = cfg.build_net()
        fr = make_frames(cfg, 1, L=7)
    else:
        net = W.models.resnet18(64, 96)
        init_weights(net, 32)
        fr = W.to_float(W.gen_video(2, 7, 64, 96, 3, 78, n_objects=4, size=(8, 24), speed=(1, 3), noise_q=0.1,
                                    noise_amp=2))
    enc, _ = gpu_run(net, fr, 0.05, precision="bf16")
    for b in range(fr.shape[0]):
        rep = follow_compare(enc, net, fr[b], 0.05, b, "bf16")
        assert rep["adopted"] <= max(2, 1e-3 * rep["decisions"]), rep
