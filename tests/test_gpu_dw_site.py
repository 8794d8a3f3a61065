"""Depthwise conv + pointwise site in one pass (SURVEY §8(f) N2 for depthwise
convs; Eq.2 then Eq.3), -m gpu.

The fused kernel computes an output pixel's depthwise delta rows frame by
frame and steps the ReLU / SiLU site on them at once, so the conv's delta
rows never reach HBM.  It must give bit-identical results to the separate
conv and site kernels (ST_NO_FUSE_DW=1) in both modes, and in FP32 mode
match the oracle (masks exact; ReLU values exact, SiLU within R29) -- also
with debug_retain, where the fused pass writes the conv's own rows too."""
from __future__ import annotations

import numpy as np
import pytest

import workloads as W
from workloads import Net, init_weights
from gpu_harness import gpu_run, compare_chunk

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2410_20790_b200 import load_library
    load_library()


def dw_net(C, k, s, act, h, w, seed):
    """stem 3x3 3->C + act, depthwise kxk/s + act, 1x1 C->8 (+ an SE-free tail)."""
    n = Net(3, h, w, f"dw{C}k{k}s{s}{act}")
    x = n.conv(-1, C, 3, 1, 1)
    x = n.relu(x) if act == "relu" else n.silu(x)
    x = n.conv(x, C, k, s, k // 2, groups=C)
    x = n.relu(x) if act == "relu" else n.silu(x)
    x = n.conv(x, 8, 1, 1, 0)
    n.output(x)
    init_weights(n, seed)
    return n


CASES = [(8, 3, 1, "relu", 19, 23), (24, 3, 2, "silu", 21, 26), (64, 5, 1, "relu", 14, 17),
         (136, 3, 1, "silu", 12, 13), (264, 5, 2, "relu", 11, 14), (520, 3, 1, "silu", 9, 10),
         (672, 5, 1, "silu", 9, 11), (1152, 5, 1, "relu", 6, 7), (32, 3, 1, "silu", 18, 21),
         (16, 3, 2, "relu", 20, 37), (240, 5, 1, "silu", 10, 12)]


def frames_for(h, w, seed, B=2, L=9):
    return W.to_float(W.gen_video(B, L, h, w, 3, seed, n_objects=3, size=(3, 7), speed=(1, 2),
                                  noise_q=0.08, noise_amp=2))


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("C,k,s,act,h,w", CASES)
def test_fused_dw_site_matches_separate(C, k, s, act, h, w, precision, monkeypatch):
    import torch
    from paper_2410_20790_b200 import Encoder
    net = dw_net(C, k, s, act, h, w, 5 + C)
    fr = torch.from_numpy(frames_for(h, w, 900 + C)).cuda()
    outs = {}
    for mode in ("fused", "separate"):
        if mode == "separate":
            monkeypatch.setenv("ST_NO_FUSE_DW", "1")
        enc = Encoder(net, fr.shape[0], fr.shape[1], precision=precision)
        res = []
        for th in (0.02, 0.0, 0.08):
            enc.encode_reference(fr[:, 0])
            enc.encode_diff(fr[:, 1:], th)
            torch.cuda.synchronize()
            res.append(([enc.outputs(t).cpu().numpy().copy() for t in enc.taps], enc.get_sparsity()[0].copy()))
        outs[mode] = res
        enc.close()
    for (og, cg), (oe, ce) in zip(outs["fused"], outs["separate"]):
        assert np.array_equal(cg, ce), "per-site per-frame counts"
        for a, b in zip(og, oe):
            assert np.array_equal(a, b), f"tap outputs differ (max {np.abs(a - b).max():.3e})"


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("C,k,s,act,h,w", CASES)
def test_dw_site_forms_identical(C, k, s, act, h, w, precision, monkeypatch):
    """The tile form for C <= 32 (ST_DW_TILE=1: shared-memory staged
    footprint rows), the team forms (ST_DW_TEAM=2: every C): the channel-strided warp form
    for C <= 64 (ST_DW_STRIDED=1), the 8-channel sequential-pipeline team
    kernel (ST_DWT_TB=0), the frame-pair kernel (ST_DWT_TB=2/4), and the
    narrow / warp / wide forms (ST_DW_TEAM=0) give the same bits: the
    per-channel operations are the same, only the work split differs."""
    import torch
    from paper_2410_20790_b200 import Encoder
    net = dw_net(C, k, s, act, h, w, 7 + C)
    fr = torch.from_numpy(frames_for(h, w, 300 + C)).cuda()
    outs = []
    for env in ({"ST_DW_TEAM": "2", "ST_DWT_TB": "0", "ST_DW_STRIDED": "1", "ST_DW_TILE": "1"},
                {"ST_DW_TEAM": "2", "ST_DWT_TB": "0", "ST_DW_STRIDED": "1", "ST_DW_TILE": "0"},
                {"ST_DW_TEAM": "2", "ST_DWT_TB": "0", "ST_DW_STRIDED": "0", "ST_DW_TILE": "0"},
                {"ST_DW_TEAM": "2", "ST_DWT_TB": "2", "ST_DW_STRIDED": "1", "ST_DW_TILE": "0"},
                {"ST_DW_TEAM": "2", "ST_DWT_TB": "4", "ST_DW_STRIDED": "1", "ST_DW_TILE": "0"},
                {"ST_DW_TEAM": "0", "ST_DWT_TB": "0", "ST_DW_STRIDED": "1", "ST_DW_TILE": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        enc = Encoder(net, fr.shape[0], fr.shape[1], precision=precision)
        res = []
        for th in (0.03, 0.0):
            enc.encode_reference(fr[:, 0])
            enc.encode_diff(fr[:, 1:], th)
            torch.cuda.synchronize()
            res.append(([enc.outputs(t).cpu().numpy().copy() for t in enc.taps], enc.get_sparsity()[0].copy()))
        outs.append(res)
        enc.close()
    for other in outs[1:]:
        for (og, cg), (oe, ce) in zip(outs[0], other):
            assert np.array_equal(cg, ce), "per-site per-frame counts"
            for a, b in zip(og, oe):
                assert np.array_equal(a, b), f"tap outputs differ (max {np.abs(a - b).max():.3e})"


@pytest.mark.parametrize("C,k,s,act,h,w", CASES)
def test_fused_dw_site_vs_oracle_fp32(C, k, s, act, h, w):
    """debug_retain run (the fused pass also writes the conv's rows): every
    layer's mask / index list and rows against the oracle."""
    net = dw_net(C, k, s, act, h, w, 5 + C)
    fr = frames_for(h, w, 900 + C)
    th = [0.02] * (1 + sum(l["kind"] in W.NONLINEAR for l in net.layers))
    enc, _ = gpu_run(net, fr, th)
    for b in range(fr.shape[0]):
        compare_chunk(enc, net, fr[b], th, b, exact=(act == "relu"))
    enc.close()


# ---- 1x1/s1 convs in the input's row layout ("rowmap"): no dilation, scan or
# gather; the sites that feed them zero their touched-but-not-emitted slots
def _bottleneck_net(seed):
    """ResNet-style bottleneck and MBConv-style blocks: 1x1 convs reading a
    ReLU, an SE, an ADD and another 1x1 conv."""
    n = Net(3, 20, 28, "rowmap")
    x = n.relu(n.conv(-1, 32, 3, 1, 1))
    y = n.relu(n.conv(x, 16, 1, 1, 0))        # 1x1 on a ReLU (in place in the stem conv's layout)
    y = n.relu(n.conv(y, 16, 3, 1, 1))
    y = n.conv(y, 32, 1, 1, 0)                # 1x1 on a ReLU
    x = n.relu(n.add(y, x))
    z = n.conv(x, 24, 1, 1, 0)                # 1x1 on a ReLU of an ADD
    z = n.conv(z, 24, 1, 1, 0)                # 1x1 on a 1x1 conv
    z = n.silu(z)
    z = n.se(z, 6)
    z = n.conv(z, 32, 1, 1, 0)                # 1x1 on an SE (MBConv project)
    n.output(n.add(z, x))
    init_weights(n, seed)
    return n


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("model", ["bottleneck", "effnet"])
def test_rowmap_matches_gathered(model, precision, monkeypatch):
    import torch
    from paper_2410_20790_b200 import Encoder
    if model == "effnet":
        net = W.models.efficientnet_b0(64, 96)
        init_weights(net, 31)
        h, w = 64, 96
    else:
        net = _bottleneck_net(7)
        h, w = 20, 28
    fr = torch.from_numpy(frames_for(h, w, 77)).cuda()
    outs = {}
    for mode in ("rowmap", "gathered"):
        if mode == "gathered":
            monkeypatch.setenv("ST_NO_ROWMAP", "1")
        enc = Encoder(net, fr.shape[0], fr.shape[1], precision=precision)
        res = []
        for th in (0.03, 0.0):
            for _ in range(2):   # eager, then graph replay
                enc.encode_reference(fr[:, 0])
                enc.encode_diff(fr[:, 1:], th)
            torch.cuda.synchronize()
            res.append(([enc.outputs(t).cpu().numpy().copy() for t in enc.taps], enc.get_sparsity()[0].copy()))
        outs[mode] = res
        enc.close()
    for (og, cg), (oe, ce) in zip(outs["rowmap"], outs["gathered"]):
        assert np.array_equal(cg, ce), "per-site per-frame counts"
        for a, b in zip(og, oe):
            assert np.array_equal(a, b), f"tap outputs differ (max {np.abs(a - b).max():.3e})"


def test_rowmap_vs_oracle_fp32():
    net = _bottleneck_net(9)
    fr = frames_for(20, 28, 78)
    th = 0.03
    enc, _ = gpu_run(net, fr, th)
    for b in range(fr.shape[0]):
        compare_chunk(enc, net, fr[b], th, b, exact=False)
    enc.close()


# ---- tcgen05 conv + ReLU / SiLU site in the conv's epilogue (N2; BF16 mode)
def _tc_site_net(cout, act, k, seed):
    n = Net(3, 26, 34, f"tcsite{cout}{act}{k}")
    x = n.relu(n.conv(-1, 32, 3, 1, 1))
    y = n.conv(x, cout, k, 1, k // 2)                  # tcgen05 conv, c_out <= 256
    y = n.relu(y) if act == "relu" else n.silu(y)      # its only consumer: site in the epilogue
    y = n.conv(y, 32, 3, 1, 1)
    x = n.relu(n.add(y, x))
    z = n.conv(x, cout, 1, 1, 0)                       # 1x1 on an ADD layout (rowmap) + site
    z = n.relu(z) if act == "relu" else n.silu(z)
    n.output(n.conv(z, 16, 1, 1, 0))
    init_weights(n, seed)
    return n


@pytest.mark.parametrize("cout,act,k", [(32, "relu", 3), (96, "silu", 3), (136, "relu", 1), (256, "silu", 3)])
def test_tc_site_epilogue_matches_separate(cout, act, k, monkeypatch):
    """The epilogue site (opt-in, ST_FUSE_TC=1) is bit-identical to the
    separate conv + site kernels: pixels continuing across 128-row tiles (the
    fix-up kernel) included -- 2 chunks x 12 frames of 26x34 give hundreds of
    tiles per conv."""
    import torch
    from paper_2410_20790_b200 import Encoder
    net = _tc_site_net(cout, act, k, 40 + cout)
    fr = torch.from_numpy(frames_for(26, 34, 500 + cout, L=12)).cuda()
    outs = {}
    for mode in ("fused", "separate"):
        if mode == "fused":
            monkeypatch.setenv("ST_FUSE_TC", "1")
        else:
            monkeypatch.delenv("ST_FUSE_TC", raising=False)
        enc = Encoder(net, fr.shape[0], fr.shape[1], precision="bf16")
        res = []
        for th in (0.02, 0.0, 0.08):
            for _ in range(2):
                enc.encode_reference(fr[:, 0])
                enc.encode_diff(fr[:, 1:], th)
            torch.cuda.synchronize()
            res.append(([enc.outputs(t).cpu().numpy().copy() for t in enc.taps], enc.get_sparsity()[0].copy()))
        outs[mode] = res
        enc.close()
    for (og, cg), (oe, ce) in zip(outs["fused"], outs["separate"]):
        assert np.array_equal(cg, ce), "per-site per-frame counts"
        for a, b in zip(og, oe):
            assert np.array_equal(a, b), f"tap outputs differ (max {np.abs(a - b).max():.3e})"


def test_depthwise_over_25_taps_rejected():
    """Depthwise kernels take at most 5x5 taps; a 7x7 depthwise conv is
    rejected at create (ST_ERR_UNSUPPORTED) instead of silently dropping
    taps 25-48."""
    from paper_2410_20790_b200 import Encoder
    from paper_2410_20790_b200.binding import StError
    n = Net(3, 16, 16, "dw7")
    x = n.relu(n.conv(-1, 16, 3, 1, 1))
    x = n.relu(n.conv(x, 16, 7, 1, 3, groups=16))
    n.output(n.conv(x, 8, 1, 1, 0))
    init_weights(n, 3)
    with pytest.raises(StError, match="unsupported|UNSUPPORTED"):
        Encoder(n, 1, 4, precision="bf16")
