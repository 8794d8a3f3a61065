"""GPU parity: the CUDA path through the C ABI vs the oracle (-m gpu).

FP32 mode: masks / active-index lists of every layer and frame are
bit-exact, delta rows, tap outputs and per-site counts are bit-exact
(fixed fma order, reading R18).  Sizes span several tiles and a ragged tail;
full BASELINE sizes are checked on sampled chunks (chunks are independent,
P:113, so the oracle computes a sampled chunk exactly)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from workloads import Net, init_weights
from gpu_harness import gpu_run, compare_chunk, make_frames, within
from netgen import random_net, random_frames

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2410_20790_b200 import load_library
    load_library()


def test_cfg1_toy_exact():
    cfg = W.get_config(1)
    net = cfg.build_net()
    fr = make_frames(cfg, 3)
    enc, _ = gpu_run(net, fr, cfg.theta_fixed)
    for b in range(3):
        compare_chunk(enc, net, fr[b], cfg.theta_fixed, b)


@pytest.mark.parametrize("theta", [0.0, 0.02, 0.1])
def test_cfg1_thresholds(theta):
    cfg = W.get_config(1)
    net = cfg.build_net()
    fr = make_frames(cfg, 2)
    enc, _ = gpu_run(net, fr, theta)
    for b in range(2):
        compare_chunk(enc, net, fr[b], theta, b)


def test_cfg2_crnn_exact():
    cfg = W.get_config(2)
    net = cfg.build_net()
    fr = make_frames(cfg, 2, L=12)
    enc, _ = gpu_run(net, fr, cfg.theta_fixed)
    for b in range(2):
        compare_chunk(enc, net, fr[b], cfg.theta_fixed, b)


def test_resnet18_small_exact():
    net = W.models.resnet18(64, 96)
    init_weights(net, 11)
    cfg = W.get_config(4)
    u8 = W.gen_video(2, 6, 64, 96, 3, 77, n_objects=4, size=(8, 24), speed=(1, 3), noise_q=0.1, noise_amp=2)
    fr = W.to_float(u8)
    enc, _ = gpu_run(net, fr, 0.05)
    for b in range(2):
        compare_chunk(enc, net, fr[b], 0.05, b)


@pytest.mark.parametrize("seed", range(16))
def test_random_nets(seed):
    net = random_net(900 + seed, allow_se=False, allow_silu=(seed % 2 == 0))
    fr = np.stack([random_frames(seed * 3 + b, 7, net.in_h, net.in_w, net.in_c) for b in range(2)])
    th = 0.03 + 0.01 * (seed % 4)
    enc, _ = gpu_run(net, fr, th)
    exact = not any(l["kind"] == W.SILU for l in net.layers)
    for b in range(2):
        compare_chunk(enc, net, fr[b], th, b, exact=exact)


def test_identical_frames_empty_masks():
    cfg = W.get_config(1)
    net = cfg.build_net()
    fr = np.repeat(make_frames(cfg, 1, L=1), 5, axis=1)
    enc, _ = gpu_run(net, fr, 0.05)
    act, sa, _ = enc.get_sparsity()
    assert act.sum() == 0 and sa.sum() == 0
    out = enc.outputs(3)[0].cpu().numpy()
    for t in range(1, 5):
        assert np.array_equal(out[t], out[0])


def test_dense_only_and_max_frames():
    cfg = W.get_config(1)
    net = cfg.build_net()
    fr = make_frames(cfg, 1, L=33, h=24, w=40)
    net = W.models.toy_encoder(24, 40)
    init_weights(net, 3)
    enc, _ = gpu_run(net, fr, 0.05)                  # 32 diff frames: full frame word
    compare_chunk(enc, net, fr[0], 0.05, 0)
    enc0, _ = gpu_run(net, fr[:, :1], 0.05)          # n_diff = 0: dense pass only
    o = enc0.outputs(3)[0, 0].cpu().numpy()
    assert np.array_equal(o, oracle.dense_forward(net, fr[0, 0])[2])


def test_cfg2_full_size_sampled():
    """BASELINE cfg2 at full size (B=64 chunks x L=32) in the bench's launch
    configuration; sampled chunks checked exactly against the oracle."""
    cfg = W.get_config(2)
    net = cfg.build_net()
    fr = make_frames(cfg, cfg.chunks_per_step)
    enc, _ = gpu_run(net, fr, cfg.theta_fixed, debug=False)
    act, _, _ = enc.get_sparsity()
    tap = enc.taps[0]
    out = enc.outputs(tap)
    for b in (0, 37, 63):
        r = oracle.run_chunk(net, fr[b], cfg.theta_fixed, want_masks=False)
        assert np.array_equal(out[b].cpu().numpy(), r["taps"][tap]), f"chunk {b}"
        assert np.array_equal(act[b], r["counts"])


@pytest.mark.parametrize("theta", [0.0, 0.01, 0.05])
def test_se_site(theta):
    """SE site (reading R8): gate refresh schedule, touched sets, values.
    SiLU/sigmoid use (float)exp((double)x) on both sides (R10); the SE mean
    is an fp64 sum in a different order on the GPU, so values are compared
    at the fp32 tolerance and masks exactly (a rounding-order flip of the
    fp32 mean would show up here)."""
    n = Net(3, 12, 14)
    x = n.silu(n.conv(-1, 24, 3))
    s = n.se(x, 6)
    n.output(n.conv(s, 16, 1, 1, 0))
    init_weights(n, 21)
    fr = np.stack([random_frames(40 + b, 9, 12, 14, 3, p_change=0.25, scale=0.3) for b in range(3)])
    enc, _ = gpu_run(n, fr, theta)
    for b in range(3):
        compare_chunk(enc, n, fr[b], theta, b, exact=False)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_se_sums_forms_identical(precision, monkeypatch):
    """The SE per-frame delta sums (R8) from per-frame row lists
    (ST_SE_SUMS=3) and from the per-(frame, channel group) sweep (0) give the
    same outputs and counts: the fp64 sums of the same rows in another order."""
    import torch
    from paper_2410_20790_b200 import Encoder
    net = W.models.efficientnet_b0(64, 96)
    init_weights(net, 17)
    u8 = W.gen_video(2, 9, 64, 96, 3, 77, n_objects=4, size=(8, 24), speed=(1, 3), noise_q=0.1, noise_amp=2)
    fr = torch.from_numpy(W.to_float(u8)).cuda()
    outs = []
    for mode in ("0", "3"):
        monkeypatch.setenv("ST_SE_SUMS", mode)
        enc = Encoder(net, fr.shape[0], fr.shape[1], precision=precision)
        res = []
        for th in (0.03, 0.0):
            enc.encode_reference(fr[:, 0])
            enc.encode_diff(fr[:, 1:], th)
            torch.cuda.synchronize()
            res.append(([enc.outputs(t).cpu().numpy().copy() for t in enc.taps], enc.get_sparsity()[0].copy()))
        outs.append(res)
        enc.close()
    for (og, cg), (oe, ce) in zip(*outs):
        assert np.array_equal(cg, ce)
        for a, b in zip(og, oe):
            assert np.array_equal(a, b), f"max {np.abs(a - b).max():.3e}"


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_tc_dense_act_epilogue_identical(precision, monkeypatch):
    """A tensor-core conv whose only consumer is a ReLU / SiLU writes the
    site's dense output f(x0) (+ bf16 shadow) from its staged epilogue
    (opt-in, ST_TC_ACT=1); the results equal the separate dense activation
    pass (ST_TC_ACT=0) bit for bit (MBConv expand convs, ResNet-style 3x3
    convs, a stem)."""
    import torch
    from paper_2410_20790_b200 import Encoder
    n = Net(3, 24, 40, "tcact")
    x = n.relu(n.conv(-1, 32, 3, 2, 1))                 # stem (tcgen05 small) + ReLU
    y = n.silu(n.conv(x, 96, 1, 1, 0))                  # expand 1x1 + SiLU
    y = n.silu(n.conv(y, 96, 3, 1, 1, groups=96))
    y = n.conv(y, 40, 1, 1, 0)
    z = n.relu(n.conv(y, 72, 3, 1, 1))                  # 3x3 tcgen05 + ReLU (c_out not a multiple of 32)
    n.output(n.conv(z, 16, 1, 1, 0))
    init_weights(n, 23)
    u8 = W.gen_video(2, 7, 24, 40, 3, 55, n_objects=3, size=(4, 12), speed=(1, 2), noise_q=0.1, noise_amp=2)
    fr = torch.from_numpy(W.to_float(u8)).cuda()
    outs = []
    for mode in ("1", "0"):
        monkeypatch.setenv("ST_TC_ACT", mode)
        enc = Encoder(n, fr.shape[0], fr.shape[1], precision=precision)
        res = []
        for th in (0.03, 0.0):
            enc.encode_reference(fr[:, 0])
            enc.encode_diff(fr[:, 1:], th)
            torch.cuda.synchronize()
            res.append(([enc.outputs(t).cpu().numpy().copy() for t in enc.taps], enc.get_sparsity()[0].copy()))
        outs.append(res)
        enc.close()
    for (og, cg), (oe, ce) in zip(*outs):
        assert np.array_equal(cg, ce)
        for a, b in zip(og, oe):
            assert np.array_equal(a, b), f"max {np.abs(a - b).max():.3e}"


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("model", ["effnet", "resnet"])
def test_dense_diff_overlap_identical(precision, model, monkeypatch):
    """The reference (dense) pass on its own stream, up to ST_OVERLAP_K layers
    ahead of the diff pass (arena lifetimes extended to match), gives the same
    outputs and counts as one stream (ST_OVERLAP=0), eager and replayed from
    the captured graph, with lookahead 1, 3 and 12."""
    import torch
    from paper_2410_20790_b200 import Encoder
    if model == "effnet":
        net = W.models.efficientnet_b0(64, 96)
    else:
        net = W.models.resnet18(64, 96)
    init_weights(net, 29)
    u8 = W.gen_video(2, 9, 64, 96, 3, 81, n_objects=4, size=(8, 24), speed=(1, 3), noise_q=0.1, noise_amp=2)
    fr = torch.from_numpy(W.to_float(u8)).cuda()
    outs = []
    for ov, k in (("0", "3"), ("1", "1"), ("1", "3"), ("1", "12")):
        monkeypatch.setenv("ST_OVERLAP", ov)
        monkeypatch.setenv("ST_OVERLAP_K", k)
        enc = Encoder(net, fr.shape[0], fr.shape[1], precision=precision)
        res = []
        for th in (0.03, 0.03, 0.0):   # first sight eager, then graph capture + replay
            enc.encode_reference(fr[:, 0])
            enc.encode_diff(fr[:, 1:], th)
            torch.cuda.synchronize()
            res.append(([enc.outputs(t).cpu().numpy().copy() for t in enc.taps], enc.get_sparsity()[0].copy()))
        outs.append(res)
        enc.close()
    for other in outs[1:]:
        for (og, cg), (oe, ce) in zip(outs[0], other):
            assert np.array_equal(cg, ce)
            for a, b in zip(og, oe):
                assert np.array_equal(a, b), f"max {np.abs(a - b).max():.3e}"


def test_efficientnet_small():
    net = W.models.efficientnet_b0(64, 64)
    init_weights(net, 13)
    u8 = W.gen_video(2, 6, 64, 64, 3, 99, n_objects=4, size=(8, 24), speed=(1, 3), noise_q=0.1, noise_amp=2)
    fr = W.to_float(u8)
    enc, _ = gpu_run(net, fr, 0.05)
    for b in range(2):
        compare_chunk(enc, net, fr[b], 0.05, b, exact=False)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_graph_replay_matches_eager(precision, monkeypatch):
    """Steps replayed from a captured CUDA graph (thresholds refreshed from
    device memory each step) are bit-identical to eager launches, and the
    FP32 ones to the oracle."""
    import torch
    from paper_2410_20790_b200 import Encoder
    cfg = W.get_config(2)
    net = cfg.build_net()
    fr_np = make_frames(cfg, 4, L=9)
    fr = torch.from_numpy(fr_np).cuda()
    thetas = [0.05, 0.03, 0.08, 0.05]
    outs = {}
    for mode in ("graph", "eager"):
        if mode == "eager":
            monkeypatch.setenv("ST_NO_GRAPHS", "1")
        enc = Encoder(net, 4, 9, precision=precision)
        res = []
        for th in thetas:
            enc.encode_reference(fr[:, 0])
            enc.encode_diff(fr[:, 1:], th)
            torch.cuda.synchronize()
            res.append((enc.outputs(enc.taps[0]).cpu().numpy().copy(), enc.get_sparsity()[0].copy()))
        outs[mode] = res
        enc.close()
    for (og, cg), (oe, ce) in zip(outs["graph"], outs["eager"]):
        assert np.array_equal(og, oe) and np.array_equal(cg, ce)
    if precision == "fp32":
        r = oracle.run_chunk(net, fr_np[2], thetas[3], want_masks=False)
        assert np.array_equal(outs["graph"][3][0][2], r["taps"][max(r["taps"])])


def test_errors_and_state():
    from paper_2410_20790_b200 import Encoder, StError
    import torch
    net = W.get_config(1).build_net()
    enc = Encoder(net, 2, 4)
    fr = torch.zeros(2, 3, 64, 64, 3, device="cuda")
    with pytest.raises(StError):            # diff before reference
        enc.encode_diff(fr, 0.05)
    enc.encode_reference(fr[:, 0])
    with pytest.raises(StError):            # too many frames
        enc.encode_diff(torch.zeros(2, 5, 64, 64, 3, device="cuda"), 0.05)
    with pytest.raises(StError):            # negative threshold
        enc.encode_diff(fr, -1.0)
    enc.encode_diff(fr, 0.05)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("model", ["crnn", "resnet18"])
def test_fused_relu_maxpool_matches_unfused(precision, model, monkeypatch):
    """The ReLU -> maxpool pass (one tile-resident kernel, ReLU rows kept on
    chip) gives bit-identical tap outputs and per-site counts to the separate
    ReLU and maxpool site kernels (ST_NO_FUSE=1), in both modes."""
    import torch
    from paper_2410_20790_b200 import Encoder
    if model == "crnn":
        cfg = W.get_config(2)
        net = cfg.build_net()
        fr_np = make_frames(cfg, 3, L=10)
    else:
        net = W.models.resnet18(72, 104)
        init_weights(net, 12)
        fr_np = W.to_float(W.gen_video(2, 9, 72, 104, 3, 78, n_objects=4, size=(8, 24), speed=(1, 3),
                                       noise_q=0.1, noise_amp=2))
    fr = torch.from_numpy(fr_np).cuda()
    outs = {}
    for mode in ("fused", "separate"):
        if mode == "separate":
            monkeypatch.setenv("ST_NO_FUSE", "1")
        enc = Encoder(net, fr.shape[0], fr.shape[1], precision=precision)
        res = []
        for th in (0.05, 0.0, 0.1):
            enc.encode_reference(fr[:, 0])
            enc.encode_diff(fr[:, 1:], th)
            torch.cuda.synchronize()
            res.append(([enc.outputs(t).cpu().numpy().copy() for t in enc.taps], enc.get_sparsity()[0].copy()))
        outs[mode] = res
        enc.close()
    for (og, cg), (oe, ce) in zip(outs["fused"], outs["separate"]):
        assert np.array_equal(cg, ce)
        for a, b in zip(og, oe):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("C,k,s,p,h,w", [(16, 2, 2, 0, 20, 36), (32, 3, 2, 1, 23, 41), (64, 2, 1, 0, 9, 30),
                                         (16, 3, 1, 1, 17, 17), (128, 2, 2, 0, 13, 21), (32, 3, 3, 0, 19, 26)])
def test_relu_maxpool_geometries_exact(C, k, s, p, h, w):
    """conv -> ReLU -> maxpool at tile-kernel widths over pool geometries with
    and without full window coverage (odd maps, k < s gaps): FP32 bit-exact
    against the oracle, fused or not."""
    net = Net(3, h, w)
    c1 = net.conv(-1, C, 3, 1, 1)
    r1 = net.relu(c1)
    mp = net.maxpool(r1, k, s, p)
    c2 = net.conv(mp, 8, 3, 1, 1)
    net.output(net.relu(c2))
    init_weights(net, 100 + C + k)
    fr = np.stack([random_frames(C + b, 6, h, w, 3) for b in range(2)])
    for th in (0.0, 0.04):
        enc, _ = gpu_run(net, fr, th)
        for b in range(2):
            compare_chunk(enc, net, fr[b], th, b)
        enc.close()


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("model", ["crnn", "resnet18"])
def test_u8_frames_match_float(precision, model):
    """st_encode_reference_u8 / st_encode_diff_u8 on uint8 frames are
    bit-identical to the fp32 calls on v / 255.0f (reading R20), including a
    streaming continuation."""
    import torch
    from paper_2410_20790_b200 import Encoder
    if model == "crnn":
        cfg = W.get_config(2)
        net = cfg.build_net()
        u8 = W.gen_video(3, 10, cfg.h, cfg.w, cfg.c, 2024, **cfg.video)
    else:
        net = W.models.resnet18(72, 104)
        init_weights(net, 14)
        u8 = W.gen_video(2, 10, 72, 104, 3, 80, n_objects=4, size=(8, 24), speed=(1, 3), noise_q=0.1, noise_amp=2)
    xf = torch.from_numpy(W.to_float(u8)).cuda()
    xu = torch.from_numpy(np.ascontiguousarray(u8)).cuda()
    res = {}
    for kind, x in (("f32", xf), ("u8", xu)):
        enc = Encoder(net, x.shape[0], 6, precision=precision, streaming=True)
        enc.encode_reference(x[:, 0])
        outs = []
        for a, b in ((1, 6), (6, 10)):
            enc.encode_diff(x[:, a:b], 0.05)
            torch.cuda.synchronize()
            outs.append(([enc.outputs(t).cpu().numpy().copy() for t in enc.taps], enc.get_sparsity()[0].copy()))
        res[kind] = outs
        enc.close()
    for (of, cf), (ou, cu) in zip(res["f32"], res["u8"]):
        assert np.array_equal(cf, cu)
        for a, b in zip(of, ou):
            assert np.array_equal(a, b)


def test_resnet152_small_exact():
    """N3: the paper's ResNet-152 backbone (2048-channel ReLU sites on the
    wide shared-memory site kernel, bottleneck joins), FP32 bit-exact."""
    net = W.models.resnet152(48, 64)
    init_weights(net, 21)
    u8 = W.gen_video(2, 5, 48, 64, 3, 81, n_objects=3, size=(8, 20), speed=(1, 3), noise_q=0.1, noise_amp=2)
    fr = W.to_float(u8)
    enc, _ = gpu_run(net, fr, 0.05)
    for b in range(2):
        compare_chunk(enc, net, fr[b], 0.05, b)


def test_resnet152_bf16():
    """N3 ResNet-152 in BF16 mode (tcgen05 convs, 155 of them): band-follow
    parity (O12) against the oracle's BF16 contract -- zero decisions outside
    the R23 band disagree, masks / index lists / counts exact, rows and taps
    within R29-BF16."""
    from gpu_harness import follow_compare, gpu_run
    net = W.models.resnet152(64, 64)
    init_weights(net, 22)
    fr = W.to_float(W.gen_video(2, 6, 64, 64, 3, 82, n_objects=3, size=(8, 20), speed=(1, 3), noise_q=0.1,
                                noise_amp=2))
    enc, _ = gpu_run(net, fr, 0.05, precision="bf16")
    for b in range(2):
        rep = follow_compare(enc, net, fr[b], 0.05, b, "bf16")
        assert rep["adopted"] <= max(3, 1e-3 * rep["decisions"]), rep
