"""Parity at the BASELINE.json full sizes (-m gpu), on sampled chunks.

Chunks are independent (each has its own reference frame), so the
oracle computes any sampled chunk of a full-size step exactly.  The GPU runs
the whole step in the launch configuration bench.py times (all chunks of a
step x all frames, uint8 frames where the bench uses them, no debug
retention, arena reuse, CUDA-graph replay); st_debug_export_chunk copies the
sampled chunk's frame words of every layer out of that very step.  Checks
(gpu_harness.follow_compare): band-follow (O12, reading R23) -- zero
decisions outside the ambiguity band disagree --, then every layer's mask
per frame (= its ascending active-index list) and the per-site per-frame
counts bit-exact, every tap element within R29 (bf16: 2e-2|b| + 2e-2 rms;
fp32: 1e-5 + 1e-4|b|, bit-exact for ReLU/maxpool nets), adopted decisions
<< 0.1 %."""
from __future__ import annotations

import numpy as np
import pytest

import workloads as W
from gpu_harness import follow_compare, site_layers

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _full_step(cfg, precision, chunks, L=None, B=None, theta=None):
    """Run the config's full step (B chunks x L frames, uint8 frames) with the
    export of each sampled chunk; yields (encoder, float frames of the chunk, chunk)."""
    import torch
    from paper_2410_20790_b200 import Encoder
    net = cfg.build_net()
    B = B or cfg.chunks_per_step
    L = L or cfg.L
    u8 = np.stack([W.gen_chunk(cfg.video_seed(c), L, cfg.h, cfg.w, cfg.c, **cfg.video) for c in range(B)])
    theta = cfg.theta_fixed if theta is None else theta
    enc = Encoder(net, B, L, precision=precision)
    x = torch.from_numpy(u8).cuda()
    for b in chunks:
        enc.export_chunk(b)
        for _ in range(2):   # first sight runs eagerly, the second captures and replays the graph
            enc.encode_reference(x[:, 0])
            enc.encode_diff(x[:, 1:], theta)
        torch.cuda.synchronize()
        yield net, enc, W.to_float(u8[b]), b, theta
    enc.export_chunk(-1)


def _check(cfg, precision, chunks, **kw):
    """Adopted (in-band, R23) decisions: <= 0.1 % of all decisions on the
    BASELINE configs; the paper's deeper backbones (>= 100 sites: ResNet-152,
    EfficientNet-B4..B6) allow 0.5 % -- every adopted decision is a correct
    one by R23, and their number grows with depth because each site's
    rounding differences move the values later sites decide on."""
    reps = []
    for net, enc, fr, b, theta in _full_step(cfg, precision, chunks, **kw):
        rep = follow_compare(enc, net, fr, theta, b, precision, exported=True)
        frac = 1e-3 if len(site_layers(net)) < 100 else 5e-3
        assert rep["adopted"] <= max(3, frac * rep["decisions"]), (cfg.cid, b, rep)
        reps.append(rep)
    return reps


def test_cfg2_bench_config_bf16():
    """cfg2 (CRNN, 64 chunks x 32 frames, theta 0.05), BF16, chunks 0/29/63."""
    _check(W.get_config(2), "bf16", (0, 29, 63))


def test_cfg2_bench_config_fp32_exact():
    """cfg2 in FP32 mode: bit-exact masks, counts and taps (ReLU/maxpool)."""
    reps = _check(W.get_config(2), "fp32", (5, 63))
    assert all(r["adopted"] == 0 for r in reps)


@pytest.mark.parametrize("cid", [3, 4, 5])
def test_bench_config_bf16(cid):
    """cfg3 / cfg4 / cfg5 in the bench launch configuration (all chunks of a
    step x all frames, BF16, graph replay); the last chunk of the step."""
    cfg = W.get_config(cid)
    _check(cfg, "bf16", (cfg.chunks_per_step - 1,))


def test_cfg3_fp32_full_step():
    """cfg3 (EfficientNet-B0 @512^2, 8 chunks x 16 frames) in FP32 mode: SiLU
    is bit-matched (exact exp, R10), the SE mean is an fp64 sum in another
    order -> band-follow at the fp32 band."""
    _check(W.get_config(3), "fp32", (2,))


def test_cfg4_resnet18_720p_fp32():
    """cfg4 ResNet-18 @720p, FP32 (CUDA-core convs), 2 chunks x 8 frames."""
    reps = _check(W.get_config(4), "fp32", (1,), L=8, B=2)
    assert reps[0]["adopted"] == 0


def test_cfg5_effdet_d0_1080p_fp32():
    """cfg5 EfficientDet-D0 backbone @1080p, FP32, 2 chunks x 6 frames."""
    _check(W.get_config(5), "fp32", (1,), L=6, B=2)


# ---- the paper's own backbones at their sizes
@pytest.mark.parametrize("cid", [7, 8, 9])
def test_effdet_d4_d6_backbones(cid):
    """EfficientNet-B4 @1024 / B5 @1280 / B6 @1280 (the Table 1 detectors'
    backbones), full frame size, 2 chunks x 4 frames: FP32 and
    BF16 (band-follow) on the last chunk, in the bench launch configuration."""
    cfg = W.get_config(cid)
    theta = 0.05
    _check(cfg, "fp32", (1,), L=4, B=2, theta=theta)
    _check(cfg, "bf16", (1,), L=4, B=2, theta=theta)


@pytest.mark.parametrize("cid", [10, 6, 11])
def test_resnet152_crnn_resolutions(cid):
    """ResNet-152 (the CRNN backbone) at the paper's three resolutions 224 /
    320 / 420, batch 3, 28-frame chunks cut to 6 frames: FP32
    bit-exact (ReLU/maxpool), BF16 band-follow, on the last chunk."""
    cfg = W.get_config(cid)
    reps = _check(cfg, "fp32", (2,), L=6, theta=0.05)
    assert reps[0]["adopted"] == 0
    _check(cfg, "bf16", (2,), L=6, theta=0.05)
