"""Streaming continuation (-m gpu): with cfg.streaming the
per-site caches of the vanilla DeltaCNN schedule (the Subtraction
buffer S, each site's x_acc / y_acc, each tap's last output) persist across
st_encode_diff calls, so a chunk split over several calls gives exactly the
results of one call over all its frames (Diff Computation is frame-
sequential per pixel, Eq.3), and chunks may be longer than one call's
33-frame window (reading R25)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import workloads as W
from workloads import init_weights
from gpu_harness import make_frames
from netgen import random_net, random_frames

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _single(net, fr, th, precision):
    import torch
    from paper_2410_20790_b200 import Encoder
    B, L = fr.shape[:2]
    enc = Encoder(net, B, L, precision=precision)
    x = torch.from_numpy(fr).cuda()
    enc.encode_reference(x[:, 0])
    enc.encode_diff(x[:, 1:], th)
    torch.cuda.synchronize()
    out = [enc.outputs(t).cpu().numpy().copy() for t in enc.taps]
    cnt = enc.get_sparsity()[0].copy()
    enc.close()
    return out, cnt


def _streamed(net, fr, th, precision, splits, max_frames):
    """reference + one diff call per split; returns per-tap outputs [B][L]..."""
    import torch
    from paper_2410_20790_b200 import Encoder
    B, L = fr.shape[:2]
    enc = Encoder(net, B, max_frames, precision=precision, streaming=True)
    x = torch.from_numpy(fr).cuda()
    enc.encode_reference(x[:, 0])
    outs = [[] for _ in enc.taps]
    cnts = []
    t0 = 1
    for k, n in enumerate(splits):
        enc.encode_diff(x[:, t0:t0 + n].contiguous() if n else None, th)
        torch.cuda.synchronize()
        for j, t in enumerate(enc.taps):
            o = enc.outputs(t).cpu().numpy()
            outs[j].append(o if k == 0 else o[:, 1:])   # frame 0 of a continuation = previous last frame
        if n:
            cnts.append(enc.get_sparsity()[0].copy())
        t0 += n
    enc.close()
    assert t0 == L
    return [np.concatenate(o, axis=1) for o in outs], np.concatenate(cnts, axis=2)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("model", ["crnn", "resnet18", "random"])
def test_streaming_equals_single_call(precision, model):
    if model == "crnn":
        cfg = W.get_config(2)
        net = cfg.build_net()
        fr = make_frames(cfg, 3, L=14)
    elif model == "resnet18":
        net = W.models.resnet18(72, 104)
        init_weights(net, 13)
        fr = W.to_float(W.gen_video(2, 14, 72, 104, 3, 79, n_objects=4, size=(8, 24), speed=(1, 3),
                                    noise_q=0.1, noise_amp=2))
    else:
        net = random_net(4242, allow_se=False)
        fr = np.stack([random_frames(70 + b, 14, net.in_h, net.in_w, net.in_c) for b in range(2)])
    th = 0.05
    ref_out, ref_cnt = _single(net, fr, th, precision)
    out, cnt = _streamed(net, fr, th, precision, splits=[5, 0, 1, 7], max_frames=8)
    assert np.array_equal(cnt, ref_cnt)
    for a, b in zip(out, ref_out):
        assert a.shape == b.shape
        assert np.array_equal(a, b)


def test_streaming_long_chunk_vs_oracle():
    """A 45-frame chunk (beyond one call's 33-frame window) streamed in three
    calls matches the oracle over all 45 frames bit-exactly (FP32 mode)."""
    cfg = W.get_config(1)
    net = cfg.build_net()
    fr = W.to_float(W.gen_video(2, 45, cfg.h, cfg.w, cfg.c, 4545, **cfg.video))
    out, cnt = _streamed(net, fr, cfg.theta_fixed, "fp32", splits=[20, 20, 4], max_frames=21)
    for b in range(2):
        r = oracle.run_chunk(net, fr[b], cfg.theta_fixed, want_masks=False)
        tap = max(r["taps"])
        assert np.array_equal(out[-1][b], r["taps"][tap])
        assert np.array_equal(cnt[b], r["counts"])


def test_streaming_rejects_se_and_reference_restarts():
    import torch
    from paper_2410_20790_b200 import Encoder, StError
    net = W.models.efficientnet_b0(64, 64)
    init_weights(net, 5)
    with pytest.raises(StError):
        Encoder(net, 1, 4, streaming=True)
    # a new st_encode_reference restarts the chunks: same results as a fresh encoder
    cfg = W.get_config(1)
    net = cfg.build_net()
    fr = make_frames(cfg, 2, L=6)
    ref_out, _ = _single(net, fr, 0.05, "fp32")
    enc = Encoder(net, 2, 6, streaming=True)
    x = torch.from_numpy(fr).cuda()
    for _ in range(2):
        enc.encode_reference(x[:, 0])
        enc.encode_diff(x[:, 1:], 0.05)
    torch.cuda.synchronize()
    assert np.array_equal(enc.outputs(enc.taps[0]).cpu().numpy(), ref_out[0])
