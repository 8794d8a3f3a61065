"""Cache-lifetime scheduler memory (PAPER.md P:139 vs P:152:
"SparseBatch ... keeps only one buffer for Subtraction and one for
Accumulation", DeltaCNN's caches grow with the number of non-linear layers),
-m gpu, through the C ABI.

* Row capacity from measured occupancy: st_encoder_fit_capacity re-plans the
  arena from the largest row counts seen; the step re-issued on the smaller
  arena gives bit-identical results.
* Overflow: an encoder whose capacities are too small reports
  ST_ERR_CAPACITY (nothing is written past a buffer), and fit + re-issue
  recovers the exact results.
* PIN13 on the product: SparseBatch persistent bytes do not depend on the
  number of non-linear layers; the streaming (vanilla) caches grow with it.
"""
from __future__ import annotations

import numpy as np
import pytest

import workloads as W
from workloads import Net, init_weights

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2410_20790_b200 import load_library
    load_library()


def _run(enc, fr, th):
    import torch
    enc.encode_reference(fr[:, 0])
    enc.encode_diff(fr[:, 1:], th)
    torch.cuda.synchronize()
    ok = enc.step_ok()
    return ok, ([enc.outputs(t).cpu().numpy().copy() for t in enc.taps] if ok else None)


def _case(model):
    if model == "crnn":
        cfg = W.get_config(2)
        net = cfg.build_net()
        from gpu_harness import make_frames
        return net, make_frames(cfg, 4, L=12)
    net = W.models.efficientnet_b0(96, 128) if model == "effnet" else W.models.resnet18(72, 104)
    init_weights(net, 21)
    fr = W.to_float(W.gen_video(2, 9, net.in_h, net.in_w, 3, 321, n_objects=4, size=(8, 24), speed=(1, 3),
                                noise_q=0.1, noise_amp=2))
    return net, fr


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("model", ["crnn", "resnet18", "effnet"])
def test_fit_capacity_bit_identical(model, precision):
    import torch
    from paper_2410_20790_b200 import Encoder
    net, fr_np = _case(model)
    fr = torch.from_numpy(fr_np).cuda()
    enc = Encoder(net, fr.shape[0], fr.shape[1], precision=precision)
    ok, full = _run(enc, fr, 0.03)
    assert ok
    _, _, arena_full = enc.memory_report().values()
    cap0, peak = enc.capacity()
    own = cap0 >= 0
    assert np.all(peak[own] <= cap0[own])
    enc.fit_capacity(1.25)
    cap1, _ = enc.capacity()
    assert np.all(cap1[own] <= cap0[own]) and np.all(cap1[own] >= np.minimum(cap0[own], peak[own]))
    arena_fit = enc.memory_report()["arena_bytes"]
    assert arena_fit < arena_full
    for _ in range(2):   # graph capture on the new arena (first sight eager, then replay)
        ok, got = _run(enc, fr, 0.03)
        assert ok
        for a, b in zip(got, full):
            assert np.array_equal(a, b)
    enc.close()


@pytest.mark.parametrize("model", ["crnn", "effnet"])
def test_capacity_overflow_reissue(model):
    import torch
    from paper_2410_20790_b200 import Encoder, CapacityError
    net, fr_np = _case(model)
    fr = torch.from_numpy(fr_np).cuda()
    ref = Encoder(net, fr.shape[0], fr.shape[1], precision="fp32")
    _, full = _run(ref, fr, 0.0)   # theta 0: many rows
    ref.close()
    enc = Encoder(net, fr.shape[0], fr.shape[1], precision="fp32", row_frac=1e-6)   # 4096-row floor
    enc.encode_reference(fr[:, 0])
    enc.encode_diff(fr[:, 1:], 0.0)
    assert not enc.step_ok()
    with pytest.raises(CapacityError):
        enc.get_sparsity()
    for it in range(len(net.layers) + 1):   # clamped tensors hide downstream rows: a few rounds
        enc.fit_capacity(1.0)
        ok, got = _run(enc, fr, 0.0)
        if ok:
            break
    assert ok, "re-issue did not converge"
    for a, b in zip(got, full):
        assert np.array_equal(a, b)
    enc.get_sparsity()   # valid again
    enc.close()


def _chain(k, streaming):
    n = Net(3, 24, 40, f"chain{k}")
    x = n.conv(-1, 16, 3, 1, 1)
    for _ in range(k):
        x = n.relu(x)
        x = n.conv(x, 16, 3, 1, 1)
    n.output(x)
    init_weights(n, 5)
    return n


def test_persistent_bytes_independent_of_depth():
    """PIN13 on the product (P:139 vs P:152): SparseBatch persistent bytes
    (staged reference + Accumulation outputs) are the same for 2, 4 and 8
    non-linear layers; the streaming encoder's caches grow by the same
    amount per added site (affine in the number of sites)."""
    from paper_2410_20790_b200 import Encoder
    sb, va = [], []
    for k in (2, 4, 8):
        net = _chain(k, False)
        e = Encoder(net, 2, 9, precision="bf16")
        sb.append(e.memory_report()["persistent_bytes"])
        e.close()
        e = Encoder(net, 2, 9, precision="bf16", streaming=True)
        va.append(e.memory_report()["persistent_bytes"])
        e.close()
    assert sb[0] == sb[1] == sb[2]
    assert va[1] - va[0] > 0 and (va[2] - va[1]) == 2 * (va[1] - va[0])
