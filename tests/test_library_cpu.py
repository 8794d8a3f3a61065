"""CPU-side checks of libsparsetem.so (-m "not gpu"): it loads, exports every
symbol include/sparsetem.h declares, refuses to create an encoder without a
GPU (no CPU fallback), and its host controller agrees with the
oracle's independently written controller."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2410_20790_b200 import build as B
    B.build()
    from paper_2410_20790_b200 import load_library
    return load_library()


def _declared():
    src = open(os.path.join(ROOT, "include", "sparsetem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(st_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    from paper_2410_20790_b200.binding import SIGNATURES
    assert set(SIGNATURES) == set(names)


def test_no_cpu_fallback(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2410_20790_b200 import Encoder, StError
    import workloads as W
    with pytest.raises(StError):
        Encoder(W.get_config(1).build_net(), 1, 8)


def test_status_strings(L):
    assert L.st_status_string(0) == b"ok"
    assert L.st_status_string(4) == b"unsupported"


@pytest.mark.parametrize("policy", ["fixed", "bst", "ibst"])
def test_controller_matches_oracle(L, policy):
    from paper_2410_20790_b200 import ThresholdController
    rng = np.random.default_rng(1)
    a = ThresholdController(6, policy=policy, cycle=4)
    b = oracle.Controller(oracle.ControllerConfig(policy=policy, cycle=4), 6)
    for _ in range(60):
        px = rng.integers(1000, 10 ** 6, 6)
        act = (px * rng.random(6)).astype(np.int64)
        a.observe(act, px)
        b.observe(act, px)
        assert np.array_equal(a.thresholds(), b.thresholds())
        th, lo, hi, fr = a.state()
        assert np.array_equal(fr.astype(bool), np.array(b.frozen))


def test_controller_rejects_bad_config(L):
    from paper_2410_20790_b200 import ThresholdController, StError
    with pytest.raises(StError):
        ThresholdController(3, policy="bst", T=0.99, eps=0.05)
