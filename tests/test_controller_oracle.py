"""PIN11: the BST/IBST controller (readings R15/R16) against
properties fixed by binary search, not by re-typing the rule:
termination bound, band achievement vs an exhaustive grid scan, and IBST
re-convergence after a regime switch."""
from __future__ import annotations

import math

import numpy as np

from oracle import Controller, ControllerConfig


def _env(rng):
    s0, s1 = rng.uniform(0.0, 0.8), rng.uniform(0.96, 1.0)
    g = rng.uniform(0.2, 3.0)
    return lambda th: s0 + (s1 - s0) * (min(max(th, 0.0), 1.0) ** g)


def _run(ctl, env, n, px=10 ** 6):
    hist = []
    for _ in range(n):
        th = float(ctl.thresholds()[0])
        s = env(th)
        act = int(round((1 - s) * px))
        ctl.observe([act], [px])
        hist.append((th, 1 - act / px))
    return hist


def test_bst_termination_bound():
    cfg = ControllerConfig(policy="bst")
    bound = math.ceil(math.log2(cfg.theta_max / cfg.theta_res)) + 1
    assert bound == 11
    rng = np.random.default_rng(0)
    for _ in range(200):
        ctl = Controller(cfg, 1)
        for k in range(1, 40):
            ctl.observe([int(rng.integers(0, 1001))], [1000])
            if ctl.frozen[0]:
                break
        assert ctl.frozen[0] and k <= bound
        assert 0.0 <= ctl.lo[0] <= ctl.theta[0] <= ctl.hi[0] <= cfg.theta_max


def test_bst_band_vs_grid_scan():
    cfg = ControllerConfig(policy="bst", T=0.9, eps=0.05)
    rng = np.random.default_rng(1)
    grid = np.linspace(0, 1, 20001)
    for _ in range(50):
        env = _env(rng)
        ctl = Controller(cfg, 1)
        _run(ctl, env, 12)
        assert ctl.frozen[0]
        s = env(float(np.float32(ctl.theta[0])))
        in_band = cfg.T - cfg.eps <= s <= cfg.T + cfg.eps
        # grid-scan oracle: a band solution exists and lies inside [lo, hi]
        sols = grid[[cfg.T - cfg.eps <= env(g) <= cfg.T + cfg.eps for g in grid]]
        assert sols.size > 0
        assert in_band or (ctl.hi[0] - ctl.lo[0] <= cfg.theta_res)
        assert np.any((sols >= ctl.lo[0] - 1e-9) & (sols <= ctl.hi[0] + 1e-9))


def test_ibst_reconverges_after_regime_switch():
    """Environment switches at observation 16; IBST (cycle 8) regains the
    band within one more cycle; a frozen BST stays out of band."""
    cfg_i = ControllerConfig(policy="ibst", cycle=8)
    cfg_b = ControllerConfig(policy="bst")
    e1 = lambda th: 0.5 + 0.5 * min(th / 0.2, 1.0)          # band near theta ~ 0.16
    e2 = lambda th: 0.3 + 0.7 * min(th / 0.9, 1.0) ** 2      # band near theta ~ 0.82
    for cfg in (cfg_i, cfg_b):
        ctl = Controller(cfg, 1)
        h1 = _run(ctl, e1, 16)
        assert 0.85 <= h1[-1][1] <= 0.95
        h2 = _run(ctl, e2, 24)
        tail = [s for _, s in h2[-8:]]
        ok = all(0.85 <= s <= 0.95 for s in tail)
        assert ok == (cfg.policy == "ibst"), (cfg.policy, tail)


def test_fixed_policy_inert():
    ctl = Controller(ControllerConfig(policy="fixed", theta_fixed=0.05), 3)
    ctl.observe([1, 2, 3], [10, 10, 10])
    assert np.all(ctl.thresholds() == np.float32(0.05))
