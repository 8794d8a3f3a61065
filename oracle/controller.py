"""Online Truncation Threshold Adjustment: BST / IBST (oracle side).

TEST INFRASTRUCTURE, NOT PRODUCT CODE (the product controller is C++ inside
libsparsetem.so; the two share no code).

PAPER.md P:171-181 (§3.4): per-layer thresholds steer each non-linear layer's
sparsity into [T - eps, T + eps] by binary search (BST), re-run
every cycle (IBST).  The paper gives no constants or update rule;
this follows DESIGN.md readings R15/R16 (= SPEC S:442, S:464-467 with the
per-step cadence of R15):

* init: theta = theta_max/2, lo = 0, hi = theta_max, not frozen;
* observe(sparsity s), s = 1 - active/pixels over all diff frames of all
  chunks of one step (fp64):
    s > T + eps  -> hi = theta          (too sparse: threshold too high)
    s < T - eps  -> lo = theta
    in band, or hi - lo <= theta_res -> frozen
    otherwise theta = (lo + hi)/2
* IBST: after every ``cycle`` observations restart with lo = 0, hi = theta_max,
  frozen = False, theta kept as the first probe;
* theta is handed to kernels as fp32 (round-to-nearest).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ControllerConfig:
    policy: str = "ibst"       # fixed | bst | ibst
    T: float = 0.9
    eps: float = 0.05
    theta_max: float = 1.0
    theta_res: float = 1e-3
    theta_fixed: float = 0.05
    cycle: int = 8


class Controller:
    def __init__(self, cfg: ControllerConfig, n_sites: int):
        self.cfg = cfg
        self.n = n_sites
        if cfg.policy == "fixed":
            self.theta = [float(cfg.theta_fixed)] * n_sites
        else:
            self.theta = [cfg.theta_max / 2.0] * n_sites
        self.lo = [0.0] * n_sites
        self.hi = [float(cfg.theta_max)] * n_sites
        self.frozen = [False] * n_sites
        self.count = [0] * n_sites
        self.last = [float("nan")] * n_sites

    def observe(self, site_active, site_pixels):
        cfg = self.cfg
        for i in range(self.n):
            px = int(site_pixels[i])
            if px <= 0:
                continue
            s = 1.0 - float(int(site_active[i])) / float(px)
            if not (0.0 <= s <= 1.0):
                raise ValueError("sparsity outside [0,1]")
            self.last[i] = s
            if cfg.policy == "fixed":
                continue
            if not self.frozen[i]:
                if s > cfg.T + cfg.eps:
                    self.hi[i] = self.theta[i]
                elif s < cfg.T - cfg.eps:
                    self.lo[i] = self.theta[i]
                in_band = cfg.T - cfg.eps <= s <= cfg.T + cfg.eps
                if in_band or self.hi[i] - self.lo[i] <= cfg.theta_res:
                    self.frozen[i] = True
                else:
                    self.theta[i] = (self.lo[i] + self.hi[i]) / 2.0
            if cfg.policy == "ibst":
                self.count[i] += 1
                if self.count[i] >= cfg.cycle:
                    self.count[i] = 0
                    self.lo[i] = 0.0
                    self.hi[i] = float(cfg.theta_max)
                    self.frozen[i] = False

    def thresholds(self):
        return np.asarray(self.theta, np.float64).astype(np.float32)
