"""Memory accountant: SparseBatch vs vanilla (DeltaCNN-style) schedule.

TEST INFRASTRUCTURE, NOT PRODUCT CODE.

PAPER.md P:139: DeltaCNN caches the dense input and output of every
non-linear layer, "proportional to the number of non-linear layers";
P:152: SparseBatch "keeps only one buffer for Subtraction and one for
Accumulation".  Element counts per video chunk:

* SparseBatch persistent = |input| + sum |output taps|
  peak transient         = max over non-linear sites (|x_acc| + |y_acc|)
* vanilla persistent     = |input| + sum |output taps|
                           + sum over non-linear sites (|x_acc| + |y_acc|)
* pass count: SparseBatch 1, vanilla L (Fig. orchestration).
"""
from __future__ import annotations

from .core import shapes

_NONLINEAR = (1, 2, 3, 5)
_OUTPUT = 6


def account_memory(net, schedule: str, n_videos: int = 1, L: int = 1):
    shp = shapes(net)

    def ne(i):
        h, w, c = (net.in_h, net.in_w, net.in_c) if i < 0 else shp[i]
        return h * w * c

    inp = ne(-1)
    outs = sum(ne(i) for i, l in enumerate(net.layers) if l["kind"] == _OUTPUT)
    site = [ne(l["src"]) + ne(i) for i, l in enumerate(net.layers) if l["kind"] in _NONLINEAR]
    base = inp + outs
    if schedule == "sparsebatch":
        persistent = base
        transient = max(site) if site else 0
        passes = 1
    elif schedule == "vanilla":
        persistent = base + sum(site)
        transient = 0
        passes = L
    else:
        raise ValueError(schedule)
    return dict(persistent_values=persistent * n_videos, peak_transient_values=transient * n_videos,
                pass_count=passes, per_site=site)
