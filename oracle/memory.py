"""Memory accountant: SparseBatch vs vanilla (DeltaCNN-style) schedule.

TEST INFRASTRUCTURE, NOT PRODUCT CODE.

PAPER.md P:139: DeltaCNN caches the dense input and output of every
non-linear layer, "proportional to the number of non-linear layers";
P:152: SparseBatch processes a batch layer by layer ("N" order) and "keeps
only one buffer for Subtraction and one for Accumulation".  Element counts
per video chunk of L frames (SPEC S:369-379 for the cache model):

SparseBatch (one pass over all L-1 diff frames, layer by layer)
* persistent = |input| (the Subtraction buffer: the reference frame)
             + L * sum |output taps| (the Accumulation buffer holds every
               frame's output until the step ends)
* a layer's tensor = its dense reference activation (|x0|, the state every
  site starts from) + its delta rows (rows * C: every diff frame's
  active pixels, as the batch is processed layer by layer); the input
  site's tensor is its delta rows.  A tensor is live from the step of its
  producer to the step of its last consumer (OUTPUT taps alias their
  source).  peak transient = max over steps of the live tensors' sum.
  ``rows`` (layer -> active pixel-frames over the step, -1 = input site,
  e.g. from an oracle run's masks) gives the data-dependent part; without
  it every tensor is counted at the all-active bound (L-1) * N.

vanilla (DeltaCNN: one pass through all layers per frame index, caches kept)
* persistent = |input| + sum |output taps|
             + sum over non-linear sites (|x_acc| + |y_acc|) (dense caches)
* transient  = the same liveness rule over one frame's dense tensors.
* pass count: SparseBatch 1, vanilla L (reference + L - 1 diff passes;
  P:168, Fig. orchestration).
"""
from __future__ import annotations

from .core import shapes

_NONLINEAR = (1, 2, 3, 5)
_OUTPUT = 6


def rows_from_run(run, net):
    """Active pixel-frames per layer (and -1: the input site) of an oracle
    run_chunk result with masks."""
    rows = {-1: int(run["in_mask"].sum())}
    for i in range(len(net.layers)):
        if i in run["masks"]:
            rows[i] = int(run["masks"][i].sum())
    return rows


def account_memory(net, schedule: str, n_videos: int = 1, L: int = 1, rows=None):
    shp = shapes(net)
    layers = net.layers
    n = len(layers)

    def hwc(i):
        return (net.in_h, net.in_w, net.in_c) if i < 0 else shp[i]

    def ne(i):
        h, w, c = hwc(i)
        return h * w * c

    def owner(i):   # OUTPUT taps alias their source tensor
        while i >= 0 and layers[i]["kind"] == _OUTPUT:
            i = layers[i]["src"]
        return i

    inp = ne(-1)
    taps = [i for i, l in enumerate(layers) if l["kind"] == _OUTPUT]
    outs = sum(ne(i) for i in taps)
    site = [ne(l["src"]) + ne(i) for i, l in enumerate(layers) if l["kind"] in _NONLINEAR]
    # last consumer step of every tensor (step of layer i = i + 1, input = 0)
    last = {-1: 0}
    for i, l in enumerate(layers):
        last.setdefault(i, i + 1)
        for s in (l["src"], l.get("src2", -1) if l["kind"] == 4 else -2):
            if s >= -1:
                o = owner(s)
                last[o] = max(last.get(o, 0), i + 1)
    F = max(L - 1, 1)

    def tensor(i, per_frame):
        h, w, c = hwc(i)
        if per_frame:                       # one frame's dense delta (DeltaCNN)
            r = h * w
        else:
            r = (rows or {}).get(i, F * h * w)
        dense = 0 if i < 0 else h * w * c   # the reference activation x0 / y0
        return dense + r * c

    def peak(per_frame):
        best = 0
        for t in range(n + 2):
            live = 0
            for i in [-1] + list(range(n)):
                if i >= 0 and layers[i]["kind"] == _OUTPUT:
                    continue
                first = 0 if i < 0 else i + 1
                if first <= t <= last.get(i, first):
                    live += tensor(i, per_frame)
            best = max(best, live)
        return best

    if schedule == "sparsebatch":
        persistent = inp + L * outs
        transient = peak(False)
        passes = 1
    elif schedule == "vanilla":
        persistent = inp + outs + sum(site)
        transient = peak(True)
        passes = L
    else:
        raise ValueError(schedule)
    return dict(persistent_values=persistent * n_videos, peak_transient_values=transient * n_videos,
                pass_count=passes, per_site=site)
