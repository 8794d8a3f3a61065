"""Random small networks for property tests (SPEC S:572 recipe: 2-12 layers
mixing conv / relu / silu / maxpool / add / SE, plus depthwise)."""
from __future__ import annotations

import numpy as np

from workloads import Net, init_weights, infer_shapes, CONV


def random_net(seed, in_c=None, h=None, w=None, max_layers=10, allow_silu=True, allow_se=True,
               allow_dw=True):
    rng = np.random.default_rng(seed)
    in_c = in_c or int(rng.integers(1, 4))
    h = h or int(rng.integers(6, 13))
    w = w or int(rng.integers(6, 13))
    n = Net(in_c, h, w, f"rand{seed}")
    cur = -1
    hist = [(-1, (h, w, in_c))]
    n_layers = int(rng.integers(2, max_layers + 1))
    while len(n.layers) < n_layers:
        shp = infer_shapes(n)
        ch, cw, cc = (h, w, in_c) if cur < 0 else shp[cur]
        r = rng.random()
        if r < 0.35:
            k = int(rng.choice([1, 2, 3]))
            s = int(rng.choice([1, 1, 2])) if min(ch, cw) > 4 else 1
            p = int(rng.integers(0, k // 2 + 1))
            if (ch + 2 * p - k) // s + 1 < 2 or (cw + 2 * p - k) // s + 1 < 2:
                continue
            co = int(rng.integers(1, 9))
            cur = n.conv(cur, co, k, s, p)
        elif r < 0.45 and allow_dw and cc > 1:
            k = int(rng.choice([3, 5])) if min(ch, cw) >= 5 else 3
            cur = n.conv(cur, cc, k, 1, k // 2, groups=cc)
        elif r < 0.62:
            cur = n.relu(cur)
        elif r < 0.70 and allow_silu:
            cur = n.silu(cur)
        elif r < 0.80:
            k = int(rng.choice([2, 3]))
            s = int(rng.choice([1, 2]))
            p = int(rng.integers(0, k // 2 + 1))
            if (ch + 2 * p - k) // s + 1 < 2 or (cw + 2 * p - k) // s + 1 < 2:
                continue
            cur = n.maxpool(cur, k, s, p)
        elif r < 0.90:
            cands = [i for i, s in hist if s == (ch, cw, cc) and i != cur]
            if not cands:
                continue
            cur = n.add(cur, int(rng.choice(cands)))
        elif allow_se:
            cur = n.se(cur, max(1, cc // 2))
        else:
            continue
        hist.append((cur, infer_shapes(n)[cur]))
    n.output(cur)
    init_weights(n, seed + 17)
    return n


def random_frames(seed, L, h, w, c, p_change=0.3, scale=0.3):
    """Float frames with sparse changes (a fraction of pixels move each frame)."""
    rng = np.random.default_rng(seed)
    f = np.empty((L, h, w, c), np.float32)
    f[0] = rng.random((h, w, c))
    for t in range(1, L):
        ch = rng.random((h, w, 1)) < p_change
        f[t] = np.where(ch, f[t - 1] + scale * rng.standard_normal((h, w, c)), f[t - 1])
    return f.astype(np.float32)
