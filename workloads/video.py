"""Seeded synthetic video shaped like the paper's workloads.

The paper's inputs are UCF101 action clips and MOT16 street video
(PAPER.md P:217); its own characterisation of adjacent-frame differences is
"sparse true motion + many small differences from camera jitter and noise"
(P:106).  The generator reproduces exactly that structure:

* a static textured background (smooth value noise + hard-edged blocks);
* K moving rectangles/discs with integer positions, reflective bounds and a
  per-object speed (px per ``frames_per_px`` frames);
* sensor noise: every pixel-channel, with probability ``q``, gets an integer
  offset in [-amp, amp] \\ {0} (LSBs), independently per frame;
* optional global flicker (a hard case: every pixel changes).

Frames are uint8 ``[n_chunks][L][H][W][C]``; the float input of both the
oracle and the CUDA path is ``v / 255.0f`` (reading R20), converted once by
``to_float``.  Chunks are independent (each has its own reference frame,
P:113); chunk j of a config is seeded with ``seed + j``.
"""
from __future__ import annotations

import numpy as np


def _value_noise(rng, h, w, c, cell):  # float32 map
    gh, gw = h // cell + 2, w // cell + 2
    g = rng.uniform(40, 215, (gh, gw, c))
    ys = np.arange(h) / cell
    xs = np.arange(w) / cell
    y0 = ys.astype(int)
    x0 = xs.astype(int)
    fy = (ys - y0)[:, None, None]
    fx = (xs - x0)[None, :, None]
    a = g[y0][:, x0]
    b = g[y0][:, x0 + 1]
    cc = g[y0 + 1][:, x0]
    d = g[y0 + 1][:, x0 + 1]
    return (a * (1 - fy) * (1 - fx) + b * (1 - fy) * fx + cc * fy * (1 - fx) + d * fy * fx).astype(np.float32)


def _background(rng, h, w, c, n_blocks):
    bg = _value_noise(rng, h, w, c, max(4, min(h, w) // 8))
    for _ in range(n_blocks):  # hard edges
        bh = int(rng.integers(2, max(3, h // 4)))
        bw = int(rng.integers(2, max(3, w // 4)))
        y = int(rng.integers(0, max(1, h - bh)))
        x = int(rng.integers(0, max(1, w - bw)))
        bg[y:y + bh, x:x + bw] = rng.uniform(0, 255, c)
    return bg


def _reflect(p, lo, hi):
    """Reflective bounds for an integer coordinate trajectory."""
    span = hi - lo
    if span <= 0:
        return lo
    m = (p - lo) % (2 * span)
    return lo + (m if m <= span else 2 * span - m)


def gen_chunk(seed, L, h, w, c, n_objects=3, size=(8, 16), speed=(1, 1), frames_per_px=1,
              noise_q=0.05, noise_amp=1, flicker=0, n_blocks=6, text=False):
    """One chunk of L uint8 frames [L][h][w][c]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if text:
        base = _text_strip(rng, h, w + L + 8)
    else:
        base = _background(rng, h, w, c, n_blocks)
    objs = []
    for _ in range(n_objects):
        sz_y = int(rng.integers(size[0], size[1] + 1))
        sz_x = int(rng.integers(size[0], size[1] + 1))
        objs.append(dict(
            y=int(rng.integers(0, max(1, h - sz_y))), x=int(rng.integers(0, max(1, w - sz_x))),
            hy=sz_y, hx=sz_x,
            vy=int(rng.integers(-speed[1], speed[1] + 1)),
            vx=int(rng.choice([-1, 1]) * rng.integers(speed[0], speed[1] + 1)),
            disc=bool(rng.integers(0, 2)), col=rng.uniform(0, 255, c)))
    frames = np.empty((L, h, w, c), np.uint8)
    for t in range(L):
        steps = t // frames_per_px
        if text:
            img = base[:, steps:steps + w].copy()
            # blinking cursor (2 px wide bar) at a fixed column
            if (t // 4) % 2 == 0:
                cx = w - 12
                img[h // 4: 3 * h // 4, cx:cx + 2] = 20
        else:
            img = base.copy()
        for o in objs:
            py = _reflect(o["y"] + o["vy"] * steps, 0, h - o["hy"])
            px = _reflect(o["x"] + o["vx"] * steps, 0, w - o["hx"])
            box = img[py:py + o["hy"], px:px + o["hx"]]
            if o["disc"]:   # ellipse inscribed in the object's box
                yy = (np.arange(box.shape[0])[:, None] + 0.5 - o["hy"] / 2.0) / (o["hy"] / 2.0)
                xx = (np.arange(box.shape[1])[None, :] + 0.5 - o["hx"] / 2.0) / (o["hx"] / 2.0)
                box[yy * yy + xx * xx <= 1.0] = o["col"]
            else:
                box[...] = o["col"]
        if flicker:
            img = img + flicker * (1 if t % 2 else -1)
        if noise_q > 0:
            # one uniform draw per pixel-channel: u < q is a hit; u / q picks
            # the offset uniformly from {-amp..-1, 1..amp}
            u = rng.random((h, w, c), dtype=np.float32).ravel()
            hit = np.flatnonzero(u < np.float32(noise_q))
            k = np.minimum((u[hit] * np.float32(2 * noise_amp / noise_q)).astype(np.int32), 2 * noise_amp - 1)
            tab = np.array([(1 + j // 2) * (1 if j % 2 == 0 else -1) for j in range(2 * noise_amp)], np.float32)
            img = img.reshape(-1)
            img[hit] += tab[k]
            img = img.reshape(h, w, c)
        frames[t] = np.clip(np.rint(img), 0, 255).astype(np.uint8)
    return frames


def _text_strip(rng, h, w):
    """Grayscale text line: random glyphs of 2-3 px strokes on a light field."""
    img = np.full((h, w, 1), 225.0)
    x = 2
    top, bot = h // 4, 3 * h // 4
    while x < w - 10:
        gw = int(rng.integers(6, 11))
        sw = int(rng.integers(2, 4))
        ink = float(rng.uniform(10, 70))
        kind = int(rng.integers(0, 4))
        if kind in (0, 1, 3):  # vertical stems
            img[top:bot, x:x + sw] = ink
        if kind in (1, 3):
            img[top:bot, x + gw - sw:x + gw] = ink
        if kind in (0, 2, 3):  # horizontal bars
            yb = int(rng.integers(top, bot - sw))
            img[yb:yb + sw, x:x + gw] = ink
        if kind == 2:
            img[top:top + sw, x:x + gw] = ink
            img[bot - sw:bot, x:x + gw] = ink
        x += gw + int(rng.integers(2, 6))
    return img


def gen_video(n_chunks, L, h, w, c, seed, **kw):
    """uint8 [n_chunks][L][h][w][c]; chunk j seeded with seed + j."""
    out = np.empty((n_chunks, L, h, w, c), np.uint8)
    for j in range(n_chunks):
        out[j] = gen_chunk(seed + j, L, h, w, c, **kw)
    return out


def to_float(u8):
    """float32 = v / 255.0f (reading R20); the one conversion both sides use."""
    return (u8.astype(np.float32) / np.float32(255.0)).astype(np.float32)
