"""ctypes wrapper of ``sparsetem_oracle.c`` (test infrastructure only)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sparsetem_oracle.c")
_LIB = os.path.join(_HERE, "libsparsetem_oracle.so")
_lib = None


class _Layer(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("kind", "src", "src2", "c_out", "groups", "k_h", "k_w", "s_h", "s_w",
                 "p_h", "p_w", "se_hidden")] + \
               [(n, C.POINTER(C.c_float)) for n in ("w", "b", "w2", "b2")]


class _Follow(C.Structure):
    _fields_ = [("masks", C.c_void_p), ("a_theta", C.c_float), ("a_rms", C.c_float), ("a_abs", C.c_float),
                ("stats", C.c_void_p)]


# Ambiguity bands of reading R23 (tau = a_theta*theta + a_rms*rms + a_abs)
TAU_FP32 = (1e-4, 0.0, 1e-5)
TAU_BF16 = (2e-2, 2e-2, 0.0)


def lib_path():
    return _LIB


def build(force=False):
    """Compile the oracle with gcc (fp32, -ffp-contract=off, explicit fmaf)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
               "-fno-fast-math", "-mfma", "-fopenmp", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        P = C.c_void_p
        lib.orc_shapes.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, P]
        lib.orc_num_sites.argtypes = [P, C.c_int]
        lib.orc_dense_forward.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, P, P]
        lib.orc_run_chunk.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P,
                                      C.c_int, P, P, P, P, P, P, P]
        lib.orc_run_chunk_follow.argtypes = lib.orc_run_chunk.argtypes + [P]
        lib.orc_dilate.argtypes = [P] + [C.c_int] * 10 + [P]
        lib.orc_set_precision.argtypes = [C.c_int]
        _lib = lib
    return _lib


def _fptr(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_float))


class _Spec:
    """Keeps the ctypes layer array and the numpy weight arrays alive."""

    def __init__(self, net):
        self.net = net
        n = len(net.layers)
        self.arr = (_Layer * max(n, 1))()
        self.keep = []
        for i, l in enumerate(net.layers):
            L = self.arr[i]
            for f in ("kind", "src", "src2", "c_out", "groups", "k_h", "k_w", "s_h", "s_w",
                      "p_h", "p_w", "se_hidden"):
                setattr(L, f, int(l[f]))
            for f in ("w", "b", "w2", "b2"):
                a = l.get(f)
                if a is not None:
                    a = np.ascontiguousarray(a, np.float32)
                    self.keep.append(a)
                    setattr(L, f, _fptr(a))
        self.n = n

    @property
    def ptr(self):
        return C.cast(self.arr, C.c_void_p)


def shapes(net):
    lib = _load()
    sp = _Spec(net)
    hwc = np.zeros((sp.n, 3), np.int32)
    r = lib.orc_shapes(sp.ptr, sp.n, net.in_h, net.in_w, net.in_c, hwc.ctypes.data)
    if r:
        raise ValueError(f"oracle: bad network spec (code {r})")
    return [tuple(int(v) for v in row) for row in hwc]


def num_sites(net):
    return int(_load().orc_num_sites(_Spec(net).ptr, len(net.layers)))


def dense_forward(net, frame, precision="fp32"):
    """Dense forward of one float32 frame [H][W][C]; list of per-layer outputs."""
    lib = _load()
    lib.orc_set_precision(1 if precision == "bf16" else 0)
    sp = _Spec(net)
    shp = shapes(net)
    x = np.ascontiguousarray(frame, np.float32)
    outs = [np.empty(s, np.float32) for s in shp]
    ptrs = (C.c_void_p * sp.n)(*[o.ctypes.data for o in outs])
    r = lib.orc_dense_forward(sp.ptr, sp.n, net.in_h, net.in_w, net.in_c, x.ctypes.data, ptrs)
    if r:
        raise ValueError(f"oracle dense_forward failed ({r})")
    return outs


def run_chunk(net, frames, thresholds, layer_outer=False, want_masks=True, want_deltas=False,
              want_dense0=False, mask_layers=None, delta_layers=None, precision="fp32",
              follow=None, tau=None):
    """Run one chunk (frames float32 [L][H][W][C]) through dense + diff.

    Returns dict with
      masks[l]  uint8 [L-1][H_l][W_l]     (layers in mask_layers, default all)
      deltas[l] float32 [L-1][H_l][W_l][C_l]
      dense0[l] float32 [H_l][W_l][C_l]
      taps[l]   float32 [L][H_l][W_l][C_l] for OUTPUT layers
      counts    int64 [n_sites][L-1]
      in_mask   uint8 [L-1][H][W]   input-site mask; in_delta float32 [L-1][H][W][C]

    follow: band-follow mode (O12, reading R23) -- {site layer: GPU emitted
    mask uint8 [L-1][H_l][W_l]}; inside the ambiguity band (tau, default the
    precision's R23 band) the oracle adopts the GPU's decision, elsewhere it
    keeps its own.  Adds follow_stats int64 [n_layers][4] = (decisions, in
    band, adopted, violations).
    """
    lib = _load()
    lib.orc_set_precision(1 if precision == "bf16" else 0)
    sp = _Spec(net)
    shp = shapes(net)
    fr = np.ascontiguousarray(frames, np.float32)
    Lf = fr.shape[0]
    F = Lf - 1
    ns = num_sites(net)
    th = np.ascontiguousarray(np.broadcast_to(np.asarray(thresholds, np.float32), (ns,)), np.float32)
    n = sp.n
    masks, deltas, dense0, taps = {}, {}, {}, {}
    mp, dp, zp, tp = (C.c_void_p * n)(), (C.c_void_p * n)(), (C.c_void_p * n)(), (C.c_void_p * n)()
    for i, s in enumerate(shp):
        if want_masks and (mask_layers is None or i in mask_layers):
            masks[i] = np.zeros((F, s[0], s[1]), np.uint8)
            mp[i] = masks[i].ctypes.data
        if want_deltas and (delta_layers is None or i in delta_layers):
            deltas[i] = np.zeros((F,) + s, np.float32)
            dp[i] = deltas[i].ctypes.data
        if want_dense0:
            dense0[i] = np.zeros(s, np.float32)
            zp[i] = dense0[i].ctypes.data
        if net.layers[i]["kind"] == 6:
            taps[i] = np.zeros((Lf,) + s, np.float32)
            tp[i] = taps[i].ctypes.data
    counts = np.zeros((ns, max(F, 1)), np.int64)
    in_mask = np.zeros((max(F, 1), net.in_h, net.in_w), np.uint8)
    in_delta = np.zeros((max(F, 1), net.in_h, net.in_w, net.in_c), np.float32) if want_deltas else None
    fl, fstats, keep = None, None, []
    if follow is not None:
        fp = (C.c_void_p * n)()
        for li, m in follow.items():
            m = np.ascontiguousarray(m, np.uint8).reshape(F, -1)
            assert m.shape[1] == shp[li][0] * shp[li][1], f"follow mask of layer {li} has the wrong size"
            keep.append(m)
            fp[li] = m.ctypes.data
        keep.append(fp)
        fstats = np.zeros((n, 4), np.int64)
        a = tau if tau is not None else (TAU_BF16 if precision == "bf16" else TAU_FP32)
        fl = _Follow(C.cast(fp, C.c_void_p), float(a[0]), float(a[1]), float(a[2]), fstats.ctypes.data)
    r = lib.orc_run_chunk_follow(sp.ptr, n, net.in_h, net.in_w, net.in_c, Lf, fr.ctypes.data,
                                 th.ctypes.data, int(bool(layer_outer)), mp, dp, zp, tp, counts.ctypes.data,
                                 in_mask.ctypes.data, None if in_delta is None else in_delta.ctypes.data,
                                 None if fl is None else C.addressof(fl))
    if r:
        raise ValueError(f"oracle run_chunk failed ({r})")
    out = dict(masks=masks, deltas=deltas, dense0=dense0, taps=taps, counts=counts[:, :F],
               in_mask=in_mask[:F], in_delta=None if in_delta is None else in_delta[:F])
    if fstats is not None:
        out["follow_stats"] = fstats
    return out


def dilate(mask, k, s, p, out_hw):
    """Mask dilation of a uint8 [H][W] mask; returns uint8 [Ho][Wo]."""
    lib = _load()
    m = np.ascontiguousarray(mask, np.uint8)
    kh, kw = k
    sh, sw = s
    ph, pw = p
    Ho, Wo = out_hw
    mo = np.zeros((Ho, Wo), np.uint8)
    lib.orc_dilate(m.ctypes.data, m.shape[0], m.shape[1], kh, kw, sh, sw, ph, pw, Ho, Wo, mo.ctypes.data)
    return mo
