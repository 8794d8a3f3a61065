"""ctypes binding of libsparsetem.so (include/sparsetem.h) -- marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; torch is
used for device memory, streams and process groups.  No CPU fallback: if the
library is missing, ``load_library`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ST_LIB: another in-tree build of the same library (the checked build,
# libsparsetem_checked.so) -- never a fallback
LIB_PATH = os.environ.get("ST_LIB") or os.path.join(HERE, "libsparsetem.so")

KIND = dict(conv=0, relu=1, silu=2, maxpool=3, add=4, se=5, output=6)
PRECISION = dict(fp32=0, bf16=1)
STATUS = {0: "ST_OK", 1: "ST_ERR_ARG", 2: "ST_ERR_SHAPE", 3: "ST_ERR_STATE", 4: "ST_ERR_UNSUPPORTED",
          5: "ST_ERR_OOM", 6: "ST_ERR_CUDA", 7: "ST_ERR_INTERNAL", 8: "ST_ERR_CAPACITY"}
ST_ERR_CAPACITY = 8


class StError(RuntimeError):
    def __init__(self, fn, status, msg=""):
        self.status = status
        super().__init__(f"{fn} failed: {STATUS.get(status, status)} {msg}".strip())


class CapacityError(StError):
    """The last step needed more delta rows than a tensor's capacity
    (ST_ERR_CAPACITY): its results are invalid; fit_capacity() and re-issue."""


class st_layer_spec(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("kind", "src", "src2", "c_out", "groups", "k_h", "k_w", "s_h", "s_w",
                                         "p_h", "p_w", "se_hidden")] + \
               [(n, C.POINTER(C.c_float)) for n in ("w", "b", "w2", "b2")]


class st_encoder_config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("in_c", "in_h", "in_w", "max_chunks", "max_frames", "precision",
                                         "device", "debug_retain", "streaming")] + [("row_frac", C.c_float)]


class st_ctl_config(C.Structure):
    _fields_ = [("policy", C.c_int32), ("T", C.c_float), ("eps", C.c_float), ("theta_max", C.c_float),
                ("theta_res", C.c_float), ("theta_fixed", C.c_float), ("cycle", C.c_int32)]


# name -> (restype, argtypes); the full exported surface of sparsetem.h
P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
SIGNATURES = {
    "st_encoder_create": (I32, [P, P, I32, P]),
    "st_encoder_destroy": (None, [P]),
    "st_encoder_num_sites": (I32, [P]),
    "st_layer_shape": (I32, [P, I32, P]),
    "st_encode_reference": (I32, [P, P, I32, I64, P]),
    "st_encode_diff": (I32, [P, P, I32, I64, P, P]),
    "st_encode_reference_u8": (I32, [P, P, I32, I64, P]),
    "st_encode_diff_u8": (I32, [P, P, I32, I64, P, P]),
    "st_get_sparsity": (I32, [P, P, P, P]),
    "st_copy_site_counts": (I32, [P, P, P]),
    "st_get_layer_counts": (I32, [P, P, P, P]),
    "st_get_output": (I32, [P, I32, I32, I32, P, P]),
    "st_debug_get_mask": (I32, [P, I32, I32, I32, P]),
    "st_debug_get_rows": (I32, [P, I32, I32, I32, P, P, P]),
    "st_debug_get_dense0": (I32, [P, I32, I32, P]),
    "st_debug_export_chunk": (I32, [P, I32]),
    "st_debug_get_words": (I32, [P, I32, P]),
    "st_memory_report": (I32, [P, P, P, P]),
    "st_device_bytes": (I32, [P, P]),
    "st_step_status": (I32, [P]),
    "st_get_capacity": (I32, [P, P, P]),
    "st_encoder_fit_capacity": (I32, [P, C.c_double]),
    "st_set_profiling": (I32, [P, I32]),
    "st_num_kernel_classes": (I32, []),
    "st_kernel_class_name": (C.c_char_p, [I32]),
    "st_get_kernel_times": (I32, [P, P, P, P, P, I32]),
    "st_last_launch_count": (I32, [P]),
    "st_status_string": (C.c_char_p, [I32]),
    "st_last_error": (C.c_char_p, [P]),
    "st_controller_create": (I32, [P, I32, P]),
    "st_controller_observe": (I32, [P, P, P]),
    "st_controller_thresholds": (I32, [P, P]),
    "st_controller_state": (I32, [P, P, P, P, P]),
    "st_controller_destroy": (None, [P]),
}

_lib = None


def load_library(path=LIB_PATH):
    """Load libsparsetem.so.  Raises loudly if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built: run `python -m paper_2410_20790_b200.build` "
                               "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def lib():
    return load_library()


def _np_ptr(a):
    return a.ctypes.data


class _CudaView:
    """Zero-copy torch view of a borrowed device pointer."""

    def __init__(self, ptr, shape, dtype="<f4"):
        self.__cuda_array_interface__ = dict(shape=tuple(shape), typestr=dtype, data=(int(ptr), False),
                                             version=3, strides=None)


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(int(stream.cuda_stream))


class Encoder:
    """One encoder = one network on one device (st_encoder_create)."""

    def __init__(self, net, max_chunks, max_frames, precision="fp32", device=0, debug_retain=False,
                 streaming=False, row_frac=0.0):
        L = lib()
        self.net = net
        self.n_layers = len(net.layers)
        arr = (st_layer_spec * self.n_layers)()
        keep = []
        for i, l in enumerate(net.layers):
            s = arr[i]
            for f in ("kind", "src", "src2", "c_out", "groups", "k_h", "k_w", "s_h", "s_w", "p_h", "p_w", "se_hidden"):
                setattr(s, f, int(l[f]))
            for f in ("w", "b", "w2", "b2"):
                a = l.get(f)
                if a is not None:
                    a = np.ascontiguousarray(a, np.float32)
                    keep.append(a)
                    setattr(s, f, a.ctypes.data_as(C.POINTER(C.c_float)))
        cfg = st_encoder_config(net.in_c, net.in_h, net.in_w, max_chunks, max_frames, PRECISION[precision],
                                device, int(bool(debug_retain)), int(bool(streaming)), float(row_frac))
        h = C.c_void_p()
        r = L.st_encoder_create(C.byref(cfg), C.cast(arr, C.c_void_p), self.n_layers, C.byref(h))
        if r != 0:
            raise StError("st_encoder_create", r)
        self.h = h
        self.max_chunks, self.max_frames = max_chunks, max_frames
        self.device = device
        self.n_sites = L.st_encoder_num_sites(h)
        self.taps = [i for i, l in enumerate(net.layers) if l["kind"] == KIND["output"]]
        self.n_chunks = 0
        self.n_diff = -1

    # -- helpers
    def _check(self, fn, r):
        if r != 0:
            cls = CapacityError if r == ST_ERR_CAPACITY else StError
            raise cls(fn, r, lib().st_last_error(self.h).decode(errors="replace"))

    def close(self):
        if getattr(self, "h", None):
            lib().st_encoder_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def layer_shape(self, layer):
        hwc = np.zeros(3, np.int32)
        self._check("st_layer_shape", lib().st_layer_shape(self.h, layer, _np_ptr(hwc)))
        return tuple(int(v) for v in hwc)

    # -- the hot path
    def encode_reference(self, ref, stream=None):
        """ref: torch float32 or uint8 cuda [B][H][W][C] (chunk dim may be
        strided); uint8 frames mean v / 255 (reading R20)."""
        import torch
        u8 = ref.dtype == torch.uint8
        assert (u8 or ref.dtype == torch.float32) and ref.is_cuda
        per = self.net.in_h * self.net.in_w * self.net.in_c
        assert ref[0].is_contiguous(), "frame must be contiguous NHWC"
        stride = ref.stride(0) if ref.shape[0] > 1 else per
        fn = "st_encode_reference_u8" if u8 else "st_encode_reference"
        self._check(fn, getattr(lib(), fn)(
            self.h, C.c_void_p(ref.data_ptr()), ref.shape[0], stride, _stream_handle(stream)))
        self.n_chunks = ref.shape[0]

    def encode_diff(self, frames, thresholds, stream=None):
        """frames: torch float32 or uint8 cuda [B][n_diff][H][W][C] (chunk dim
        may be strided), or None for n_diff = 0."""
        import torch
        th = np.ascontiguousarray(np.broadcast_to(np.asarray(thresholds, np.float32), (self.n_sites,)))
        n_diff = 0 if frames is None else frames.shape[1]
        ptr, stride, u8 = None, 0, False
        if n_diff:
            u8 = frames.dtype == torch.uint8
            assert frames.is_cuda and (u8 or frames.dtype == torch.float32)
            assert frames[0].is_contiguous(), "frames of a chunk must be contiguous"
            ptr = frames.data_ptr()
            stride = frames.stride(0) if frames.shape[0] > 1 else 0
        fn = "st_encode_diff_u8" if u8 else "st_encode_diff"
        self._check(fn, getattr(lib(), fn)(
            self.h, C.c_void_p(ptr), n_diff, stride, _np_ptr(th), _stream_handle(stream)))
        self.n_diff = n_diff

    def get_sparsity(self):
        F = max(self.n_diff, 0)
        act = np.zeros((self.n_chunks, self.n_sites, max(F, 1)), np.int64)
        sa = np.zeros(self.n_sites, np.int64)
        sp = np.zeros(self.n_sites, np.int64)
        self._check("st_get_sparsity", lib().st_get_sparsity(self.h, _np_ptr(act), _np_ptr(sa), _np_ptr(sp)))
        return act[:, :, :F], sa, sp

    def copy_site_counts(self, dst, stream=None):
        self._check("st_copy_site_counts", lib().st_copy_site_counts(self.h, C.c_void_p(dst.data_ptr()),
                                                                     _stream_handle(stream)))

    def layer_counts(self):
        a = np.zeros((3, self.n_layers), np.int64)
        self._check("st_get_layer_counts", lib().st_get_layer_counts(self.h, _np_ptr(a[0]), _np_ptr(a[1]),
                                                                     _np_ptr(a[2])))
        return dict(rows_in=a[0], rows_out=a[1], touched=a[2])

    def output_ptr(self, tap, chunk, frame):
        p = C.c_void_p()
        hwc = np.zeros(3, np.int32)
        self._check("st_get_output", lib().st_get_output(self.h, tap, chunk, frame, C.byref(p), _np_ptr(hwc)))
        return p.value, tuple(int(v) for v in hwc)

    def get_output(self, tap, chunk, frame):
        """Borrowed zero-copy torch view [H][W][C] (valid until the next encode)."""
        import torch
        ptr, hwc = self.output_ptr(tap, chunk, frame)
        return torch.as_tensor(_CudaView(ptr, hwc), device=f"cuda:{self.device}")

    def outputs(self, tap):
        """Borrowed view of all frames of all chunks: [B][L][H][W][C]."""
        import torch
        ptr, hwc = self.output_ptr(tap, 0, 0)
        shape = (self.n_chunks, self.n_diff + 1) + hwc
        return torch.as_tensor(_CudaView(ptr, shape), device=f"cuda:{self.device}")

    # -- debug
    def debug_mask(self, layer, chunk, frame):
        h, w, _ = self.layer_shape(layer)
        words = np.zeros((h * w + 31) // 32, np.uint32)
        self._check("st_debug_get_mask", lib().st_debug_get_mask(self.h, layer, chunk, frame, _np_ptr(words)))
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[: h * w]
        return bits.reshape(h, w).astype(np.uint8)

    def debug_rows(self, layer, chunk, frame):
        h, w, c = self.layer_shape(layer)
        n = C.c_int64()
        self._check("st_debug_get_rows", lib().st_debug_get_rows(self.h, layer, chunk, frame, None, None,
                                                                 C.byref(n)))
        idx = np.zeros(max(n.value, 1), np.int32)
        rows = np.zeros((max(n.value, 1), c), np.float32)
        self._check("st_debug_get_rows", lib().st_debug_get_rows(self.h, layer, chunk, frame, _np_ptr(idx),
                                                                 _np_ptr(rows), C.byref(n)))
        return idx[: n.value], rows[: n.value]

    def debug_dense0(self, layer, chunk):
        h, w, c = self.layer_shape(layer)
        out = np.zeros((h, w, c), np.float32)
        self._check("st_debug_get_dense0", lib().st_debug_get_dense0(self.h, layer, chunk, _np_ptr(out)))
        return out

    def export_chunk(self, chunk):
        """Mask export of one chunk from the production step (st_debug_export_chunk)."""
        self._check("st_debug_export_chunk", lib().st_debug_export_chunk(self.h, int(chunk)))

    def exported_masks(self, layer):
        """uint8 [n_diff][H][W] masks of `layer` for the exported chunk."""
        h, w, _ = self.layer_shape(layer)
        words = np.zeros(h * w, np.uint32)
        self._check("st_debug_get_words", lib().st_debug_get_words(self.h, layer, _np_ptr(words)))
        F = self.n_diff
        bits = (words[None, :] >> np.arange(F, dtype=np.uint32)[:, None]) & 1
        return bits.reshape(F, h, w).astype(np.uint8)

    def memory_report(self):
        v = np.zeros(3, np.int64)
        self._check("st_memory_report", lib().st_memory_report(self.h, _np_ptr(v[0:]), _np_ptr(v[1:]),
                                                               _np_ptr(v[2:])))
        return dict(persistent_bytes=int(v[0]), peak_transient_bytes=int(v[1]), arena_bytes=int(v[2]))

    def device_bytes(self):
        v = np.zeros(1, np.int64)
        self._check("st_device_bytes", lib().st_device_bytes(self.h, _np_ptr(v)))
        return int(v[0])

    # -- row capacity (a9)
    def step_ok(self):
        """False if the last step exceeded a row capacity (synchronizes)."""
        r = lib().st_step_status(self.h)
        if r == ST_ERR_CAPACITY:
            return False
        self._check("st_step_status", r)
        return True

    def capacity(self):
        """(rows_cap, rows_peak) per delta tensor: layers, then the input site (-1: no own rows)."""
        cap = np.zeros(self.n_layers + 1, np.int64)
        pk = np.zeros(self.n_layers + 1, np.int64)
        self._check("st_get_capacity", lib().st_get_capacity(self.h, _np_ptr(cap), _np_ptr(pk)))
        return cap, pk

    def fit_capacity(self, headroom=1.25):
        """Re-plan the arena from the measured row counts (x headroom)."""
        self._check("st_encoder_fit_capacity", lib().st_encoder_fit_capacity(self.h, C.c_double(headroom)))
        self.n_diff = -1

    # -- profiling
    def set_profiling(self, on):
        self._check("st_set_profiling", lib().st_set_profiling(self.h, int(bool(on))))

    def kernel_times(self, reset=True):
        L = lib()
        n = L.st_num_kernel_classes()
        ms = np.zeros(n)
        cnt = np.zeros(n, np.int64)
        by = np.zeros(n)
        fl = np.zeros(n)
        self._check("st_get_kernel_times", L.st_get_kernel_times(self.h, _np_ptr(ms), _np_ptr(cnt), _np_ptr(by),
                                                                 _np_ptr(fl), int(bool(reset))))
        return {L.st_kernel_class_name(i).decode(): dict(ms=float(ms[i]), launches=int(cnt[i]),
                                                         bytes=float(by[i]), flops=float(fl[i]))
                for i in range(n)}

    def last_launch_count(self):
        return int(lib().st_last_launch_count(self.h))


class ThresholdController:
    """BST / IBST controller (st_controller_*)."""
    POLICY = dict(fixed=0, bst=1, ibst=2)

    def __init__(self, n_sites, policy="ibst", T=0.9, eps=0.05, theta_max=1.0, theta_res=1e-3, theta_fixed=0.05,
                 cycle=8):
        cfg = st_ctl_config(self.POLICY[policy], T, eps, theta_max, theta_res, theta_fixed, cycle)
        h = C.c_void_p()
        r = lib().st_controller_create(C.byref(cfg), n_sites, C.byref(h))
        if r != 0:
            raise StError("st_controller_create", r)
        self.h = h
        self.n = n_sites

    def observe(self, site_active, site_pixels):
        a = np.ascontiguousarray(site_active, np.int64)
        p = np.ascontiguousarray(site_pixels, np.int64)
        r = lib().st_controller_observe(self.h, _np_ptr(a), _np_ptr(p))
        if r != 0:
            raise StError("st_controller_observe", r)

    def thresholds(self):
        out = np.zeros(self.n, np.float32)
        lib().st_controller_thresholds(self.h, _np_ptr(out))
        return out

    def state(self):
        th, lo, hi = np.zeros(self.n), np.zeros(self.n), np.zeros(self.n)
        fr = np.zeros(self.n, np.int32)
        lib().st_controller_state(self.h, _np_ptr(th), _np_ptr(lo), _np_ptr(hi), _np_ptr(fr))
        return th, lo, hi, fr

    def __del__(self):
        try:
            if self.h:
                lib().st_controller_destroy(self.h)
                self.h = None
        except Exception:
            pass
