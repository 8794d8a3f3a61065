"""Build libsparsetem.so in-tree with nvcc for sm_100a (no JIT, no torch ext).

    python -m paper_2410_20790_b200.build [--force] [--checked]

Every .cu/.cpp under csrc/ is compiled to an object (in parallel) and linked
into paper_2410_20790_b200/libsparsetem.so.  Flags: -gencode
arch=compute_100a,code=sm_100a -lineinfo -O3 --fmad=false (no implicit
mul+add contraction: the FP32 path is bit-exact with the oracle's explicit
fmaf order; explicit fmaf() calls still emit FFMA).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# --checked: -DST_BOUNDS_CHECK (row-index asserts, csrc/common.cuh ST_CHECK) into
# libsparsetem_checked.so (load it with ST_LIB=<path>); objects kept apart
CHECKED = "--checked" in sys.argv or os.environ.get("ST_BUILD_CHECKED") == "1"
OBJ = os.path.join(ROOT, "build", "obj_checked" if CHECKED else "obj")
LIB = os.path.join(HERE, "libsparsetem_checked.so" if CHECKED else "libsparsetem.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC,-O3",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC, "--expt-relaxed-constexpr"] + \
    (["-DST_BOUNDS_CHECK"] if CHECKED else [])


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(ROOT, "include", "sparsetem.h")])


def _compile(src, force):
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    newest_dep = max([os.path.getmtime(src)] + [os.path.getmtime(d) for d in _deps()])
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj, None
    cmd = [NVCC] + ARCH + COMMON + ["-c", src, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC] + COMMON + ["-x", "cu", "-c", src, "-o", obj] + ARCH
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return obj, f"{' '.join(cmd)}\n{r.stdout}\n{r.stderr}"
    return obj, (r.stderr.strip() or None) and ("warn:" + r.stderr)


def build(force=False, verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, force), srcs))
    errs = [e for _, e in results if e and not e.startswith("warn:")]
    if errs:
        raise RuntimeError("nvcc failed:\n" + "\n".join(errs))
    if verbose:
        for _, e in results:
            if e:
                print(e)
    objs = [o for o, _ in results]
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + ["-lcudart", "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
