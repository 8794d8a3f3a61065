"""paper_2410_20790_b200 -- B200-native Diff Computation hot path of SparseTem
(arXiv 2410.20790).

The compute path is ``libsparsetem.so`` (hand-written sm_100a CUDA behind
the C ABI in ``include/sparsetem.h``); this package is a thin ctypes binding
with the same names (argument marshalling only).  There is no CPU fallback:
loading fails loudly when the library is missing.
"""
from .binding import (  # noqa: F401
    lib, load_library, StError, CapacityError, Encoder, ThresholdController, KIND, PRECISION,
)
