"""CPU oracle of SparseTem's Diff Computation (arXiv 2410.20790).

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with
``paper_2410_20790_b200`` and never imports it; the CUDA path never imports
this package.

* ``sparsetem_oracle.c`` -- dense forward (Eq.1) and the diff path
  (Subtraction, Eq.2 sparse conv, Eq.3 non-linear correction, truncation,
  Accumulation) in fp32 with a fixed fma order; see its header.
* ``controller.py``      -- BST / IBST threshold controller.
* ``memory.py``          -- SparseBatch vs vanilla memory accountant
  (SPEC S:386-394).

Parity status per function is listed in DESIGN.md ("Oracle pins").
"""
from .core import (  # noqa: F401
    build, lib_path, shapes, num_sites, dense_forward, run_chunk, dilate,
)
from .controller import Controller, ControllerConfig  # noqa: F401
from .memory import account_memory, rows_from_run  # noqa: F401
