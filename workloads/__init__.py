"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no subtraction, truncation,
convolution, activation or accumulation).  It only produces:

* layer-spec lists (network topologies) -- ``workloads.models``;
* seeded random weights                  -- ``workloads.models.init_weights``;
* seeded uint8 synthetic video           -- ``workloads.video``;
* the five BASELINE.json configurations  -- ``workloads.configs``.

Both ``oracle/`` and ``paper_2410_20790_b200/`` may import it; neither may
import the other.
"""
from .models import (  # noqa: F401
    CONV, RELU, SILU, MAXPOOL, ADD, SE, OUTPUT, KIND_NAMES, NONLINEAR,
    Net, infer_shapes, init_weights, site_layers,
)
from .video import gen_video, gen_chunk, to_float  # noqa: F401
from .configs import CONFIGS, get_config  # noqa: F401
