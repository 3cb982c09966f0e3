"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This package holds NO arithmetic of the ContiguousKV method (no softmax, no
scoring, no selection, no attention): only random-number generation and
rounding of the generated values to the dtype the GPU path consumes.  Both the
oracle (``oracle/``) and the CUDA path receive exactly the same arrays.
"""
from .workload import (  # noqa: F401
    CONFIGS,
    ShapeConfig,
    bf16_round,
    bf16_bits,
    make_prefix,
    make_request,
)
