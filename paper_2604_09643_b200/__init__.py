"""PA-SFM differentiable acoustic radiation operator on B200 (arXiv 2604.09643).

The operator lives in libpa.so (hand-written CUDA for sm_100a behind the C ABI of
include/pa.h); `_pa` is its thin ctypes binding, `dist` the frame-sharding / NCCL plumbing,
`gen` the seeded synthetic-input generators.
"""
from ._pa import Context, PAError, load, plan_info  # noqa: F401

__all__ = ["Context", "PAError", "load"]
