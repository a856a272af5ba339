"""paper_2201_12854_b200 — Monte-Carlo Attention (arXiv 2201.12854) forward on
NVIDIA B200 (sm_100a).

The compute lives in ``lib/libmca_b200.so`` (hand-written CUDA, C ABI in
``include/mca/mca_cuda.h``); this package is the thin Python host mirror of
the reference's operator interface (see ``api``). Importing it does not load
CUDA; the first call that needs the library loads it and raises if it is
missing — there is no CPU fallback.
"""
from ._lib import LIB_PATH, build  # noqa: F401
from .api import (  # noqa: F401
    AttentionOutput,
    AttentionWeights,
    ConfigError,
    CudaError,
    DegenerateError,
    DomainError,
    FlopsReport,
    McaConfig,
    McaError,
    ShapeError,
    UnsupportedError,
    forward_given_attention,
    mca_forward,
    multihead_forward,
    regular_forward,
    sample_budgets,
)

from .pipeline import HostPipeline  # noqa: F401,E402

__version__ = "0.1.0"
