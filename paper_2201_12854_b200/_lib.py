"""ctypes binding of libmca_b200.so (the C ABI in include/mca/mca_cuda.h).

This module is the only place the Python side touches the library. It fails
loudly when the library is missing: there is no CPU fallback for any stage of
the MCA forward.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libmca_b200.so")
CSRC = os.path.join(_PKG, "csrc")

# mca_status
MCA_OK, MCA_ERR_SHAPE, MCA_ERR_DOMAIN, MCA_ERR_DEGENERATE, MCA_ERR_CONFIG = 0, 1, 2, 3, 4
MCA_ERR_CUDA, MCA_ERR_ALLOC, MCA_ERR_UNSUPPORTED, MCA_ERR_NULL = 5, 6, 7, 8
# mca_dtype / mca_mode
MCA_F32, MCA_BF16 = 0, 1
MCA_MODE_REGULAR, MCA_MODE_APPROX = 0, 1


class McaConfigC(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_double), ("scale", ctypes.c_double), ("min_samples", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("certify", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class McaFlopsC(ctypes.Structure):
    _fields_ = [("exact_encoding", ctypes.c_uint64), ("approx_encoding", ctypes.c_uint64),
                ("aggregation", ctypes.c_uint64), ("samples", ctypes.c_uint64), ("exact_tokens", ctypes.c_uint64),
                ("reduction_factor", ctypes.c_double), ("total_reduction", ctypes.c_double),
                ("certified", ctypes.c_uint64)]


class McaDebugC(ctypes.Structure):
    _fields_ = [("cmax_out", ctypes.c_void_p), ("lse_out", ctypes.c_void_p), ("h_out", ctypes.c_void_p),
                ("draws_out", ctypes.c_void_p), ("draws_stride", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("cmax_override", ctypes.c_void_p), ("budgets_override", ctypes.c_void_p),
                ("exact_override", ctypes.c_void_p), ("q_out", ctypes.c_void_p), ("k_out", ctypes.c_void_p)]


# Every symbol declared in include/mca/mca_cuda.h (tests/test_capi.py checks both directions).
EXPORTS = (
    "mca_prepare_weights", "mca_weights_free", "mca_weights_export", "mca_set_projections", "mca_reserve",
    "mca_forward", "mca_forward_ex", "mca_forward_attn",
    "mca_regular_forward", "mca_stage_budgets", "mca_set_timing", "mca_last_stage_ms", "mca_last_launch_count",
    "mca_device_alloc", "mca_device_free", "mca_copy", "mca_stream_sync", "mca_last_error", "mca_version",
)


def build(verbose: bool = False) -> str:
    """Compile the sm_100a library in-tree (nvcc cross-compiles without a GPU)."""
    cmd = ["make", "-C", CSRC]
    if not verbose:
        cmd.append("-s")
    subprocess.run(cmd, check=True)
    return LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the MCA forward has no CPU path)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u32, u64, d = (ctypes.c_void_p, ctypes.c_int, ctypes.c_long, ctypes.c_uint32, ctypes.c_uint64,
                                 ctypes.c_double)
    L.mca_last_error.restype = ctypes.c_char_p
    L.mca_version.restype = ctypes.c_char_p
    L.mca_prepare_weights.argtypes = [vp, i32, i32, i32, i32, vp, ctypes.POINTER(vp)]
    L.mca_weights_free.argtypes = [vp]
    L.mca_weights_free.restype = None
    L.mca_weights_export.argtypes = [vp, vp, vp]
    L.mca_set_projections.argtypes = [vp, vp, vp, vp]
    L.mca_reserve.argtypes = [vp, i64, vp]
    L.mca_forward.argtypes = [vp, vp, vp, vp, i32, i32, i32, i64, u32, ctypes.POINTER(McaConfigC), u64, vp, vp, vp,
                              ctypes.POINTER(McaFlopsC), vp]
    L.mca_forward_ex.argtypes = L.mca_forward.argtypes[:-1] + [ctypes.POINTER(McaDebugC), vp]
    L.mca_forward_attn.argtypes = [vp, vp, vp, i32, i32, i32, i64, u32, ctypes.POINTER(McaConfigC), u64, vp, vp, vp,
                                   ctypes.POINTER(McaFlopsC), vp]
    L.mca_regular_forward.argtypes = [vp, vp, vp, vp, i32, i32, i32, d, vp, vp]
    L.mca_stage_budgets.argtypes = [vp, i64, i32, i32, ctypes.POINTER(McaConfigC), vp, vp, vp]
    L.mca_set_timing.argtypes = [vp, i32]
    L.mca_last_stage_ms.argtypes = [vp, ctypes.POINTER(ctypes.c_float), i32]
    L.mca_last_stage_ms.restype = i32
    L.mca_last_launch_count.argtypes = [vp]
    L.mca_last_launch_count.restype = i32
    L.mca_device_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(vp)]
    L.mca_device_free.argtypes = [vp]
    L.mca_device_free.restype = None
    L.mca_copy.argtypes = [vp, vp, ctypes.c_size_t, i32]
    L.mca_stream_sync.argtypes = [vp]
    for name in ("mca_prepare_weights", "mca_weights_export", "mca_reserve", "mca_forward", "mca_forward_ex",
                 "mca_forward_attn", "mca_regular_forward", "mca_stage_budgets", "mca_set_timing", "mca_device_alloc",
                 "mca_copy", "mca_stream_sync"):
        getattr(L, name).restype = i32
    _lib = L
    return L
