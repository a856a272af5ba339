"""ctypes front end of the fp64 CPU oracle (oracle/*.cpp).

TEST INFRASTRUCTURE ONLY. Importable from tests/, __graft_entry__.smoke() and
bench.py's CPU legs (``cpu_baseline`` and ``--impl reference``), and there only
as the checker / the CPU baseline — never from the product package
``paper_2201_12854_b200``.

The functions mirror the SPEC op names and raise the SPEC
error classes as Python exceptions.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libmca_oracle.so")

_D = ctypes.POINTER(ctypes.c_double)
_I32 = ctypes.POINTER(ctypes.c_int32)
_I64 = ctypes.POINTER(ctypes.c_int64)
_U8 = ctypes.POINTER(ctypes.c_uint8)
_U32 = ctypes.POINTER(ctypes.c_uint32)
_U64 = ctypes.POINTER(ctypes.c_uint64)


class OracleShapeError(ValueError):
    pass


class OracleDomainError(ValueError):
    pass


class OracleDegenerateError(ValueError):
    pass


class OracleConfigError(ValueError):
    pass


_ERRORS = {1: OracleShapeError, 2: OracleDomainError, 3: OracleDegenerateError, 4: OracleConfigError}


def build(force: bool = False) -> str:
    """Compile the oracle with oracle/Makefile (g++, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.oracle_last_error.restype = ctypes.c_char_p
        _lib.oracle_bits53.restype = ctypes.c_uint64
        _lib.oracle_bits53.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]
        for name in ("oracle_verify_exactness", "oracle_verify_unbiased", "oracle_verify_lemma1",
                     "oracle_verify_scaling"):
            getattr(_lib, name).restype = ctypes.c_double
        _lib.oracle_verify_exactness.argtypes = [ctypes.c_int, ctypes.c_uint64]
        _lib.oracle_verify_unbiased.argtypes = [ctypes.c_long, ctypes.c_uint64]
        _lib.oracle_verify_lemma1.argtypes = [ctypes.c_int, ctypes.c_long, ctypes.c_uint64]
        _lib.oracle_verify_scaling.argtypes = [ctypes.c_long, ctypes.c_uint64]
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().oracle_last_error().decode()
        raise _ERRORS.get(rc, RuntimeError)(msg)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def set_threads(t: int) -> int:
    return lib().oracle_set_threads(ctypes.c_int(t))


# ------------------------------------------------------------------ tensor
def matmul(a, b) -> np.ndarray:
    a, b = _f64(np.atleast_2d(a)), _f64(np.atleast_2d(b))
    out = np.zeros((a.shape[0], b.shape[1]))
    _check(lib().oracle_matmul(_d(a), a.shape[0], a.shape[1], _d(b), b.shape[0], b.shape[1], _d(out)))
    return out


def matmul_nt(a, b) -> np.ndarray:
    a, b = _f64(np.atleast_2d(a)), _f64(np.atleast_2d(b))
    out = np.zeros((a.shape[0], b.shape[0]))
    _check(lib().oracle_matmul_nt(_d(a), a.shape[0], a.shape[1], _d(b), b.shape[0], b.shape[1], _d(out)))
    return out


def transpose(a) -> np.ndarray:
    a = _f64(np.atleast_2d(a))
    out = np.zeros((a.shape[1], a.shape[0]))
    _check(lib().oracle_transpose(_d(a), a.shape[0], a.shape[1], _d(out)))
    return out


def frobenius_norm(a) -> float:
    a = _f64(np.atleast_2d(a))
    out = ctypes.c_double()
    _check(lib().oracle_frobenius_norm(_d(a), a.shape[0], a.shape[1], ctypes.byref(out)))
    return out.value


def row_l2_norms(a) -> np.ndarray:
    a = _f64(np.atleast_2d(a))
    out = np.zeros(a.shape[0])
    _check(lib().oracle_row_l2_norms(_d(a), a.shape[0], a.shape[1], _d(out)))
    return out


def col_l2_norms(a) -> np.ndarray:
    a = _f64(np.atleast_2d(a))
    out = np.zeros(a.shape[1])
    _check(lib().oracle_col_l2_norms(_d(a), a.shape[0], a.shape[1], _d(out)))
    return out


def softmax_rows(a, scale: float) -> np.ndarray:
    a = _f64(np.atleast_2d(a))
    out = np.zeros_like(a)
    _check(lib().oracle_softmax_rows(_d(a), a.shape[0], a.shape[1], ctypes.c_double(scale), _d(out)))
    return out


def col_max(a, j: int) -> float:
    a = _f64(np.atleast_2d(a))
    out = ctypes.c_double()
    _check(lib().oracle_col_max(_d(a), a.shape[0], a.shape[1], ctypes.c_long(j), ctypes.byref(out)))
    return out.value


def matrix_check(rows: int, cols: int) -> None:
    _check(lib().oracle_matrix_check(rows, cols))


# ---------------------------------------------------------------- sampling
def philox4x32_10(ctr, key) -> tuple[int, int, int, int]:
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().oracle_philox4x32_10(c, k, o)
    return tuple(o)


def bits53(seed: int, stream: int, layer: int, k: int) -> int:
    return lib().oracle_bits53(seed, stream, layer, k)


@dataclass
class Distribution:
    probs: np.ndarray
    cdf: np.ndarray


def make_distribution(weights) -> Distribution:
    w = _f64(weights).ravel()
    p, c = np.zeros_like(w), np.zeros_like(w)
    _check(lib().oracle_make_distribution(_d(w), len(w), _d(p), _d(c)))
    return Distribution(p, c)


def weight_probs(w) -> Distribution:
    w = _f64(np.atleast_2d(w))
    p, c = np.zeros(w.shape[0]), np.zeros(w.shape[0])
    _check(lib().oracle_weight_probs(_d(w), w.shape[0], w.shape[1], _d(p), _d(c)))
    return Distribution(p, c)


def optimal_probs(a, b) -> Distribution:
    a, b = _f64(np.atleast_2d(a)), _f64(np.atleast_2d(b))
    p, c = np.zeros(a.shape[1]), np.zeros(a.shape[1])
    _check(lib().oracle_optimal_probs(_d(a), a.shape[0], a.shape[1], _d(b), b.shape[0], b.shape[1], _d(p), _d(c)))
    return Distribution(p, c)


def draw_indices(dist: Distribution, r: int, seed: int, stream: int, layer: int = 0) -> np.ndarray:
    out = np.zeros(max(r, 1), dtype=np.int64)
    p, c = _f64(dist.probs), _f64(dist.cdf)
    _check(lib().oracle_draw_indices(_d(p), _d(c), len(p), ctypes.c_uint64(seed), ctypes.c_uint64(stream),
                                     ctypes.c_uint32(layer), ctypes.c_long(r), out.ctypes.data_as(_I64)))
    return out[:r]


def approx_matmul(a, b, dist: Distribution, r: int, seed: int, stream: int = 0) -> np.ndarray:
    a, b = _f64(np.atleast_2d(a)), _f64(np.atleast_2d(b))
    out = np.zeros((a.shape[0], b.shape[1]))
    _check(lib().oracle_approx_matmul(_d(a), a.shape[0], a.shape[1], _d(b), b.shape[0], b.shape[1],
                                      _d(_f64(dist.probs)), _d(_f64(dist.cdf)), ctypes.c_long(r),
                                      ctypes.c_uint64(seed), ctypes.c_uint64(stream), _d(out)))
    return out


def approx_encode_row(x_row, w, dist: Distribution, r: int, seed: int, stream: int, layer: int = 0) -> np.ndarray:
    x, w = _f64(x_row).ravel(), _f64(np.atleast_2d(w))
    out = np.zeros(w.shape[1])
    _check(lib().oracle_approx_encode_row(_d(x), _d(w), w.shape[0], w.shape[1], _d(_f64(dist.probs)),
                                          _d(_f64(dist.cdf)), ctypes.c_long(r), ctypes.c_uint64(seed),
                                          ctypes.c_uint64(stream), ctypes.c_uint32(layer), _d(out)))
    return out


# --------------------------------------------------------------- attention
def budget_for(cmax: float, n: int, alpha: float, min_samples: int, d: int) -> tuple[int, bool]:
    r, ex = ctypes.c_long(), ctypes.c_int()
    lib().oracle_budget_for(ctypes.c_double(cmax), ctypes.c_long(n), ctypes.c_double(alpha),
                            ctypes.c_long(min_samples), ctypes.c_long(d), ctypes.byref(r), ctypes.byref(ex))
    return r.value, bool(ex.value)


def sample_budgets_from_cmax(cmax, n: int, alpha: float, min_samples: int, d: int):
    c = _f64(cmax).ravel()
    b = np.zeros(len(c), dtype=np.int32)
    e = np.zeros(len(c), dtype=np.uint8)
    _check(lib().oracle_sample_budgets_from_cmax(_d(c), ctypes.c_long(len(c)), ctypes.c_long(n),
                                                 ctypes.c_double(alpha), ctypes.c_long(min_samples),
                                                 ctypes.c_long(d), b.ctypes.data_as(_I32), e.ctypes.data_as(_U8)))
    return b.reshape(np.shape(cmax)), e.reshape(np.shape(cmax)).astype(bool)


def sample_budgets(attn, alpha: float, d: int, min_samples: int = 1):
    a = _f64(np.atleast_2d(attn))
    n = a.shape[0]
    b = np.zeros(n, dtype=np.int32)
    e = np.zeros(n, dtype=np.uint8)
    _check(lib().oracle_sample_budgets(_d(a), n, ctypes.c_double(alpha), ctypes.c_long(min_samples),
                                       ctypes.c_long(d), b.ctypes.data_as(_I32), e.ctypes.data_as(_U8)))
    return b, e.astype(bool)


def attention_matrix(x, w_q, w_k) -> np.ndarray:
    x, wq, wk = _f64(np.atleast_2d(x)), _f64(np.atleast_2d(w_q)), _f64(np.atleast_2d(w_k))
    out = np.zeros((x.shape[0], x.shape[0]))
    _check(lib().oracle_attention_matrix(_d(x), x.shape[0], x.shape[1], _d(wq), _d(wk), wq.shape[1], _d(out)))
    return out


@dataclass
class FlopsReport:
    exact_encoding: int
    approx_encoding: int
    aggregation: int
    reduction_factor: float
    total_reduction: float


def _flops(counts, ratios) -> FlopsReport:
    return FlopsReport(int(counts[0]), int(counts[1]), int(counts[2]), float(ratios[0]), float(ratios[1]))


@dataclass
class ForwardResult:
    y: np.ndarray
    budgets: np.ndarray
    exact: np.ndarray
    flops: FlopsReport
    draws: np.ndarray | None = None


def forward(x, w_q, w_k, w, alpha: float = 0.4, seed: int = 0, min_samples: int = 1,
            mode: str = "approximation") -> ForwardResult:
    """SPEC mca_forward (mode='approximation') or regular_forward (mode='regular')."""
    x, wq, wk, w = (_f64(np.atleast_2d(m)) for m in (x, w_q, w_k, w))
    n, d = x.shape
    y = np.zeros((n, w.shape[1]))
    b = np.zeros(n, dtype=np.int32)
    e = np.zeros(n, dtype=np.uint8)
    dr = np.zeros((n, d), dtype=np.int64)
    counts = (ctypes.c_uint64 * 3)()
    ratios = (ctypes.c_double * 2)()
    _check(lib().oracle_forward(1 if mode == "approximation" else 0, _d(x), n, d, _d(wq), _d(wk), wq.shape[1],
                                _d(w), w.shape[1], ctypes.c_double(alpha), ctypes.c_long(min_samples),
                                ctypes.c_uint64(seed), _d(y), b.ctypes.data_as(_I32), e.ctypes.data_as(_U8),
                                dr.ctypes.data_as(_I64), counts, ratios))
    return ForwardResult(y, b, e.astype(bool), _flops(counts, ratios), dr)


def multihead_forward(x, w_q, w_k, w, heads: int, alpha: float = 0.4, seed: int = 0, min_samples: int = 1,
                      mode: str = "approximation") -> ForwardResult:
    """SPEC multihead_forward; w_q/w_k: [H, d, dq], w: [H, d, dh]."""
    x = _f64(np.atleast_2d(x))
    wq, wk, w = _f64(w_q), _f64(w_k), _f64(w)
    n, d = x.shape
    dh = w.shape[-1]
    y = np.zeros((n, heads * dh))
    b = np.zeros(n * heads, dtype=np.int32)
    e = np.zeros(n * heads, dtype=np.uint8)
    counts = (ctypes.c_uint64 * 3)()
    ratios = (ctypes.c_double * 2)()
    _check(lib().oracle_multihead_forward(1 if mode == "approximation" else 0, _d(x), n, d, heads, _d(wq), _d(wk),
                                          wq.shape[-1], _d(w), dh, ctypes.c_double(alpha),
                                          ctypes.c_long(min_samples), ctypes.c_uint64(seed), _d(y),
                                          b.ctypes.data_as(_I32), e.ctypes.data_as(_U8), counts, ratios))
    return ForwardResult(y, b.reshape(heads, n), e.reshape(heads, n).astype(bool), _flops(counts, ratios))


@dataclass
class BatchedResult:
    y: np.ndarray
    h: np.ndarray
    budgets: np.ndarray
    exact: np.ndarray
    cmax: np.ndarray
    lse: np.ndarray
    probs: np.ndarray
    cdf: np.ndarray
    flops: FlopsReport


def batched_forward(q, k, x, w, heads: int, alpha: float = 0.4, seed: int = 0, *, min_samples: int = 1,
                    mode: str = "approximation", scale: float = 0.0, b_offset: int = 0, layer: int = 0,
                    budgets_override=None, exact_override=None, threads: int = 0,
                    want_h: bool = True) -> BatchedResult:
    """Device-layout multi-head forward (oracle/batched.hpp): q, k [B, n, H*dh];
    x [B, n, d_in]; w [d_in, H*dh]; per-token outputs [B, H, n]."""
    q, k, x, w = _f64(q), _f64(k), _f64(x), _f64(w)
    B, n, HD = q.shape
    d_in = x.shape[2]
    dh = HD // heads
    if threads:
        set_threads(threads)
    y = np.zeros((B, n, HD))
    h = np.zeros((B, n, HD)) if want_h else None
    b = np.zeros((B, heads, n), dtype=np.int32)
    e = np.zeros((B, heads, n), dtype=np.uint8)
    cm = np.zeros((B, heads, n))
    ls = np.zeros((B, heads, n))
    pr = np.zeros((heads, d_in))
    cd = np.zeros((heads, d_in))
    counts = (ctypes.c_uint64 * 3)()
    ratios = (ctypes.c_double * 2)()
    bo = eo = None
    if budgets_override is not None:
        bo = np.ascontiguousarray(budgets_override, dtype=np.int32)
        eo = np.ascontiguousarray(exact_override, dtype=np.uint8)
    _check(lib().oracle_batched_forward(
        _d(q), _d(k), _d(x), _d(w), B, n, heads, dh, d_in, ctypes.c_double(alpha), ctypes.c_double(scale),
        ctypes.c_long(min_samples), 1 if mode == "approximation" else 0, ctypes.c_uint64(seed), b_offset,
        ctypes.c_uint32(layer), bo.ctypes.data_as(_I32) if bo is not None else None,
        eo.ctypes.data_as(_U8) if eo is not None else None, _d(y), _d(h) if h is not None else None,
        b.ctypes.data_as(_I32), e.ctypes.data_as(_U8), _d(cm), _d(ls), _d(pr), _d(cd), counts, ratios))
    return BatchedResult(y, h, b, e.astype(bool), cm, ls, pr, cd, _flops(counts, ratios))


# ----------------------------------------------------------------- metrics
def flops_for_plan(budgets, exact, d: int, d_out: int | None = None) -> FlopsReport:
    b = np.ascontiguousarray(budgets, dtype=np.int32).ravel()
    e = np.ascontiguousarray(exact, dtype=np.uint8).ravel()
    counts = (ctypes.c_uint64 * 3)()
    ratios = (ctypes.c_double * 2)()
    _check(lib().oracle_flops_for_plan(b.ctypes.data_as(_I32), e.ctypes.data_as(_U8), ctypes.c_long(len(b)),
                                       ctypes.c_long(d), ctypes.c_long(d if d_out is None else d_out), counts, ratios))
    return _flops(counts, ratios)


def predicted_reduction(attn, alpha: float, d: int, min_samples: int = 1) -> float:
    a = _f64(np.atleast_2d(attn))
    out = ctypes.c_double()
    _check(lib().oracle_predicted_reduction(_d(a), a.shape[0], ctypes.c_double(alpha), ctypes.c_long(min_samples),
                                            ctypes.c_long(d), ctypes.byref(out)))
    return out.value


# ------------------------------------------------------------ verify suites
def verify_exactness(fixtures: int = 20, seed: int = 1) -> float:
    return lib().oracle_verify_exactness(fixtures, seed)


def verify_unbiased(seeds: int = 100_000, seed: int = 2) -> float:
    return lib().oracle_verify_unbiased(seeds, seed)


def verify_lemma1(fixtures: int = 10, trials: int = 10_000, seed: int = 3) -> float:
    return lib().oracle_verify_lemma1(fixtures, trials, seed)


def verify_scaling(trials: int = 2_000, seed: int = 4) -> float:
    return lib().oracle_verify_scaling(trials, seed)


def verify_theorem1(alpha: float, n: int = 16, d: int = 128, trials: int = 10_000, seed: int = 5,
                    delta: float = 0.1) -> tuple[float, float, float]:
    a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().oracle_verify_theorem1(ctypes.c_double(alpha), n, d, ctypes.c_long(trials), ctypes.c_uint64(seed),
                                 ctypes.c_double(delta), ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    return a.value, b.value, c.value
