"""Python mirror of the reference's MCA operator interface, backed by the
sm_100a library through the C ABI (include/mca/mca_cuda.h).

Names and argument meanings follow the SPEC ops the path replaces:

  McaConfig          SPEC.md:267-271   (alpha, mode, min_samples; + softmax scale)
  AttentionWeights   SPEC.md:260-265   (W_V on the device + its cached p(i)/cdf)
  mca_forward        SPEC.md:306-314   multi-head, batched (multihead_forward, :326-334)
  multihead_forward  SPEC.md:326-334   alias of mca_forward with explicit heads
  regular_forward
  sample_budgets     SPEC.md:296-304   Eq. 9 on given column maxima
  FlopsReport

Errors raise the SPEC error classes (ShapeError, DomainError, DegenerateError,
ConfigError) or CudaError. Tensors are torch CUDA tensors (torch is used for
device memory and streams only; all compute happens in libmca_b200.so).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _lib as L


class McaError(RuntimeError):
    status = -1


class ShapeError(McaError, ValueError):
    status = L.MCA_ERR_SHAPE


class DomainError(McaError, ValueError):
    status = L.MCA_ERR_DOMAIN


class DegenerateError(McaError, ValueError):
    status = L.MCA_ERR_DEGENERATE


class ConfigError(McaError, ValueError):
    status = L.MCA_ERR_CONFIG


class CudaError(McaError):
    status = L.MCA_ERR_CUDA


class UnsupportedError(McaError):
    status = L.MCA_ERR_UNSUPPORTED


_BY_STATUS = {c.status: c for c in (ShapeError, DomainError, DegenerateError, ConfigError, CudaError,
                                    UnsupportedError)}


def _check(rc: int) -> None:
    if rc != L.MCA_OK:
        msg = L.lib().mca_last_error().decode(errors="replace")
        raise _BY_STATUS.get(rc, McaError)(f"[mca status {rc}] {msg}")


_DTYPES = {torch.float32: L.MCA_F32, torch.bfloat16: L.MCA_BF16}


def _dt(t: torch.Tensor) -> int:
    try:
        return _DTYPES[t.dtype]
    except KeyError:
        raise ConfigError(f"unsupported dtype {t.dtype} (float32 or bfloat16)") from None


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need_cuda(name: str, t: torch.Tensor) -> None:
    if not t.is_cuda:
        raise CudaError(f"{name} must be a CUDA tensor (the MCA forward has no CPU path)")
    if not t.is_contiguous():
        raise ShapeError(f"{name} must be contiguous")


@dataclass
class McaConfig:
    """SPEC.md:267-271. scale <= 0 selects 1/sqrt(d_h).
    certify (bf16): Eq. 9 values within 1e-5 of an integer boundary are
    re-derived in binary64, so the budgets equal the fp64 reference's end to
    end instead of differing at integer boundaries."""
    alpha: float = 0.4
    mode: str = "approximation"
    min_samples: int = 1
    scale: float = 0.0
    certify: bool = False

    def to_c(self) -> L.McaConfigC:
        if self.mode not in ("approximation", "regular"):
            raise ConfigError(f"unknown mode {self.mode!r}")
        return L.McaConfigC(float(self.alpha), float(self.scale), int(self.min_samples),
                            L.MCA_MODE_APPROX if self.mode == "approximation" else L.MCA_MODE_REGULAR,
                            1 if self.certify else 0, 0)


@dataclass
class FlopsReport:
    exact_encoding: int
    approx_encoding: int
    aggregation: int
    samples: int
    exact_tokens: int
    reduction_factor: float
    total_reduction: float
    certified: int = 0          # token-heads whose budget was re-derived in binary64 (k2c_certify)

    @classmethod
    def from_c(cls, f: L.McaFlopsC) -> "FlopsReport":
        return cls(f.exact_encoding, f.approx_encoding, f.aggregation, f.samples, f.exact_tokens,
                   f.reduction_factor, f.total_reduction, f.certified)


class AttentionWeights:
    """SPEC.md:260-265 AttentionWeights{w_q, w_k, w, cached_dist} on the device:
    W_V with its per-head sampling distributions p(i) = ||W_h[i]||^2 /
    ||W_h||_F^2, built once (K0) and cached, and optionally
    W_q / W_k ([d_in, heads*d_h]): with them, mca_forward takes x alone and
    projects q = x W_q, k = x W_k on the device."""

    def __init__(self, w_v: torch.Tensor, heads: int, d_h: int = 64, stream=None, w_q: torch.Tensor | None = None,
                 w_k: torch.Tensor | None = None):
        _need_cuda("w_v", w_v)
        if w_v.dim() != 2 or w_v.shape[1] != heads * d_h:
            raise ShapeError(f"w_v must be [d_in, heads*d_h] = [*, {heads * d_h}], got {tuple(w_v.shape)}")
        self.d_in, self.heads, self.d_h = int(w_v.shape[0]), heads, d_h
        self.dtype = w_v.dtype
        self.device = w_v.device
        h = ctypes.c_void_p()
        with torch.cuda.device(w_v.device):
            _check(L.lib().mca_prepare_weights(_ptr(w_v), _dt(w_v), self.d_in, heads, d_h, _stream(stream),
                                               ctypes.byref(h)))
        self._h = h
        self.has_projections = False
        if (w_q is None) != (w_k is None):
            raise ConfigError("pass both w_q and w_k, or neither")
        if w_q is not None:
            for name, t in (("w_q", w_q), ("w_k", w_k)):
                _need_cuda(name, t)
                if t.shape != w_v.shape or t.dtype != w_v.dtype:
                    raise ShapeError(f"{name} must match w_v: {tuple(w_v.shape)} {w_v.dtype}")
            with torch.cuda.device(w_v.device):
                _check(L.lib().mca_set_projections(self._h, _ptr(w_q), _ptr(w_k), _stream(stream)))
            self.has_projections = True

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise McaError("weights were freed")
        return self._h

    def distributions(self):
        """(probs, cdf) as float64 CPU tensors [heads, d_in]."""
        p = torch.empty((self.heads, self.d_in), dtype=torch.float64)
        c = torch.empty_like(p)
        torch.cuda.synchronize(self.device)
        _check(L.lib().mca_weights_export(self.handle, ctypes.c_void_p(p.data_ptr()), ctypes.c_void_p(c.data_ptr())))
        return p, c

    def reserve(self, max_tokens: int, stream=None) -> None:
        _check(L.lib().mca_reserve(self.handle, int(max_tokens), _stream(stream)))

    def set_timing(self, enable: bool = True) -> None:
        _check(L.lib().mca_set_timing(self.handle, 1 if enable else 0))

    def last_stage_ms(self) -> list[float]:
        buf = (ctypes.c_float * 8)()
        k = L.lib().mca_last_stage_ms(self.handle, buf, 8)
        return [float(buf[i]) for i in range(k)]

    def last_launch_count(self) -> int:
        return int(L.lib().mca_last_launch_count(self.handle))

    def free(self) -> None:
        if self._h is not None:
            L.lib().mca_weights_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


@dataclass
class AttentionOutput:
    """SPEC.md:280-283 (attn itself is never materialised on the device)."""
    y: torch.Tensor
    budgets: torch.Tensor | None = None
    exact_mask: torch.Tensor | None = None
    flops: FlopsReport | None = None
    debug: dict = field(default_factory=dict)


def _check_inputs(weights: AttentionWeights, q, k, x):
    """q and k may both be None when the weights carry W_q / W_k."""
    if (q is None) != (k is None):
        raise ShapeError("pass both q and k, or neither (then the weights must carry W_q / W_k)")
    if q is None and not weights.has_projections:
        raise ConfigError("q / k omitted but the weights carry no W_q / W_k")
    for name, t in (("q", q), ("k", k), ("x", x)):
        if t is None:
            continue
        _need_cuda(name, t)
        if t.dtype != weights.dtype:
            raise ConfigError(f"{name}.dtype {t.dtype} != weights dtype {weights.dtype}")
    if x.dim() != 3 or x.shape[2] != weights.d_in:
        raise ShapeError(f"x must be [B, n, {weights.d_in}], got {tuple(x.shape)}")
    if q is not None:
        if q.dim() != 3 or q.shape != k.shape or q.shape[2] != weights.heads * weights.d_h:
            raise ShapeError(f"q, k must be [B, n, {weights.heads * weights.d_h}], got {tuple(q.shape)}, {tuple(k.shape)}")
        if x.shape[:2] != q.shape[:2]:
            raise ShapeError(f"x must be [B, n, {weights.d_in}] with q's B, n, got {tuple(x.shape)}")
    return int(x.shape[0]), int(x.shape[1])


def mca_forward(weights: AttentionWeights, q: torch.Tensor | None, k: torch.Tensor | None, x: torch.Tensor,
                cfg: McaConfig | None = None, seed: int = 0, *, b_offset: int = 0, layer: int = 0,
                y: torch.Tensor | None = None, return_plan: bool = False, flops: bool = False,
                debug: dict | None = None, stream=None) -> AttentionOutput:
    """Monte-Carlo Attention forward for a batch of sequences and all heads.

    q, k: [B, n, heads*64] (or both None: weights with W_q / W_k project them
    from x on the device, SPEC.md:306-314's mca_forward(x, weights, ...));
    x: [B, n, d_in]; returns y [B, n, heads*64] in the input dtype. Head h of sequence b draws from Philox stream
    ((b_offset + b) * heads + h) * n + j (SPEC.md:356 generalised). With
    return_plan the per-token budgets / exact mask [B, heads, n] come back on
    the device; with flops=True the FlopsReport is read back (synchronises).

    debug (parity testing) may hold CUDA tensors under the mca_debug field
    names: cmax_out (f64), lse_out (f32), h_out (H~: fp32 for fp32 inputs, fp16
    for bf16 inputs), draws_out (+ draws_stride),
    cmax_override (f64), budgets_override (i32) + exact_override (u8), and for
    q = k = None forwards q_out / k_out (the projected q, k).
    """
    cfg = cfg or McaConfig()
    B, n = _check_inputs(weights, q, k, x)
    if y is None:
        y = torch.empty((B, n, weights.heads * weights.d_h), dtype=x.dtype, device=x.device)
    budgets = exact = None
    if return_plan:
        budgets = torch.empty((B, weights.heads, n), dtype=torch.int32, device=x.device)
        exact = torch.empty((B, weights.heads, n), dtype=torch.uint8, device=x.device)
    fl = L.McaFlopsC() if flops else None
    c = cfg.to_c()
    dbg = None
    if debug:
        dbg = L.McaDebugC()
        for name in ("cmax_out", "lse_out", "h_out", "draws_out", "cmax_override", "budgets_override",
                     "exact_override", "q_out", "k_out"):
            t = debug.get(name)
            if t is not None:
                _need_cuda(name, t)
                setattr(dbg, name, t.data_ptr())
        dbg.draws_stride = int(debug.get("draws_stride", 0))
    with torch.cuda.device(x.device):
        args = (weights.handle, _ptr(q), _ptr(k), _ptr(x), _dt(x), B, n, int(b_offset), int(layer), ctypes.byref(c),
                ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), _ptr(y), _ptr(budgets), _ptr(exact),
                ctypes.byref(fl) if fl is not None else None)
        if dbg is not None:
            _check(L.lib().mca_forward_ex(*args, ctypes.byref(dbg), _stream(stream)))
        else:
            _check(L.lib().mca_forward(*args, _stream(stream)))
    return AttentionOutput(y=y, budgets=budgets, exact_mask=exact,
                           flops=FlopsReport.from_c(fl) if fl is not None else None, debug=debug or {})


def forward_given_attention(weights: AttentionWeights, attn: torch.Tensor, x: torch.Tensor,
                            cfg: McaConfig | None = None, seed: int = 0, *, b_offset: int = 0, layer: int = 0,
                            y: torch.Tensor | None = None, return_plan: bool = False, flops: bool = False,
                            stream=None) -> AttentionOutput:
    """The layer on a given attention matrix (what the reference's cli drives
    with an imported or synthetic dump): budgets from attn's
    column maxima, H~ from the forward's encoding kernels, y = attn . H~.
    attn: float64 CUDA [B, heads, n, n] (row i = query i); x: [B, n, d_in].
    cfg.mode "approximation", or "regular" (attn . (x W_V))."""
    cfg = cfg or McaConfig()
    _need_cuda("attn", attn)
    _need_cuda("x", x)
    if x.dtype != weights.dtype:
        raise ConfigError(f"x.dtype {x.dtype} != weights dtype {weights.dtype}")
    if x.dim() != 3 or x.shape[2] != weights.d_in:
        raise ShapeError(f"x must be [B, n, {weights.d_in}], got {tuple(x.shape)}")
    B, n = int(x.shape[0]), int(x.shape[1])
    if attn.dtype != torch.float64 or tuple(attn.shape) != (B, weights.heads, n, n) or not attn.is_contiguous():
        raise ShapeError(f"attn must be contiguous float64 [{B}, {weights.heads}, {n}, {n}], got "
                         f"{attn.dtype} {tuple(attn.shape)}")
    if y is None:
        y = torch.empty((B, n, weights.heads * weights.d_h), dtype=x.dtype, device=x.device)
    budgets = exact = None
    if return_plan:
        budgets = torch.empty((B, weights.heads, n), dtype=torch.int32, device=x.device)
        exact = torch.empty((B, weights.heads, n), dtype=torch.uint8, device=x.device)
    fl = L.McaFlopsC() if flops else None
    c = cfg.to_c()
    with torch.cuda.device(x.device):
        _check(L.lib().mca_forward_attn(weights.handle, _ptr(attn), _ptr(x), _dt(x), B, n, int(b_offset), int(layer),
                                        ctypes.byref(c), ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), _ptr(y),
                                        _ptr(budgets), _ptr(exact), ctypes.byref(fl) if fl is not None else None,
                                        _stream(stream)))
    return AttentionOutput(y=y, budgets=budgets, exact_mask=exact,
                           flops=FlopsReport.from_c(fl) if fl is not None else None)


def multihead_forward(weights: AttentionWeights, q, k, x, cfg: McaConfig | None = None, seed: int = 0, **kw):
    """every head runs the MCA forward on its slice with its
    own cached distribution and stream namespace; outputs are concatenated on
    the feature axis (the [B, n, heads*64] layout) and FLOPs summed."""
    return mca_forward(weights, q, k, x, cfg, seed, **kw)


def regular_forward(weights: AttentionWeights, q, k, x, scale: float = 0.0, y: torch.Tensor | None = None,
                    stream=None) -> torch.Tensor:
    """Exact Y = softmax(a Q K^T) (X W_V); q = k = None with
    projection-carrying weights, as in mca_forward."""
    B, n = _check_inputs(weights, q, k, x)
    if y is None:
        y = torch.empty((B, n, weights.heads * weights.d_h), dtype=x.dtype, device=x.device)
    with torch.cuda.device(x.device):
        _check(L.lib().mca_regular_forward(weights.handle, _ptr(q), _ptr(k), _ptr(x), _dt(x), B, n, float(scale),
                                           _ptr(y), _stream(stream)))
    return y


def sample_budgets(cmax: torch.Tensor, n: int, d: int, cfg: McaConfig | None = None, stream=None):
    """Eq. 9 on given column maxima (float64 CUDA tensor):
    returns (budgets int32, exact_mask uint8) of the same shape."""
    cfg = cfg or McaConfig()
    _need_cuda("cmax", cmax)
    if cmax.dtype != torch.float64:
        raise ConfigError("cmax must be float64")
    b = torch.empty(cmax.shape, dtype=torch.int32, device=cmax.device)
    e = torch.empty(cmax.shape, dtype=torch.uint8, device=cmax.device)
    c = cfg.to_c()
    with torch.cuda.device(cmax.device):
        _check(L.lib().mca_stage_budgets(_ptr(cmax), cmax.numel(), int(n), int(d), ctypes.byref(c), _ptr(b), _ptr(e),
                                         _stream(stream)))
    return b, e
