"""Synthetic BERT-shaped inputs for the MCA layer.

No datasets or checkpoints are reachable, so benchmarks and parity tests use
seeded synthetic tensors of the shapes BASELINE.json names. Plain N(0,1)
logits make almost every column maximum large enough to clamp to the exact
branch (98% at n=512, alpha=0.2), which would never exercise sampling, so the
queries/keys follow a "sink" model that reproduces BERT's [CLS]/[SEP]-style
attention sinks:

  Q[..., 1:] = 0.8 N(0,1), Q[..., 0] = 1
  K[..., 1:] = N(0,1),     K[..., 0] = 0 except 6% sink keys with 3.5 sqrt(d_h)
  X ~ N(0,1)
  W_V ~ N(0, 0.02^2) (BERT init) x log-normal row scales (sigma 0.5), so the
        weight-norm distribution p(i) is non-uniform like a trained model's.

Generation is on the CPU with a seeded torch.Generator (bit-reproducible
across machines), in float32; callers cast to the compute dtype.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class LayerInputs:
    q: torch.Tensor  # [B, n, H*dh]
    k: torch.Tensor  # [B, n, H*dh]
    x: torch.Tensor  # [B, n, d_in]


def make_weights(d_in: int, heads: int, d_h: int = 64, seed: int = 1234) -> torch.Tensor:
    g = torch.Generator().manual_seed(seed)
    w = torch.randn((d_in, heads * d_h), generator=g) * 0.02
    row_scale = torch.exp(0.5 * torch.randn((d_in, 1), generator=g))
    return (w * row_scale).contiguous()


def make_inputs(B: int, n: int, d_in: int, heads: int, d_h: int = 64, seed: int = 1234,
                sink_frac: float = 0.06) -> LayerInputs:
    g = torch.Generator().manual_seed(seed + 1)
    q = 0.8 * torch.randn((B, n, heads, d_h), generator=g)
    q[..., 0] = 1.0
    k = torch.randn((B, n, heads, d_h), generator=g)
    k[..., 0] = 0.0
    sinks = torch.rand((B, n, heads), generator=g) < sink_frac
    k[..., 0] = torch.where(sinks, torch.tensor(3.5 * d_h ** 0.5), torch.tensor(0.0))
    x = torch.randn((B, n, d_in), generator=g)
    return LayerInputs(q.reshape(B, n, heads * d_h).contiguous(), k.reshape(B, n, heads * d_h).contiguous(),
                       x.contiguous())


@dataclass
class ProjectedInputs:
    x: torch.Tensor    # [B, n, d_in]
    w_q: torch.Tensor  # [d_in, H*dh]
    w_k: torch.Tensor  # [d_in, H*dh]


def make_projected_inputs(B: int, n: int, d_in: int, heads: int, d_h: int = 64, seed: int = 1234,
                          sink_frac: float = 0.06) -> ProjectedInputs:
    """x and W_q, W_k whose projections q = x W_q, k = x W_k follow the same
    sink model as `make_inputs` (so the budgets are BERT-like, not the
    near-uniform attention random projections would give):

      x[..., 0] = 1                      a constant feature (BERT's outlier dims)
      x[..., 1 + h] = 3.5 sqrt(d_h)      on 6% sink tokens of head h, else 0
      x[..., 1 + H:] ~ N(0, 1)
      W_q[0, h*dh] = 1                   -> q[..., h*dh] = 1
      W_k[1 + h, h*dh] = 1               -> k[..., h*dh] = 3.5 sqrt(d_h) on sinks
      other columns from the N(0, 1) features with std 0.8 (q) and 1 (k)
    Needs d_in > heads + 1. Float32 on the CPU, seeded."""
    if d_in <= heads + 1:
        raise ValueError("d_in must exceed heads + 1")
    g = torch.Generator().manual_seed(seed + 7)
    rest = d_in - 1 - heads
    x = torch.randn((B, n, d_in), generator=g)
    x[..., 0] = 1.0
    sinks = torch.rand((B, n, heads), generator=g) < sink_frac
    x[..., 1:1 + heads] = torch.where(sinks, torch.tensor(3.5 * d_h ** 0.5), torch.tensor(0.0))
    w_q = torch.zeros((d_in, heads * d_h))
    w_k = torch.zeros((d_in, heads * d_h))
    for h in range(heads):
        c0 = h * d_h
        w_q[0, c0] = 1.0
        w_k[1 + h, c0] = 1.0
        w_q[1 + heads:, c0 + 1:c0 + d_h] = torch.randn((rest, d_h - 1), generator=g) * (0.8 / rest ** 0.5)
        w_k[1 + heads:, c0 + 1:c0 + d_h] = torch.randn((rest, d_h - 1), generator=g) * (1.0 / rest ** 0.5)
    return ProjectedInputs(x.contiguous(), w_q.contiguous(), w_k.contiguous())
