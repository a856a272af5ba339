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
