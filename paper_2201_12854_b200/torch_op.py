"""PyTorch binding of the B200 MCA layer (the
paper's "regular vs approximation mode" switch inside a BERT self-attention).

  torch.ops.mca_b200.attention(q, k, x, w_v, heads, alpha, seed, mode, layer)
      a registered custom op (torch.library) over mca_forward /
      regular_forward, with a fake (meta) kernel so it traces under
      torch.compile / FX as an opaque node (the kernels stay libmca_b200's)
  McaSelfAttention(hidden, heads)
      an nn.Module with BERT's parameter layout (query / key / value Linear,
      bias included): q and k come from the Linears, the MCA layer computes
      A . (x W_V), and the value bias is added after the aggregation, which is
      exact because every softmax row sums to 1 (A (X W + b) = A X W + b).
      `.mode` switches between "approximation" and "regular".

Forward only (the reference has no backward: SPEC.md:13). Prepared weights
(K0's sampling tables) are cached per W_V tensor: the cache entry holds a
strong reference to the tensor, so its storage cannot be freed and its
address reused by another W_V while the entry lives, and the key carries the
tensor's version counter, so an in-place update rebuilds the tables.
McaSelfAttention keeps its own transposed W_V, rebuilt when value.weight
changes (new storage or in-place update).
"""
from __future__ import annotations

import torch

from .api import AttentionWeights, McaConfig, mca_forward, regular_forward

_CACHE: dict = {}


def _weights(w_v: torch.Tensor, heads: int) -> AttentionWeights:
    key = (w_v.data_ptr(), w_v._version, tuple(w_v.shape), w_v.dtype, w_v.device, heads)
    hit = _CACHE.get(key)
    if hit is not None and hit[0] is w_v:
        return hit[1]
    if len(_CACHE) >= 64:
        _CACHE.clear()
    wt = AttentionWeights(w_v.contiguous(), heads=heads)
    _CACHE[key] = (w_v, wt)          # the strong reference pins w_v's address while cached
    return wt


@torch.library.custom_op("mca_b200::attention", mutates_args=())
def attention(q: torch.Tensor, k: torch.Tensor, x: torch.Tensor, w_v: torch.Tensor, heads: int, alpha: float,
              seed: int, mode: str, layer: int) -> torch.Tensor:
    """y = A . (x w_v) with A = softmax(q k^T / sqrt(64)) per head (mode
    "regular"), or its Monte-Carlo approximation (mode "approximation")."""
    weights = _weights(w_v, heads)
    q, k, x = q.contiguous(), k.contiguous(), x.contiguous()
    if mode == "regular":
        return regular_forward(weights, q, k, x)
    return mca_forward(weights, q, k, x, McaConfig(alpha=alpha), seed=seed, layer=layer).y


@attention.register_fake
def _(q, k, x, w_v, heads, alpha, seed, mode, layer):
    return q.new_empty(q.shape)


class McaSelfAttention(torch.nn.Module):
    """BERT self-attention (without dropout / attention mask) whose core runs on
    the B200 MCA kernels. hidden = heads * 64. Parameters are named as in
    HF's BertSelfAttention (query, key, value), so a state dict loads as is."""

    def __init__(self, hidden: int = 768, heads: int = 12, alpha: float = 0.4, mode: str = "approximation"):
        super().__init__()
        if hidden != heads * 64:
            raise ValueError("the kernels implement d_h = 64: hidden must be heads * 64")
        self.heads, self.alpha, self.mode = heads, alpha, mode
        self.query = torch.nn.Linear(hidden, hidden)
        self.key = torch.nn.Linear(hidden, hidden)
        self.value = torch.nn.Linear(hidden, hidden)
        self.seed, self.layer = 0, 0
        self._wv = None           # [in, out] copy of value.weight in the activation dtype
        self._wv_src = None       # (data_ptr, version, dtype, device) it was made from

    def _w_v(self, dtype: torch.dtype) -> torch.Tensor:
        p = self.value.weight
        src = (p.data_ptr(), p._version, dtype, p.device)
        if self._wv is None or self._wv_src != src:
            self._wv = p.detach().t().contiguous().to(dtype)   # Linear stores [out, in]
            self._wv_src = src
        return self._wv

    def forward(self, hidden_states: torch.Tensor) -> torch.Tensor:
        q = self.query(hidden_states)
        k = self.key(hidden_states)
        w_v = self._w_v(hidden_states.dtype)
        y = torch.ops.mca_b200.attention(q, k, hidden_states, w_v, self.heads, float(self.alpha), int(self.seed),
                                         self.mode, int(self.layer))
        return y + self.value.bias.to(y.dtype)
