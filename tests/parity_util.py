"""Shared parity helpers for the GPU tests (test infrastructure).

Budget mismatch accounting: a device budget may differ
from the fp64 oracle's end-to-end budget only where the oracle's raw Eq. 9
value sits at an integer boundary, i.e. where the device's column maximum
(bf16 tensor-core scores, fp32 accumulation) and the oracle's fp64 one fall on
either side of an integer of raw = (n cmax / alpha)^2.
"""
from __future__ import annotations

import numpy as np


def raw_eq9(cmax, n: int, alpha: float) -> np.ndarray:
    """raw = ((n cmax) / alpha)^2 with the oracle's operation order (one IEEE
    binary64 operation per step)."""
    t = (float(n) * np.asarray(cmax, dtype=np.float64)) / float(alpha)
    return t * t


def budget_mismatch_report(b_dev, e_dev, b_ref, e_ref, cmax_ref, n: int, alpha: float) -> dict:
    """Count of token-heads whose device budget / exact flag differs from the
    oracle's, and for those the relative distance of the oracle's raw value to
    the integer boundary between the two budgets: |raw - min(r_dev, r_ref)| /
    min(r_dev, r_ref) (ceil(raw) = r means raw in (r - 1, r])."""
    b_dev, b_ref = np.asarray(b_dev), np.asarray(b_ref)
    mism = (b_dev != b_ref) | (np.asarray(e_dev).astype(bool) != np.asarray(e_ref).astype(bool))
    count = int(mism.sum())
    if count == 0:
        return {"count": 0, "checked": int(b_dev.size), "max_dist_to_int": 0.0}
    raw = raw_eq9(np.asarray(cmax_ref)[mism], n, alpha)
    bound = np.minimum(b_dev[mism], b_ref[mism]).astype(np.float64)
    dist = np.abs(raw - bound) / np.maximum(bound, 1.0)
    return {"count": count, "checked": int(b_dev.size), "max_dist_to_int": float(dist.max())}


def row_rel(a, b) -> float:
    """max over rows of ||a_i - b_i|| / max(||b_i||, tiny) for [..., D] arrays."""
    a = np.asarray(a).reshape(-1, np.shape(a)[-1])
    b = np.asarray(b).reshape(-1, np.shape(b)[-1])
    num = np.linalg.norm(a - b, axis=1)
    den = np.maximum(np.linalg.norm(b, axis=1), 1e-30)
    return float(np.max(num / den))
