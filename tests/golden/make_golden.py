"""Generate the golden fixtures under tests/golden/ from the fp64 oracle.

The reference ships no executable code and no fixtures, so
its RNG bits are not pinnable against it. These files pin the build's chosen
rules instead: the Philox generator itself is anchored by the published
Random123 vectors (tests/test_oracle_sampling.py), and these dumps freeze the
oracle's (seed, stream, layer, r) -> indices, Eq. 9 budgets and a small
multi-head forward so that (a) the oracle cannot drift silently and (b) the
GPU path is checked against the same bytes (tests/test_gpu_parity.py).

Run:  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as orc  # noqa: E402


def draws_cases():
    cases = []
    rng = np.random.default_rng(20220130)
    specs = [  # (d, dh, r, seed, stream, layer, zero_rows)
        (16, 4, 40, 42, 0, 0, []),
        (32, 8, 100, 42, 12345, 0, [0, 5, 31]),
        (64, 8, 64, 2**63 + 17, 2**40 + 3, 5, [63]),
        (48, 16, 1, 0, 0, 0, []),
        (24, 8, 500, 7, 99, 23, list(range(0, 24, 3))),
    ]
    for d, dh, r, seed, stream, layer, zero in specs:
        w = rng.standard_normal((d, dh)) * np.exp(0.5 * rng.standard_normal((d, 1)))
        w[zero] = 0.0
        w = np.round(w, 6)  # short decimal text, exactly reproducible
        dist = orc.weight_probs(w)
        idx = orc.draw_indices(dist, r, seed, stream, layer)
        cases.append(dict(w=w.tolist(), r=r, seed=seed, stream=stream, layer=layer, indices=idx.tolist()))
    return cases


def budget_cases():
    out = []
    grid = [(0.5, 4, 0.2, 1, 64), (1 / 128, 128, 1.0, 1, 768), (1 / 512, 512, 1.0, 1, 768), (1.0, 512, 0.05, 1, 768),
            (0.0, 16, 0.4, 1, 128), (0.0, 16, 0.4, 3, 128), (0.25, 8, 1.0, 1, 4), (0.3, 100, 0.7, 2, 1024),
            (1e-5, 4096, 0.2, 1, 768), (0.031, 128, 0.4, 1, 768), (0.0123456789, 512, 0.4, 1, 768)]
    for cmax, n, alpha, mins, d in grid:
        r, ex = orc.budget_for(cmax, n, alpha, mins, d)
        out.append(dict(cmax=cmax, n=n, alpha=alpha, min_samples=mins, d=d, r=r, exact=ex))
    return out


def forward_case():
    rng = np.random.default_rng(7)
    B, n, H, dh, d_in = 2, 8, 2, 4, 16
    q = np.round(rng.standard_normal((B, n, H * dh)) * 2, 4)
    k = np.round(rng.standard_normal((B, n, H * dh)) * 2, 4)
    x = np.round(rng.standard_normal((B, n, d_in)), 4)
    w = np.round(rng.standard_normal((d_in, H * dh)) * 0.5, 4)
    res = orc.batched_forward(q, k, x, w, heads=H, alpha=0.4, seed=42)
    return dict(B=B, n=n, H=H, dh=dh, d_in=d_in, alpha=0.4, seed=42, q=q.tolist(), k=k.tolist(), x=x.tolist(),
                w=w.tolist(), y=res.y.tolist(), budgets=res.budgets.tolist(), exact=res.exact.astype(int).tolist(),
                flops=[res.flops.exact_encoding, res.flops.approx_encoding, res.flops.aggregation])


def main():
    with open(os.path.join(HERE, "draws.json"), "w") as f:
        json.dump({"generator": "philox4x32-10, ctr={k>>1,layer,stream_lo,stream_hi}, key={seed_lo,seed_hi}",
                   "cases": draws_cases()}, f)
    with open(os.path.join(HERE, "budgets.json"), "w") as f:
        json.dump({"rule": "r = clamp(ceil(((n*cmax)/alpha)^2), min_samples, d); exact = ceil(raw) >= d",
                   "cases": budget_cases()}, f, indent=0)
    with open(os.path.join(HERE, "forward_small.json"), "w") as f:
        json.dump(forward_case(), f)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
