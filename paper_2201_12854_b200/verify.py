"""GPU verify suites: SPEC's statistical acceptance criteria (SPEC.md:442-450
cmd_verify, :499-508 criteria 3-6 and 10) run through the B200 kernels at
GPU speed.

Trials are batched: T copies of one sequence go through ONE forward, and copy
b draws from Philox stream ((b_offset + b) * H + h) * n + j, so the copies are
T independent Monte-Carlo trials. Fixtures follow the SPEC's
desk scale with the kernels' head width: d_in = 128 split into two heads of
64 (W_h = W[:, 64h:64h+64]). fp32 (the parity-precision path).

  lemma1      ||H~ - x W_h|| mean over trials <= ||x|| ||W_h||_F / sqrt(r), r in {1,4,16,64}
  scaling     log-log slope of the mean ||H~ - x W_h|| over r = 1..256 in [-0.6, -0.4]
  unbiased    mean of H~ over trials within 3 standard errors of x W_h for >= 95% of components
  theorem1    per row, mean ||Y~ - Y|| <= alpha beta ||W_h||_F and the fraction above the
              bound / delta <= 0.12 (delta = 0.1), alpha in {0.2, 0.4, 0.6, 1.0}
  monotone    mean output error at alpha 0.2 < 0.6 < 1.0

  python -m paper_2201_12854_b200.verify [--suite all|lemma1|...] [--trials T] [--seed S]
prints CSV rows (suite, case, statistic, bound, pass) and exits 0 iff every case passes.
"""
from __future__ import annotations

import argparse
import math
import sys
from dataclasses import dataclass, field

import torch

from . import api

H, DH, D_IN = 2, 64, 128


@dataclass
class VerifyReport:
    suite: str
    trials: int
    cases: list = field(default_factory=list)   # (case, statistic, bound, passed)

    @property
    def passed(self) -> bool:
        return all(c[3] for c in self.cases)

    def csv(self) -> str:
        return "\n".join(f"{self.suite},{c},{s:.6g},{b:.6g},{int(p)}" for c, s, b, p in self.cases)


def _fixture(seed: int, n: int):
    g = torch.Generator().manual_seed(seed)
    w = torch.randn((D_IN, H * DH), generator=g) * torch.exp(0.5 * torch.randn((D_IN, 1), generator=g))
    x = torch.randn((1, n, D_IN), generator=g)
    q = torch.randn((1, n, H * DH), generator=g) * 0.3
    k = torch.randn((1, n, H * DH), generator=g) * 0.3
    return w.cuda(), q.cuda(), k.cuda(), x.cuda()


def _encode(weights, q, k, x, T: int, r: int, seed: int) -> torch.Tensor:
    """H~ [T, n, H*64] of T independent trials with every budget forced to r."""
    n = x.shape[1]
    rep = lambda t: t.expand(T, *t.shape[1:]).contiguous()   # noqa: E731
    h = torch.empty((T, n, H * DH), device="cuda")
    dbg = dict(h_out=h, budgets_override=torch.full((T, H, n), r, dtype=torch.int32, device="cuda"),
               exact_override=torch.zeros((T, H, n), dtype=torch.uint8, device="cuda"))
    api.mca_forward(weights, rep(q), rep(k), rep(x), api.McaConfig(alpha=1.0), seed=seed, debug=dbg)
    return h


def _exact_h(w, x) -> torch.Tensor:
    return (x[0].double() @ w.double())   # [n, H*64]


def lemma1(trials: int = 4000, seed: int = 1) -> VerifyReport:
    rep = VerifyReport("lemma1", trials)
    w, q, k, x = _fixture(seed, 8)
    weights = api.AttentionWeights(w, heads=H)
    ex = _exact_h(w, x).view(8, H, DH)
    wn = w.double().view(D_IN, H, DH).norm(dim=(0, 2))                 # ||W_h||_F
    xn = x[0].double().norm(dim=1)                                      # ||x_j||
    for r in (1, 4, 16, 64):
        h = _encode(weights, q, k, x, trials, r, seed).double().view(trials, 8, H, DH)
        err = (h - ex).norm(dim=3).mean(dim=0)                          # [n, H]
        bound = xn[:, None] * wn[None, :] / math.sqrt(r)
        ratio = float((err / bound).max())
        rep.cases.append((f"r={r}", ratio, 1.0, ratio <= 1.0))
    return rep


def scaling(trials: int = 2000, seed: int = 2) -> VerifyReport:
    rep = VerifyReport("scaling", trials)
    w, q, k, x = _fixture(seed, 8)
    weights = api.AttentionWeights(w, heads=H)
    ex = _exact_h(w, x).view(8, H, DH)
    rs, errs = [], []
    for e in range(9):
        r = 2 ** e
        h = _encode(weights, q, k, x, trials, r, seed).double().view(trials, 8, H, DH)
        rs.append(math.log(r))
        errs.append(math.log(float((h - ex).norm(dim=3).mean())))
    mr, me = sum(rs) / len(rs), sum(errs) / len(errs)
    slope = sum((a - mr) * (b - me) for a, b in zip(rs, errs)) / sum((a - mr) ** 2 for a in rs)
    rep.cases.append(("slope", slope, -0.5, -0.6 <= slope <= -0.4))
    return rep


def unbiased(trials: int = 20000, seed: int = 3) -> VerifyReport:
    rep = VerifyReport("unbiased", trials)
    w, q, k, x = _fixture(seed, 4)
    weights = api.AttentionWeights(w, heads=H)
    h = _encode(weights, q, k, x, trials, 6, seed).double()             # r = 6
    mean, se = h.mean(dim=0), h.std(dim=0) / math.sqrt(trials)
    ex = _exact_h(w, x)
    within = float(((mean - ex).abs() <= 3 * se + 1e-12).double().mean())
    rep.cases.append(("components within 3 SE", within, 0.95, within >= 0.95))
    return rep


def _theorem1_errors(alpha: float, trials: int, seed: int, n: int = 16):
    w, q, k, x = _fixture(seed, n)
    weights = api.AttentionWeights(w, heads=H)
    y = api.regular_forward(weights, q, k, x).double()                  # [1, n, H*64]
    rep = lambda t: t.expand(trials, *t.shape[1:]).contiguous()        # noqa: E731
    yt = api.mca_forward(weights, rep(q), rep(k), rep(x), api.McaConfig(alpha=alpha), seed=seed).y.double()
    errs = (yt - y).view(trials, n, H, DH).norm(dim=3)                  # [T, n, H]
    beta = x[0].double().norm(dim=1).mean()                             # mean row norm of X
    bound = alpha * beta * w.double().view(D_IN, H, DH).norm(dim=(0, 2))   # [H]
    return errs, bound


def theorem1(trials: int = 10000, seed: int = 4, delta: float = 0.1) -> VerifyReport:
    rep = VerifyReport("theorem1", trials)
    for alpha in (0.2, 0.4, 0.6, 1.0):
        errs, bound = _theorem1_errors(alpha, trials, seed)
        mean_ratio = float((errs.mean(dim=0) / bound).max())
        tail = float((errs > bound / delta).double().mean(dim=0).max())
        rep.cases.append((f"alpha={alpha} mean/bound", mean_ratio, 1.0, mean_ratio <= 1.0))
        rep.cases.append((f"alpha={alpha} tail(delta={delta})", tail, 0.12, tail <= 0.12))
    return rep


def monotone(trials: int = 2000, seed: int = 5) -> VerifyReport:
    rep = VerifyReport("monotone", trials)
    means = [float(_theorem1_errors(a, trials, seed)[0].mean()) for a in (0.2, 0.6, 1.0)]
    ok = means[0] < means[1] < means[2]
    rep.cases.append(("err(0.2) < err(0.6) < err(1.0)", means[2], means[1], ok))
    return rep


SUITES = {"lemma1": lemma1, "scaling": scaling, "unbiased": unbiased, "theorem1": theorem1, "monotone": monotone}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--suite", default="all", choices=["all", *SUITES])
    ap.add_argument("--trials", type=int, default=0, help="trials per case (default: each suite's)")
    ap.add_argument("--seed", type=int, default=None)
    args = ap.parse_args(argv)
    if not torch.cuda.is_available():
        print("verify: no CUDA device (the suites run the B200 kernels)", file=sys.stderr)
        return 2
    ok = True
    print("suite,case,statistic,bound,pass")
    for name in (SUITES if args.suite == "all" else [args.suite]):
        kw = {}
        if args.trials:
            kw["trials"] = args.trials
        if args.seed is not None:
            kw["seed"] = args.seed
        r = SUITES[name](**kw)
        print(r.csv(), flush=True)
        ok &= r.passed
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
