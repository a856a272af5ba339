"""GPU verify suites: SPEC's statistical acceptance criteria (SPEC.md:442-450
cmd_verify, :499-508 criteria 3-6 and 10) run through the B200 kernels at
GPU speed.

Trials are batched: T copies of one sequence go through ONE forward, and copy
b draws from Philox stream ((b_offset + b) * H + h) * n + j, so the copies are
T independent Monte-Carlo trials. Two fixture scales:
  desk   the SPEC's desk scale with the kernels' head width: d_in = 128 split
         into two heads of 64 (W_h = W[:, 64h:64h+64]), fp32
  bert   BERT-base: d_in = 768, 12 heads of 64, BERT-init W_V with log-normal
         row scales and the sink-model q, k of synthetic.py, 10^4 trials per
         case by default, on the bf16 performance path (theorem1, monotone:
         the whole layer) and the fp32 path (lemma1, scaling, unbiased: the
         encoder in isolation)

  lemma1      ||H~ - x W_h|| mean over trials <= ||x|| ||W_h||_F / sqrt(r), r in {1,4,16,64}
  scaling     log-log slope of the mean ||H~ - x W_h|| over r = 1..256 in [-0.6, -0.4]
  unbiased    mean of H~ over trials within 3 standard errors of x W_h for >= 95% of components
  theorem1    per row, mean ||Y~ - Y|| <= alpha beta ||W_h||_F and the fraction above the
              bound / delta <= 0.12 (delta = 0.1), alpha in {0.2, 0.4, 0.6, 1.0}
  monotone    mean output error at alpha 0.2 < 0.6 < 1.0

  python -m paper_2201_12854_b200.verify [--suite all|lemma1|...] [--trials T] [--seed S] [--scale desk|bert]
prints CSV rows (suite, case, statistic, bound, pass) and exits 0 iff every case passes.
"""
from __future__ import annotations

import argparse
import math
import sys
from dataclasses import dataclass, field

import torch

from . import api

DH = 64
SCALES = {"desk": (2, 128), "bert": (12, 768)}   # (heads, d_in)
BERT_TRIALS = 10_000


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


@dataclass
class Fixture:
    w: torch.Tensor      # [d_in, H*64]
    q: torch.Tensor      # [1, n, H*64]
    k: torch.Tensor
    x: torch.Tensor      # [1, n, d_in]
    heads: int
    d_in: int


def _fixture(seed: int, n: int, scale: str = "desk", dtype=torch.float32) -> Fixture:
    H, d_in = SCALES[scale]
    if scale == "bert":
        from . import synthetic
        w = synthetic.make_weights(d_in, H, seed=seed)
        inp = synthetic.make_inputs(1, n, d_in, H, seed=seed)
        q, k, x = inp.q, inp.k, inp.x
    else:
        g = torch.Generator().manual_seed(seed)
        w = torch.randn((d_in, H * DH), generator=g) * torch.exp(0.5 * torch.randn((d_in, 1), generator=g))
        x = torch.randn((1, n, d_in), generator=g)
        q = torch.randn((1, n, H * DH), generator=g) * 0.3
        k = torch.randn((1, n, H * DH), generator=g) * 0.3
    cast = lambda t: t.to(dtype).cuda()   # noqa: E731
    return Fixture(cast(w), cast(q), cast(k), cast(x), H, d_in)


def _encode(f: Fixture, weights, T: int, r: int, seed: int) -> torch.Tensor:
    """H~ [T, n, H*64] of T independent trials with every budget forced to r."""
    n, H = f.x.shape[1], f.heads
    rep = lambda t: t.expand(T, *t.shape[1:]).contiguous()   # noqa: E731
    hdt = torch.float16 if f.x.dtype == torch.bfloat16 else torch.float32
    h = torch.empty((T, n, H * DH), dtype=hdt, device="cuda")
    dbg = dict(h_out=h, budgets_override=torch.full((T, H, n), r, dtype=torch.int32, device="cuda"),
               exact_override=torch.zeros((T, H, n), dtype=torch.uint8, device="cuda"))
    api.mca_forward(weights, rep(f.q), rep(f.k), rep(f.x), api.McaConfig(alpha=1.0), seed=seed, debug=dbg)
    return h


def _exact_h(f: Fixture) -> torch.Tensor:
    return f.x[0].double() @ f.w.double()   # [n, H*64]


def _default_trials(trials, desk: int, scale: str) -> int:
    return trials if trials else (BERT_TRIALS if scale == "bert" else desk)


def lemma1(trials: int = 0, seed: int = 1, scale: str = "desk") -> VerifyReport:
    trials = _default_trials(trials, 4000, scale)
    rep = VerifyReport(f"lemma1[{scale}]", trials)
    f = _fixture(seed, 8, scale)
    H = f.heads
    weights = api.AttentionWeights(f.w, heads=H)
    ex = _exact_h(f).view(8, H, DH)
    wn = f.w.double().view(f.d_in, H, DH).norm(dim=(0, 2))             # ||W_h||_F
    xn = f.x[0].double().norm(dim=1)                                    # ||x_j||
    for r in (1, 4, 16, 64):
        h = _encode(f, weights, trials, r, seed).double().view(trials, 8, H, DH)
        err = (h - ex).norm(dim=3).mean(dim=0)                          # [n, H]
        bound = xn[:, None] * wn[None, :] / math.sqrt(r)
        ratio = float((err / bound).max())
        rep.cases.append((f"r={r}", ratio, 1.0, ratio <= 1.0))
    return rep


def scaling(trials: int = 0, seed: int = 2, scale: str = "desk") -> VerifyReport:
    trials = _default_trials(trials, 2000, scale)
    rep = VerifyReport(f"scaling[{scale}]", trials)
    f = _fixture(seed, 8, scale)
    H = f.heads
    weights = api.AttentionWeights(f.w, heads=H)
    ex = _exact_h(f).view(8, H, DH)
    rs, errs = [], []
    for e in range(9):
        r = 2 ** e
        h = _encode(f, weights, trials, r, seed).double().view(trials, 8, H, DH)
        rs.append(math.log(r))
        errs.append(math.log(float((h - ex).norm(dim=3).mean())))
    mr, me = sum(rs) / len(rs), sum(errs) / len(errs)
    slope = sum((a - mr) * (b - me) for a, b in zip(rs, errs)) / sum((a - mr) ** 2 for a in rs)
    rep.cases.append(("slope", slope, -0.5, -0.6 <= slope <= -0.4))
    return rep


def unbiased(trials: int = 0, seed: int = 3, scale: str = "desk") -> VerifyReport:
    trials = _default_trials(trials, 20000, scale)
    rep = VerifyReport(f"unbiased[{scale}]", trials)
    f = _fixture(seed, 4, scale)
    weights = api.AttentionWeights(f.w, heads=f.heads)
    h = _encode(f, weights, trials, 6, seed).double()                   # r = 6
    mean, se = h.mean(dim=0), h.std(dim=0) / math.sqrt(trials)
    ex = _exact_h(f)
    within = float(((mean - ex).abs() <= 3 * se + 1e-12).double().mean())
    rep.cases.append(("components within 3 SE", within, 0.95, within >= 0.95))
    return rep


def _theorem1_errors(alpha: float, trials: int, seed: int, scale: str = "desk", n: int = 0):
    bert = scale == "bert"
    n = n or (128 if bert else 16)                                      # BERT: C1's sequence length
    f = _fixture(seed, n, scale, torch.bfloat16 if bert else torch.float32)
    H = f.heads
    weights = api.AttentionWeights(f.w, heads=H)
    y = api.regular_forward(weights, f.q, f.k, f.x).double()            # [1, n, H*64]
    beta = f.x[0].double().norm(dim=1).mean()                           # mean row norm of X
    bound = alpha * beta * f.w.double().view(f.d_in, H, DH).norm(dim=(0, 2))   # [H]
    chunk = max(1, min(trials, (1 << 19) // n))                         # trials per forward (memory bound)
    errs = []
    for t0 in range(0, trials, chunk):
        T = min(chunk, trials - t0)
        rep = lambda t: t.expand(T, *t.shape[1:]).contiguous()         # noqa: E731
        yt = api.mca_forward(weights, rep(f.q), rep(f.k), rep(f.x), api.McaConfig(alpha=alpha), seed=seed,
                             b_offset=t0).y.double()
        errs.append((yt - y).view(T, n, H, DH).norm(dim=3))             # [T, n, H]
    return torch.cat(errs), bound


def theorem1(trials: int = 0, seed: int = 4, delta: float = 0.1, scale: str = "desk") -> VerifyReport:
    trials = _default_trials(trials, 10000, scale)
    rep = VerifyReport(f"theorem1[{scale}]", trials)
    for alpha in (0.2, 0.4, 0.6, 1.0):
        errs, bound = _theorem1_errors(alpha, trials, seed, scale)
        mean_ratio = float((errs.mean(dim=0) / bound).max())
        tail = float((errs > bound / delta).double().mean(dim=0).max())
        rep.cases.append((f"alpha={alpha} mean/bound", mean_ratio, 1.0, mean_ratio <= 1.0))
        rep.cases.append((f"alpha={alpha} tail(delta={delta})", tail, 0.12, tail <= 0.12))
    return rep


def monotone(trials: int = 0, seed: int = 5, scale: str = "desk") -> VerifyReport:
    trials = _default_trials(trials, 2000, scale)
    rep = VerifyReport(f"monotone[{scale}]", trials)
    means = [float(_theorem1_errors(a, trials, seed, scale)[0].mean()) for a in (0.2, 0.6, 1.0)]
    ok = means[0] < means[1] < means[2]
    rep.cases.append(("err(0.2) < err(0.6) < err(1.0)", means[2], means[1], ok))
    return rep


SUITES = {"lemma1": lemma1, "scaling": scaling, "unbiased": unbiased, "theorem1": theorem1, "monotone": monotone}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--suite", default="all", choices=["all", *SUITES])
    ap.add_argument("--trials", type=int, default=0, help="trials per case (default: each suite's)")
    ap.add_argument("--seed", type=int, default=None)
    ap.add_argument("--scale", default="desk", choices=sorted(SCALES),
                    help="desk: d_in=128, 2 heads (SPEC scale); bert: d_in=768, 12 heads, 10^4 trials")
    args = ap.parse_args(argv)
    if not torch.cuda.is_available():
        print("verify: no CUDA device (the suites run the B200 kernels)", file=sys.stderr)
        return 2
    ok = True
    print("suite,case,statistic,bound,pass")
    for name in (SUITES if args.suite == "all" else [args.suite]):
        kw = {"scale": args.scale}
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
