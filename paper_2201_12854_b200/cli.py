"""The reference's command-line harness (module cli) over the
B200 path:

  python -m paper_2201_12854_b200.cli bench  [--input PATH --format mcam|csv | --synthetic uniform|peaked|gaussian]
                                             [--alpha 0.2,0.4] [--dims NxD] [--heads H] [--seed S]
                                             [--mode approx|regular] [--dtype f32|bf16]
  python -m paper_2201_12854_b200.cli import --input PATH [--format mcam|csv] [--out OUT.mcam]
  python -m paper_2201_12854_b200.cli verify [--suite ...]        (paper_2201_12854_b200.verify)

bench (cmd_bench) runs the regular and the approximation
layer on the same attention matrix, inputs and seed through
mca_forward_attn (the device encoding kernels) and prints one CSV row per alpha:
alpha,n,d,reduction_factor,total_reduction,mean_row_error,max_row_error, the
errors being per-row Frobenius norms ||Y~_j - Y_j|| of the layer output
against the exact one. An imported n x n matrix is used for every head;
X ~ N(0, 1) [n, d] and W_V [d, heads*64] (N(0, 0.02^2) with log-normal row
scales) come from the seed. Synthetic attention (DESIGN DECISIONS,
SPEC.md:477-478): uniform; peaked (rows in blocks of --block, default all
rows, each row puts 1 - eps on its block's first column and spreads eps over
the rest: CoLA-like sink columns); gaussian
(row softmax of N(0, 1) logits / --temperature).

import (cmd_attn_import) validates a dump and optionally
writes it back as MCAM. Exit status: 0 pass, 1 verification failure,
2 usage / format / domain error. --seed falls back to MCA_SEED.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

from . import mcam


def _dims(s: str) -> tuple[int, int]:
    try:
        n, d = (int(v) for v in s.lower().split("x"))
    except ValueError:
        raise argparse.ArgumentTypeError(f"--dims must be NxD, got {s!r}") from None
    if n < 1 or d < 1:
        raise argparse.ArgumentTypeError("--dims needs positive N and D")
    return n, d


def synthetic_attention(kind: str, n: int, seed: int, temperature: float = 1.0, eps: float = 0.1,
                        block: int = 0) -> np.ndarray:
    if kind == "uniform":
        return np.full((n, n), 1.0 / n)
    if kind == "peaked":
        block = block or n
        a = np.full((n, n), eps / max(n - 1, 1)) if n > 1 else np.zeros((1, 1))
        for i in range(n):
            c = (i // block) * block
            a[i, c] = 1.0 - eps if n > 1 else 1.0
        return a / a.sum(axis=1, keepdims=True)
    if kind == "gaussian":
        g = np.random.default_rng(seed).standard_normal((n, n)) / temperature
        e = np.exp(g - g.max(axis=1, keepdims=True))
        return e / e.sum(axis=1, keepdims=True)
    raise ValueError(f"unknown synthetic attention {kind!r}")


def synthetic_inputs(n: int, d: int, heads: int, seed: int):
    rng = np.random.default_rng(seed + 1)
    x = rng.standard_normal((n, d))
    w = rng.standard_normal((d, heads * 64)) * 0.02 * np.exp(0.5 * rng.standard_normal((d, 1)))
    return x, w


def bench(args) -> int:
    import torch

    from . import api

    if args.input:
        attn = mcam.attn_import(args.input, args.format)
        if attn.shape[0] != attn.shape[1]:
            raise mcam.FormatError(f"attention must be square, got {attn.shape[0]} x {attn.shape[1]}", 8)
        n, d = attn.shape[0], args.dims[1]
    else:
        n, d = args.dims
        attn = synthetic_attention(args.synthetic, n, args.seed, args.temperature, args.eps, args.block)
    heads = args.heads or max(d // 64, 1)
    dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    x, w = synthetic_inputs(n, d, heads, args.seed)
    dev = torch.device("cuda")
    weights = api.AttentionWeights(torch.from_numpy(w).to(dev, dt), heads=heads)
    xt = torch.from_numpy(x).to(dev, dt)[None]
    at = torch.from_numpy(np.ascontiguousarray(attn)).to(dev)[None, None].expand(1, heads, n, n).contiguous()
    exact = api.forward_given_attention(weights, at, xt, api.McaConfig(alpha=1.0, mode="regular"), seed=args.seed)
    y0 = exact.y.double()
    print("alpha,n,d,reduction_factor,total_reduction,mean_row_error,max_row_error")
    for alpha in args.alpha:
        mode = "approximation" if args.mode == "approx" else "regular"
        out = api.forward_given_attention(weights, at, xt, api.McaConfig(alpha=alpha, mode=mode), seed=args.seed,
                                          flops=True)
        err = (out.y.double() - y0)[0].norm(dim=1)
        f = out.flops
        print(f"{alpha:g},{n},{d},{f.reduction_factor:.10g},{f.total_reduction:.10g},"
              f"{float(err.mean()):.10g},{float(err.max()):.10g}")
    return 0


def do_import(args) -> int:
    a = mcam.attn_import(args.input, args.format)
    s = a.sum(axis=1)
    print("rows,cols,min_row_sum,max_row_sum")
    print(f"{a.shape[0]},{a.shape[1]},{s.min():.17g},{s.max():.17g}")
    if args.out:
        mcam.write_mcam(args.out, a)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="mca", description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench")
    src = b.add_mutually_exclusive_group()
    src.add_argument("--input")
    src.add_argument("--synthetic", choices=["uniform", "peaked", "gaussian"], default="gaussian")
    b.add_argument("--format", choices=["mcam", "csv"], default="mcam")
    b.add_argument("--alpha", type=lambda s: [float(v) for v in s.split(",")], default=[0.2, 0.4, 0.6, 1.0])
    b.add_argument("--dims", type=_dims, default=(32, 128))
    b.add_argument("--heads", type=int, default=0)
    b.add_argument("--seed", type=int, default=None)
    b.add_argument("--mode", choices=["approx", "regular"], default="approx")
    b.add_argument("--dtype", choices=["f32", "bf16"], default="f32")
    b.add_argument("--temperature", type=float, default=1.0)
    b.add_argument("--eps", type=float, default=0.1)
    b.add_argument("--block", type=int, default=0, help="peaked: rows per dominant column (0: all rows, one sink column)")
    i = sub.add_parser("import")
    i.add_argument("--input", required=True)
    i.add_argument("--format", choices=["mcam", "csv"], default="mcam")
    i.add_argument("--out")
    sub.add_parser("verify", add_help=False)
    if argv is None:
        argv = sys.argv[1:]
    if argv[:1] == ["verify"]:
        from . import verify
        return verify.main(argv[1:])
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    if getattr(args, "seed", 0) is None:
        args.seed = int(os.environ.get("MCA_SEED", "0"))
    try:
        if args.cmd == "bench":
            if any(not 0.0 < a <= 1.0 for a in args.alpha):
                print("mca: alpha must be in (0, 1]", file=sys.stderr)
                return 2
            return bench(args)
        return do_import(args)
    except (mcam.FormatError, mcam.DomainError, OSError) as e:
        print(f"mca: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
