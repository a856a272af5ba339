"""fp32 path, 3xTF32 score pass: lse / cmax / y errors against the fp64 oracle
for BERT-shaped (sink-model) and plain Gaussian q, k."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2201_12854_b200 as mca
from paper_2201_12854_b200 import synthetic
from oracle import oracle as orc

H, n, d = 12, 128, 768
w = synthetic.make_weights(d, H)
weights = mca.AttentionWeights(w.cuda(), heads=H)
for name in ("sink", "gauss", "gauss_qk_same", "gauss_x3"):
    inp = synthetic.make_inputs(1, n, d, H)
    q, k, x = inp.q, inp.k, inp.x
    if name.startswith("gauss"):
        g = torch.Generator().manual_seed(5)
        q = torch.randn((1, n, H * 64), generator=g)
        k = q.clone() if name == "gauss_qk_same" else torch.randn((1, n, H * 64), generator=g)
        if name == "gauss_x3":
            q, k = 3 * q, k
    dbg = dict(cmax_out=torch.zeros((1, H, n), dtype=torch.float64, device="cuda"),
               lse_out=torch.zeros((1, H, n), device="cuda"))
    out = mca.mca_forward(weights, q.cuda(), k.cuda(), x.cuda(), mca.McaConfig(alpha=0.4), seed=1, return_plan=True,
                          debug=dbg)
    yr = mca.regular_forward(weights, q.cuda(), k.cuda(), x.cuda())
    torch.cuda.synchronize()
    ref = orc.batched_forward(q.double().numpy(), k.double().numpy(), x.double().numpy(), w.double().numpy(), heads=H,
                              alpha=0.4, seed=1, budgets_override=out.budgets.cpu().numpy(),
                              exact_override=out.exact_mask.cpu().numpy().astype(bool))
    refr = orc.batched_forward(q.double().numpy(), k.double().numpy(), x.double().numpy(), w.double().numpy(),
                               heads=H, mode="regular")
    lse_err = np.abs(dbg["lse_out"].cpu().numpy() - ref.lse).max()
    full = orc.batched_forward(q.double().numpy(), k.double().numpy(), x.double().numpy(), w.double().numpy(), heads=H,
                               alpha=0.4, seed=1)
    cm_err = np.abs(dbg["cmax_out"].cpu().numpy() / full.cmax - 1).max()
    rel = lambda a, b: float((np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)).max())  # noqa: E731
    print(f"{name:14s} max|t| {np.abs(ref.lse).max():6.2f} lse abs err {lse_err:.2e} cmax rel {cm_err:.2e} "
          f"y(mca) {rel(out.y.double().cpu().numpy(), ref.y):.2e} y(regular) {rel(yr.double().cpu().numpy(), refr.y):.2e} "
          f"mism {int((out.budgets.cpu().numpy() != full.budgets).sum())}")
