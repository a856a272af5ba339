"""fp32 path: cmax from K1b's 3xTF32 winner score (MCA_EXP_TF32_COLSCORE=1) vs
K2's binary64 re-evaluation: relative error against the fp64 oracle, in units of
the certification scale M = 1 + |ln cm| + 2 max|lse| (tau_rel = 3e-6)."""
import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import paper_2201_12854_b200 as mca
from paper_2201_12854_b200 import synthetic as syn
import oracle as orc
npf = lambda t: t.detach().cpu().double().numpy()
for seed, (B, n) in enumerate(((2, 512), (1, 1000), (4, 128))):
    H, d_in = 12, 768
    w = syn.make_weights(d_in, H, seed=50 + seed)
    inp = syn.make_inputs(B, n, d_in, H, seed=50 + seed)
    q, k, x = (t.cuda() for t in (inp.q, inp.k, inp.x))
    wts = mca.AttentionWeights(w.cuda(), heads=H)
    cm = torch.zeros((B, H, n), dtype=torch.float64, device="cuda")
    lse = torch.zeros((B, H, n), dtype=torch.float32, device="cuda")
    mca.mca_forward(wts, q, k, x, mca.McaConfig(alpha=0.4), seed=1, debug=dict(cmax_out=cm, lse_out=lse))
    torch.cuda.synchronize()
    ref = orc.batched_forward(npf(q), npf(k), npf(x), npf(w), heads=H, alpha=0.4, seed=1)
    c = npf(cm)
    lmax = np.abs(npf(lse)).max(axis=-1, keepdims=True)
    M = 1 + np.abs(np.log(ref.cmax)) + 2 * lmax
    e = np.abs(c / ref.cmax - 1) / M
    print(f"B={B} n={n}: max rel err / M = {e.max():.3e}, 99.9% = {np.percentile(e, 99.9):.3e}")
