"""Large / unusual shapes through the public API: no error, finite y, plan sane."""
import sys, torch
sys.path.insert(0, ".")
import paper_2201_12854_b200 as mca
from paper_2201_12854_b200 import synthetic as syn
cases = [(torch.bfloat16, 256, 512, 12, 768, 0.4), (torch.bfloat16, 256, 512, 12, 768, 0.03),
         (torch.bfloat16, 16, 4096, 12, 768, 0.03), (torch.bfloat16, 6000, 8, 12, 768, 0.4),
         (torch.float32, 6000, 8, 12, 768, 0.4), (torch.float32, 2, 4096, 12, 768, 0.4),
         (torch.bfloat16, 8, 512, 16, 1024, 0.2)]
for dt, B, n, H, d_in, alpha in cases:
    w = syn.make_weights(d_in, H, seed=1).to(dt).cuda()
    inp = syn.make_inputs(B, n, d_in, H, seed=2)
    q, k, x = (t.to(dt).cuda() for t in (inp.q, inp.k, inp.x))
    wts = mca.AttentionWeights(w, heads=H)
    out = mca.mca_forward(wts, q, k, x, mca.McaConfig(alpha=alpha), seed=3, return_plan=True, flops=True)
    torch.cuda.synchronize()
    fin = bool(torch.isfinite(out.y.float()).all())
    print(dt, B, n, H, d_in, alpha, "finite", fin, "exact frac", round(float(out.exact_mask.float().mean()), 3),
          "reduction", round(out.flops.reduction_factor, 2), flush=True)
    del out, wts, q, k, x, w
    torch.cuda.empty_cache()
