"""Where the fp32 y error at n = 1000 comes from: H~ (K3 / K3b) vs the
aggregation (K4 tf32), on test_random_config_sweep's case 14."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import paper_2201_12854_b200 as mca
from paper_2201_12854_b200 import synthetic as syn
import oracle as orc

def rr(a, b):
    a = a.reshape(-1, a.shape[-1]); b = b.reshape(-1, b.shape[-1])
    return float(np.max(np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), 1e-30)))

c, B, n, H, d_in, alpha = 14, 2, 1000, 12, 256, 0.4
w = syn.make_weights(d_in, H, seed=100 + c)
inp = syn.make_inputs(B, n, d_in, H, seed=100 + c)
q, k, x = (t.cuda() for t in (inp.q, inp.k, inp.x))
weights = mca.AttentionWeights(w.cuda(), heads=H)
hd = torch.empty_like(q)
lse = torch.empty((B, H, n), dtype=torch.float32, device="cuda")
out = mca.mca_forward(weights, q, k, x, mca.McaConfig(alpha=alpha, certify=True), seed=c, return_plan=True,
                      debug=dict(h_out=hd, lse_out=lse))
torch.cuda.synchronize()
npf = lambda t: t.detach().cpu().double().numpy()
ref = orc.batched_forward(npf(q), npf(k), npf(x), npf(w), heads=H, alpha=alpha, seed=c)
print("H~ row_rel", rr(npf(hd), ref.h))
print("y  row_rel", rr(npf(out.y), ref.y))
# exact attention (fp64) times the device's H~
qq, kk = npf(q).reshape(B, n, H, 64), npf(k).reshape(B, n, H, 64)
s = np.einsum("bihd,bjhd->bhij", qq, kk) / 8.0
s -= s.max(axis=-1, keepdims=True)
a = np.exp(s); a /= a.sum(axis=-1, keepdims=True)
hdev = npf(hd).reshape(B, n, H, 64)
y_hdev = np.einsum("bhij,bjhd->bihd", a, hdev).reshape(B, n, H * 64)
print("y(device H~, exact A) vs oracle y", rr(y_hdev, ref.y))
print("device y vs y(device H~, exact A)", rr(npf(out.y), y_hdev))

# exact S with the device's lse: the lse part of the error
s_nat = np.einsum("bihd,bjhd->bhij", qq, kk) / 8.0
lse_ex = np.log(np.exp(s_nat - s_nat.max(-1, keepdims=True)).sum(-1)) + s_nat.max(-1)
ld = npf(lse)
print("lse abs err max", float(np.abs(ld - lse_ex).max()), "rel", float((np.abs(ld - lse_ex) / np.abs(lse_ex)).max()))
a_l = np.exp(s_nat - ld[..., None])
y_l = np.einsum("bhij,bjhd->bihd", a_l, hdev).reshape(B, n, H * 64)
print("y(exact S, device lse, device H~) vs oracle", rr(y_l, ref.y))
