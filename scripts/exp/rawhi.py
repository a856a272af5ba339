import os, torch, paper_2201_12854_b200 as mca
torch.manual_seed(0)
B, n, d_in, H = 4, 256, 768, 12
f = torch.float32
w_v = torch.randn(d_in, H * 64).cuda()
w_q = (torch.randn(d_in, H * 64) / d_in ** 0.5).cuda()
w_k = (torch.randn(d_in, H * 64) / d_in ** 0.5).cuda()
x = torch.randn(B, n, d_in).cuda()
weights = mca.AttentionWeights(w_v, heads=H, w_q=w_q, w_k=w_k)
outs = []
for v in ("0", "1"):
    os.environ["MCA_EXP_RAW_HI"] = v
    q = torch.zeros(B, n, H * 64, device="cuda"); k = torch.zeros_like(q)
    mca.mca_forward(weights, None, None, x, mca.McaConfig(alpha=0.4), seed=1, debug=dict(q_out=q, k_out=k))
    torch.cuda.synchronize()
    outs.append((q.clone(), k.clone()))
print("q bitwise equal:", torch.equal(outs[0][0], outs[1][0]), "max diff", (outs[0][0] - outs[1][0]).abs().max().item(),
      "max |q|", outs[0][0].abs().max().item())
