import torch, paper_2201_12854_b200 as mca
torch.manual_seed(0)
B, n, d_in, H = 1, 256, 128, 1
w_v = torch.randn(d_in, H * 64).cuda()
q = torch.randn(B, n, H * 64).cuda() * 0.3
k = torch.randn(B, n, H * 64).cuda() * 0.3
x = torch.randn(B, n, d_in).cuda()
wts = mca.AttentionWeights(w_v, heads=H)
h = torch.zeros(B, n, H * 64, device="cuda")
out = mca.mca_forward(wts, q, k, x, mca.McaConfig(alpha=0.4), seed=1, debug=dict(h_out=h))
torch.cuda.synchronize()
s = (q[0].double() @ k[0].double().T) / 8.0
a = torch.softmax(s, dim=1)
ref = a @ h[0].double()
y = out.y[0].double()
print("y max", y.abs().max().item(), "ref max", ref.abs().max().item(), "err", (y - ref).abs().max().item())
# probe: is y = A @ (something) ? compare to A @ h with columns permuted in 32-blocks
print(y[0, :8]); print(ref[0, :8])
