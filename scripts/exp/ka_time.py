"""Time forward_given_attention at a BERT-base shape (B=16, n=512, H=12): the
aggregation on the tensor cores (default) vs the CUDA cores (MCA_FORCE_SIMT=1,
which also switches the score / encode kernels; compare the ka stage only via
the launch list)."""
import sys, torch
sys.path.insert(0, ".")
import paper_2201_12854_b200 as mca
from paper_2201_12854_b200.synthetic import make_weights
torch.manual_seed(0)
B, n, H, d_in = 16, 512, 12, 768
for dtype in (torch.float32, torch.bfloat16):
    w = make_weights(d_in, H, seed=3).to(dtype).cuda()
    x = torch.randn(B, n, d_in).to(dtype).cuda()
    logits = torch.randn(B, H, n, n, dtype=torch.float64, device="cuda") * 2
    attn = torch.softmax(logits, dim=-1).contiguous()
    wts = mca.AttentionWeights(w, heads=H)
    cfg = mca.McaConfig(alpha=0.4)
    for _ in range(3):
        mca.forward_given_attention(wts, attn, x, cfg, seed=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        mca.forward_given_attention(wts, attn, x, cfg, seed=1)
    e1.record()
    torch.cuda.synchronize()
    print(dtype, "ms per layer", e0.elapsed_time(e1) / 10)
