# projection GEMM shapes at C2: batched (2 x [32768 x 768] . [768 x 768]) vs one [32768 x 768] . [768 x 1536]
import torch
x = torch.randn(32768, 768, device="cuda", dtype=torch.bfloat16)
w2 = torch.randn(2, 768, 768, device="cuda", dtype=torch.bfloat16)
wc = torch.cat([w2[0], w2[1]], dim=1).contiguous()
def t(f, it=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3
xb = x.unsqueeze(0).expand(2, -1, -1)
print("batched bmm  us", round(t(lambda: torch.bmm(xb, w2)), 1))
print("concat N=1536 us", round(t(lambda: x @ wc), 1))
print("single N=768  us", round(t(lambda: x @ w2[0]), 1))
