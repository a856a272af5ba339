"""Pinned host<->device copy bandwidth on this box (the e2e leg's floor)."""
import torch

def bw(src, dst, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    return src.numel() * src.element_size() * reps / (s.elapsed_time(e) / 1e3) / 1e9

n = 151 * 2**20 // 2
h = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d = torch.empty(n, dtype=torch.bfloat16, device="cuda")
print(f"H2D {bw(h, d):.1f} GB/s  D2H {bw(d, h):.1f} GB/s")
# both directions at once
h2 = torch.empty(n // 3, dtype=torch.bfloat16).pin_memory()
d2 = torch.empty(n // 3, dtype=torch.bfloat16, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
ev0.record()
with torch.cuda.stream(s1):
    for _ in range(10):
        d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(10):
        h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
ev1.record()
torch.cuda.synchronize()
t = ev0.elapsed_time(ev1) / 10
print(f"151 MB H2D + 50 MB D2H concurrently: {t:.3f} ms per step")
