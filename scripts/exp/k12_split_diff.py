"""Which outputs differ between MCA_K12_SPLIT=1 and 0 (debug helper)."""
import os, subprocess, sys, torch
sys.path.insert(0, "tests")
from test_gpu_parity import _K12_SNIPPET
root = os.path.abspath(".")
res = {}
for mode in ("1", "0"):
    path = f"/tmp/k12_{mode}.pt"
    r = subprocess.run([sys.executable, "-c", _K12_SNIPPET.format(root=root, path=path)],
                       env=dict(os.environ, MCA_K12_SPLIT=mode), capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    res[mode] = torch.load(path)
names = ("y", "budgets", "exact", "cmax", "lse", "samples", "exact_tokens")
for key in res["1"]:
    for nm, a, b in zip(names, res["1"][key], res["0"][key]):
        if isinstance(a, torch.Tensor):
            if not torch.equal(a, b):
                d = (a.double() - b.double()).abs()
                idx = (d > 0).nonzero()
                print(key, nm, "ndiff", idx.shape[0], "max", float(d.max()), "first idx", idx[:6].tolist())
        elif a != b:
            print(key, nm, a, b)
print("done")
