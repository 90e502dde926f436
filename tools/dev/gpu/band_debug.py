"""dev: one unit band at a time, to localise a failing kernel"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
name, W = sys.argv[1], int(sys.argv[2])
prods = sys.argv[3].split(",") if len(sys.argv) > 3 else ["opg", "hessian"]
wl = CONFIGS[name]
params, x, y, lab = wl.draw()
spec = curv.ModelSpec(wl.widths, wl.activation)
d = "cuda:0"
p = torch.tensor(params, dtype=torch.float32, device=d)
xx = torch.tensor(x, dtype=torch.float32, device=d)
ll = torch.tensor(lab, dtype=torch.int32, device=d)
ld = (wl.P + 31) // 32 * 32
for prod in prods:
    for r in range(W):
        u0, u1, rows = curv.shard_units(spec, W, r)
        print(prod, r, u0, u1, rows, flush=True)
        band = torch.zeros((max(rows, 1), ld), device=d)
        curv.dev_assemble_band(spec, prod, p, xx, ll, wl.n, W, r, band, ld)
        torch.cuda.synchronize()
        print("  ok", flush=True)
