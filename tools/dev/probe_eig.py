"""Dev probe: the randomized top-k path on a mid-size model (J ~ 10 GB) so
its J X / J^T T GEMMs can be captured under ncu (config 4's 84 GB J is too
large for kernel replay).  Usage: probe_eig.py [reps]"""
import sys, time, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import glorot_params, normal, splitmix64
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
widths, n, k = [784, 160, 10], 20000, 100
spec = curv.ModelSpec(widths, "tanh")
P = curv.param_count(spec)
dev = 'cuda:0'
p = torch.tensor(glorot_params(widths, 5, 0.0), dtype=torch.float32, device=dev)
x = torch.tensor(normal(6, n * widths[0]).reshape(n, widths[0]), dtype=torch.float32, device=dev)
lab = torch.tensor((splitmix64(7, n) % 10).astype('int32'), device=dev)
q = torch.empty((P, k), dtype=torch.float32, device=dev)
lam = torch.empty(k, dtype=torch.float32, device=dev)
for it in range(reps):
    if it == reps - 1: curv.profile_begin()
    torch.cuda.synchronize(); t = time.time()
    curv.dev_opg_topk(spec, p, x, lab, n, k, 20, 2, 7, q, lam, precision="tf32")
    torch.cuda.synchronize()
    print("P", P, "topk", it, "%.1f ms" % ((time.time() - t) * 1e3), flush=True)
print({k2: (round(v["ms"], 2), v["launches"], round(v["bytes"] / v["ms"] / 1e6, 1) if v["bytes"] else None)
       for k2, v in curv.profile_end().items()})
