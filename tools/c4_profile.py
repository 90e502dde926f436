"""Region profile (library CUDA events) of the config-4 top-100 solvers:
the BASELINE setting (2 power iterations) and the converged default."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1905_05559_b200 import curv  # noqa: E402
from paper_1905_05559_b200.workloads import CONFIGS  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "tf32"
wl = CONFIGS["c4"]
params, x, _, labels = wl.draw()
dev = "cuda:0"
p = torch.tensor(params, dtype=torch.float32, device=dev)
xx = torch.tensor(x, dtype=torch.float32, device=dev)
ll = torch.tensor(labels, dtype=torch.int32, device=dev)
spec = curv.ModelSpec(wl.widths, wl.activation)
k = wl.eig_k
q = torch.empty((wl.P, k), dtype=torch.float32, device=dev)
lam = torch.empty(k, dtype=torch.float32, device=dev)
runs = {"baseline": lambda: curv.dev_opg_topk(spec, p, xx, ll, wl.n, k, wl.oversample, wl.power_iters, 7, q, lam,
                                              precision=prec),
        "auto": lambda: curv.dev_opg_topk_auto(spec, p, xx, ll, wl.n, k, wl.oversample, 7, q, lam, precision=prec)}
for name, fn in runs.items():
    fn()
    torch.cuda.synchronize()
    curv.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    prof = curv.profile_end()
    tot = e0.elapsed_time(e1)
    print(f"== {name} ({prec}): {tot:.1f} ms")
    for r, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        tf = v["flops"] / (v["ms"] / 1e3) / 1e12 if v["flops"] else 0
        print(f"  {r:24s} {v['ms']:8.2f} ms  {v['launches']:5d} launches  {tf:7.1f} TF/s")
