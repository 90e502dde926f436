import sys, time, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
wl = CONFIGS[sys.argv[1]]
prec = sys.argv[2]
dt = torch.float64 if prec == 'f64' else torch.float32
params, x, y, lab = wl.draw()
dev = 'cuda:0'
p = torch.tensor(params, dtype=dt, device=dev); xx = torch.tensor(x, dtype=dt, device=dev); l = torch.tensor(lab, dtype=torch.int32, device=dev)
spec = curv.ModelSpec(wl.widths, wl.activation)
P = wl.P; ld = (P + 3)//4*4
H = torch.zeros((P, ld), dtype=dt, device=dev)
for name, fn in (("hess", curv.dev_assemble_hessian), ("opg", curv.dev_assemble_opg)):
    for it in range(2):
        torch.cuda.synchronize(); t = time.time()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(spec, p, xx, l, wl.n, H, ld, precision=prec); e.record()
        torch.cuda.synchronize()
        print(name, prec, it, "wall %.3f s" % (time.time() - t), "event %.3f ms" % s.elapsed_time(e), "launches", curv.launch_count(), flush=True)
print("nonzero frac", (H != 0).float().mean().item())
