"""Dev timing helper: event-time dev_assemble_hessian / dev_assemble_opg for
a BASELINE config and print the library's per-region profile."""
import sys, time, json, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
wl = CONFIGS[sys.argv[1]]
prec = sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dt = torch.float64 if prec == 'f64' else torch.float32
params, x, y, lab = wl.draw()
dev = 'cuda:0'
p = torch.tensor(params, dtype=dt, device=dev); xx = torch.tensor(x, dtype=dt, device=dev); l = torch.tensor(lab, dtype=torch.int32, device=dev)
spec = curv.ModelSpec(wl.widths, wl.activation)
P = wl.P; ld = (P + 31)//32*32
H = torch.zeros((P, ld), dtype=dt, device=dev)
st = torch.cuda.current_stream()
for name, fn in (("hess", curv.dev_assemble_hessian), ("opg", curv.dev_assemble_opg)):
    for it in range(reps):
        torch.cuda.synchronize(); t = time.time()
        if it == reps - 1: curv.profile_begin()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(st); fn(spec, p, xx, l, wl.n, H, ld, precision=prec, stream=st); e.record(st)
        torch.cuda.synchronize()
        print(name, prec, it, "wall %.3f ms" % ((time.time() - t) * 1e3), "event %.3f ms" % s.elapsed_time(e), flush=True)
    prof = curv.profile_end()
    print("   ", {k: (round(v["ms"], 3), v["launches"]) for k, v in prof.items()})
