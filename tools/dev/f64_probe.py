"""Dev: per-region times of the f64 (and f32) config-1 products."""
import sys, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
wl = CONFIGS["c1"]; params, x, y, lab = wl.draw()
for prec, dt in (("f64", torch.float64), ("f32", torch.float32)):
    p = torch.tensor(params, dtype=dt, device="cuda"); xx = torch.tensor(x, dtype=dt, device="cuda")
    ll = torch.tensor(lab, dtype=torch.int32, device="cuda")
    spec = curv.ModelSpec(wl.widths, wl.activation); ld = (wl.P + 3) // 4 * 4
    H = torch.empty((wl.P, ld), dtype=dt, device="cuda")
    for f, name in ((curv.dev_assemble_hessian, "H"), (curv.dev_assemble_opg, "G")):
        f(spec, p, xx, ll, wl.n, H, ld, precision=prec); torch.cuda.synchronize()
        curv.profile_begin(); f(spec, p, xx, ll, wl.n, H, ld, precision=prec); torch.cuda.synchronize()
        print(prec, name, {k: (round(v["ms"], 2), round(v["flops"] / v["ms"] / 1e9, 1) if v["flops"] else None) for k, v in curv.profile_end().items()}, flush=True)
