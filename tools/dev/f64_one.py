import sys, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
wl = CONFIGS["c1"]; params, x, y, lab = wl.draw()
p = torch.tensor(params, dtype=torch.float64, device="cuda"); xx = torch.tensor(x, dtype=torch.float64, device="cuda")
ll = torch.tensor(lab, dtype=torch.int32, device="cuda")
spec = curv.ModelSpec(wl.widths, wl.activation); ld = (wl.P + 3) // 4 * 4
H = torch.empty((wl.P, ld), dtype=torch.float64, device="cuda")
curv.dev_assemble_hessian(spec, p, xx, ll, wl.n, H, ld, precision="f64"); torch.cuda.synchronize()
