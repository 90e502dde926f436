timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
cat > /tmp/t64.py <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
wl = CONFIGS["c1"]; params, x, y, lab = wl.draw()
for prec, dt in (("f64", torch.float64), ("f32", torch.float32)):
    p = torch.tensor(params, dtype=dt, device="cuda"); xx = torch.tensor(x, dtype=dt, device="cuda"); ll = torch.tensor(lab, dtype=torch.int32, device="cuda")
    spec = curv.ModelSpec(wl.widths, wl.activation); ld = (wl.P + 3) // 4 * 4
    H = torch.empty((wl.P, ld), dtype=dt, device="cuda")
    for f, name in ((curv.dev_assemble_hessian, "H"), (curv.dev_assemble_opg, "G")):
        for it in range(2):
            torch.cuda.synchronize(); t = time.time(); f(spec, p, xx, ll, wl.n, H, ld, precision=prec); torch.cuda.synchronize()
        print(prec, name, "%.1f ms" % ((time.time() - t) * 1e3), flush=True)
PY
timeout 300 python /tmp/t64.py
