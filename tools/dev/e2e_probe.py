"""Dev: where the e2e (host-buffer ABI) time of config 1 goes: the host-API
calls against a bare pitched D2H of the same bytes into the same pinned
buffers."""
import sys, time, ctypes as C
import numpy as np, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv, _lib
from paper_1905_05559_b200.workloads import CONFIGS
wl = CONFIGS["c1"]
params, x, y, lab = wl.draw()
P, n = wl.P, wl.n
spec = curv.ModelSpec(wl.widths, wl.activation)
lib = _lib.load()
hH = torch.empty((P, P), dtype=torch.float32, pin_memory=True)
hG = torch.empty((P, P), dtype=torch.float32, pin_memory=True)
xp, yp, pp = (np.ascontiguousarray(a) for a in (x, y, params))
cfg = curv.CurvatureConfig(batch_size_h=n, batch_size_g=n, memory_cap=1 << 40)._c()
m = spec._c()
dp = lambda a: a.ctypes.data_as(_lib.dptr)
fp = lambda t: C.cast(t.data_ptr(), _lib.fptr)
def h(): _lib.check(lib.curvkit_assemble_hessian_f32(C.byref(m), dp(pp), dp(xp), dp(yp), n, C.byref(cfg), curv.PRECISION["tf32"], fp(hH)))
def g(): _lib.check(lib.curvkit_assemble_opg_f32(C.byref(m), dp(pp), dp(xp), dp(yp), n, C.byref(cfg), curv.PRECISION["tf32"], fp(hG)))
ld = (P + 3) // 4 * 4
d = torch.empty((P, ld), device="cuda")
def d2h(): hH.copy_(d[:, :P], non_blocking=True); torch.cuda.synchronize()
for f, name in ((h, "hessian host API"), (g, "opg host API"), (d2h, "bare pitched D2H 2.59 GB")):
    f()
    ts = []
    for _ in range(8):
        t = time.perf_counter(); f(); ts.append(time.perf_counter() - t)
    print(f"{name:28s} {1e3 * min(ts):8.1f} ms  (median {1e3 * sorted(ts)[len(ts) // 2]:.1f})  all", [round(1e3 * v, 1) for v in ts])
