"""Dev: top-k Lanczos of the config-1 Hessian (P = 25450) on the GPU, and the
reference's lanczos_topk on the host for the same problem (rank 0, optional,
bounded by --ref-iters)."""
import sys, time
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
wl = CONFIGS["c1"]
params, x, y, lab = wl.draw()
spec = curv.ModelSpec(wl.widths, wl.activation)
for prec in ("f64", "f32"):
    for it in range(2):
        t = time.time()
        r = curv.hessian_lanczos_topk(spec, params, curv.Batch(x, y), wl.n,
                                      curv.LanczosConfig(k=5, max_iterations=400, residual_tol=1e-6, seed=1), precision=prec)
        print(prec, "run", it, "%.1f ms" % ((time.time() - t) * 1e3), "iterations", r.iterations,
              "lambda", [round(v, 6) for v in r.pairs.lam], flush=True)
if "--ref" in sys.argv:
    from oracle.oracle import Ref
    t = time.time()
    q, lam, res, its = Ref().hessian_lanczos({"widths": wl.widths, "activation": wl.activation}, params, x, y, wl.n, 5,
                                             400, 1e-6, 1)
    print("reference", "%.1f s" % (time.time() - t), "iterations", its, "lambda", [round(v, 6) for v in lam])
