"""dev: device timings of the eigenpair operators (materialize at config-1 size,
apply at config-4 size) against their HBM floors."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1905_05559_b200 import curv

dev = torch.device("cuda", 0)


def timeit(f, reps=20):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for p, k in ((25450, 100), (55050, 100)):
    q, _ = torch.linalg.qr(torch.randn(p, k, device=dev))
    q = q.contiguous(); lam = torch.linspace(2, 1, k, device=dev)
    for ldh in ((p + 3) // 4 * 4, (p + 31) // 32 * 32):
        h = torch.empty((p, ldh), device=dev)
        print("ldh", ldh)
        for prec in ("tf32", "f32"):
            for lt in (None, 0.5):
                ms = timeit(lambda: curv.dev_eig_materialize(p, k, q, k, lam, h, ldh, lambda_tilde=lt, precision=prec), 10)
                print(f"materialize P={p} k={k} {prec} full={lt is not None}: {ms:.3f} ms, "
                      f"{4.0 * p * p / ms / 1e6:.0f} GB/s stored, {2.0 * p * p * k / ms / 1e9:.1f} TF/s (full square)")
        del h
for p, k in ((1055242, 100), (1055242, 120), (109386, 100)):
    q = torch.randn(p, k, device=dev); lam = torch.linspace(2, 1, k, device=dev)
    for nvec in (1, 4, 16):
        xs = torch.randn(nvec, p, device=dev); y = torch.empty_like(xs)
        quad = torch.empty(nvec, dtype=torch.float64, device=dev)
        ms = timeit(lambda: curv.dev_eig_apply(p, k, q, k, lam, nvec, xs, p, y, p, quad, lambda_tilde=0.5, precision="f32"))
        passes = 2 * ((nvec + 3) // 4)
        print(f"apply P={p} k={k} nvec={nvec}: {ms:.3f} ms, {passes * 4.0 * p * k / ms / 1e6:.0f} GB/s of Q reads")
        ms = timeit(lambda: curv.dev_eig_apply(p, k, q, k, lam, nvec, xs, p, None, 0, quad, lambda_tilde=0.5, precision="f32"))
        print(f"quadform only: {ms:.3f} ms, {((nvec + 3) // 4) * 4.0 * p * k / ms / 1e6:.0f} GB/s")
