"""dev: one eigenpair materialize + one apply (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1905_05559_b200 import curv
dev = torch.device("cuda", 0)
p, k = 25450, 100
q, _ = torch.linalg.qr(torch.randn(p, k, device=dev)); q = q.contiguous()
lam = torch.linspace(2, 1, k, device=dev)
ldh = (p + 31) // 32 * 32
h = torch.empty((p, ldh), device=dev)
for _ in range(2):
    curv.dev_eig_materialize(p, k, q, k, lam, h, ldh, lambda_tilde=0.5, precision="tf32")
torch.cuda.synchronize()
p = 1055242
q = torch.randn(p, k, device=dev)
xs = torch.randn(1, p, device=dev); y = torch.empty_like(xs); quad = torch.empty(1, dtype=torch.float64, device=dev)
for _ in range(2):
    curv.dev_eig_apply(p, k, q, k, lam, 1, xs, p, y, p, quad, lambda_tilde=0.5, precision="f32")
torch.cuda.synchronize()
print("ok")
