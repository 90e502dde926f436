"""Dev / parity evidence at full size for BASELINE config 4 (P = 1 055 242,
N = 20 000): the top-k eigenvalues of G = (1/N) J^T J from the device
randomized range finder against the exact nonzero spectrum of G, taken from
the dual Gram K = (1/N) J J^T (20 000 x 20 000; fp32 products over column
chunks accumulated in fp64 -- one big SGEMM loses ~1e-3 per entry -- fp64
eigvalsh).  J (84 GB fp32) is formed only for this check.
    python tools/c4_dual_gram.py [power_iters[:oversample] | f:steps:degree[:oversample] ...]
(f: Chebyshev-filtered subspace iteration, curvkit_dev_opg_topk_filtered)"""
import sys, time, json
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS

torch.backends.cuda.matmul.allow_tf32 = False
wl = CONFIGS["c4"]
params, x, y, lab = wl.draw()
dev = "cuda:0"
p = torch.tensor(params, dtype=torch.float32, device=dev)
xx = torch.tensor(x, dtype=torch.float32, device=dev)
ll = torch.tensor(lab, dtype=torch.int32, device=dev)
spec = curv.ModelSpec(wl.widths, wl.activation)
P, n, k = wl.P, wl.n, wl.eig_k
runs = sys.argv[1:] or [str(wl.power_iters)]
lams = {}
for a in runs:
    f = a.startswith("f:")
    r = [] if a.startswith("auto") else [int(v) for v in (a[2:] if f else a).split(":")]
    q = torch.empty((P, k), dtype=torch.float32, device=dev)
    lam = torch.empty(k, dtype=torch.float32, device=dev)
    if a.startswith("auto"):
        ov = int(a.split(":")[1]) if ":" in a else wl.oversample
        call = lambda: curv.dev_opg_topk_auto(spec, p, xx, ll, n, k, ov, 7, q, lam)
        key = f"auto:{ov}"
    elif f:
        st, deg, ov = r[0], r[1], (r[2] if len(r) > 2 else wl.oversample)
        call = lambda: curv.dev_opg_topk_filtered(spec, p, xx, ll, n, k, ov, st, deg, 7, q, lam, precision="tf32")
        key = f"filtered {st}x{deg}:{ov}"
    else:
        it, ov = r[0], (r[1] if len(r) > 1 else wl.oversample)
        call = lambda: curv.dev_opg_topk(spec, p, xx, ll, n, k, ov, it, 7, q, lam, precision="tf32")
        key = f"power {it}:{ov}"
    call()
    torch.cuda.synchronize()
    t0 = time.time()
    call()
    torch.cuda.synchronize()
    lams[key] = (lam.double().cpu().numpy(), time.time() - t0)
    del q
t = time.time()
ldj = (P + 31) // 32 * 32
J = torch.empty((n, ldj), dtype=torch.float32, device=dev)
curv.dev_assemble_jacobian(spec, p, xx, ll, n, J, ldj, precision="f32")
K = torch.zeros((n, n), dtype=torch.float64, device=dev)
for c0 in range(0, P, 16384):  # fp32 products over column chunks, accumulated in fp64
    Jc = J[:, c0:min(P, c0 + 16384)]
    K += (Jc @ Jc.T).double()
del J, Jc
torch.cuda.empty_cache()
K = (K + K.T) / (2.0 * n)
ev = torch.linalg.eigvalsh(K).flip(0)[:k].cpu().numpy()
print(f"dual Gram + eigvalsh: {time.time() - t:.1f} s")
out = {"lambda_exact_top10": ev[:10].tolist(), "lambda_exact_k": float(ev[k - 1])}
for key, (l, secs) in lams.items():
    rel = np.abs(l - ev) / ev
    out[key] = {"seconds": round(secs, 3),"max_rel_err_top10": float(rel[:10].max()), "max_rel_err_top50": float(rel[:50].max()),
                                "max_rel_err_all": float(rel.max()), "median_rel_err": float(np.median(rel)),
                                "n_within_1e-3": int((rel <= 1e-3).sum())}
print(json.dumps(out, indent=1))
