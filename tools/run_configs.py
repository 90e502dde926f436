"""Dev driver: time the large BASELINE configs on one GPU.
  c2: exact Hessian (P = 55050, H = 12 GB fp32)
  c3: full OPG (P = 109386, G = 48 GB fp32)     c4: top-100 OPG eigenpairs (P = 1.05 M)"""
import sys, time, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
which = sys.argv[1:] or ["c3", "c4"]
dev = 'cuda:0'
for name in which:
    wl = CONFIGS[name]
    params, x, y, lab = wl.draw()
    p = torch.tensor(params, dtype=torch.float32, device=dev)
    xx = torch.tensor(x, dtype=torch.float32, device=dev)
    ll = torch.tensor(lab, dtype=torch.int32, device=dev)
    spec = curv.ModelSpec(wl.widths, wl.activation)
    P = wl.P
    if name == "c2":
        ld = (P + 31) // 32 * 32
        H = torch.empty((P, ld), dtype=torch.float32, device=dev)
        for it in range(2):
            if it == 1: curv.profile_begin()
            torch.cuda.synchronize(); t = time.time()
            curv.dev_assemble_hessian(spec, p, xx, ll, wl.n, H, ld, precision="tf32")
            torch.cuda.synchronize()
            print(name, "hessian", it, "%.1f ms" % ((time.time() - t) * 1e3), flush=True)
        print("  ", {k: (round(v["ms"], 2), v["launches"], round(v["flops"] / v["ms"] / 1e9, 1) if v["flops"] else None) for k, v in curv.profile_end().items()})
        print("   sym", torch.equal(H[:1024, :1024], H[:1024, :1024].T), "H[0,0]", H[0, 0].item(), "mem GB", torch.cuda.max_memory_allocated() / 1e9)
        del H
    if name == "c3":
        ld = (P + 31) // 32 * 32
        G = torch.empty((P, ld), dtype=torch.float32, device=dev)
        for it in range(2):
            if it == 1: curv.profile_begin()
            torch.cuda.synchronize(); t = time.time()
            curv.dev_assemble_opg(spec, p, xx, ll, wl.n, G, ld, precision="tf32")
            torch.cuda.synchronize()
            print(name, "opg", it, "%.1f ms" % ((time.time() - t) * 1e3), flush=True)
        print("  ", {k: (round(v["ms"], 2), v["launches"], round(v["flops"] / v["ms"] / 1e9, 1) if v["flops"] else None) for k, v in curv.profile_end().items()})
        print("   G[0,0]", G[0, 0].item(), "sym", torch.equal(G[:512, :512], G[:512, :512].T), "mem GB", torch.cuda.max_memory_allocated() / 1e9)
        del G
    if name == "c4":
        k = wl.eig_k
        q = torch.empty((P, k), dtype=torch.float32, device=dev)
        lam = torch.empty(k, dtype=torch.float32, device=dev)
        for it in range(2):
            if it == 1: curv.profile_begin()
            torch.cuda.synchronize(); t = time.time()
            curv.dev_opg_topk(spec, p, xx, ll, wl.n, k, wl.oversample, wl.power_iters, 7, q, lam, precision="tf32")
            torch.cuda.synchronize()
            print(name, "topk", it, "%.1f ms" % ((time.time() - t) * 1e3), flush=True)
        print("  ", {k2: (round(v["ms"], 2), v["launches"], round(v["flops"] / v["ms"] / 1e9, 1) if v["flops"] else None, round(v["bytes"] / v["ms"] / 1e6, 1) if v["bytes"] else None) for k2, v in curv.profile_end().items()})
        lamc = lam.cpu()
        print("   lambda[:5]", lamc[:5].tolist(), "lambda[-3:]", lamc[-3:].tolist())
        qtq = q.T @ q
        print("   orthonormality err", (qtq - torch.eye(k, device=dev)).abs().max().item())
