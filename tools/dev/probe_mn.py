import os, sys, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
M, N, K = 128, 128, 32
dev = 'cuda:0'
torch.manual_seed(0)
A = torch.randn(M, K, device=dev); B = torch.randn(N, K, device=dev)
a_mn = A.T.contiguous()  # [K][M]
ref = A.double() @ B.double().T
C = torch.zeros(M, N, device=dev)
curv.dev_gemm(M, N, K, a_mn, M, 0, B, K, 1, C, N, 1.0, precision="tf32")
torch.cuda.synchronize()
err = ((C.double() - ref).norm() / ref.norm()).item()
print(os.environ.get("CURVKIT_MN_LBO"), os.environ.get("CURVKIT_MN_SBO"), os.environ.get("CURVKIT_MN_KSTEP"), "err", err, "absmax", C.abs().max().item())
# structure probe: A one-hot at (m0,k0), B(n,k) = [n==k]
for (m0, k0) in [(0, 0), (1, 0), (0, 1), (33, 9), (64, 17), (127, 31)]:
    A2 = torch.zeros(M, K, device=dev); A2[m0, k0] = 1.0
    B2 = torch.zeros(N, K, device=dev); B2[torch.arange(K), torch.arange(K)] = 1.0
    C2 = torch.zeros(M, N, device=dev)
    curv.dev_gemm(M, N, K, A2.T.contiguous(), M, 0, B2, K, 1, C2, N, 1.0, precision="tf32")
    torch.cuda.synchronize()
    nz = (C2 != 0).nonzero().tolist()
    print("  onehot", (m0, k0), "->", nz[:4])
