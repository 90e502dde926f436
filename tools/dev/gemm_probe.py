"""Dev probe: TF32 GEMM engine throughput for shapes that isolate the
mainloop (huge K) from the epilogue (huge M x N, small K)."""
import sys, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
dev = 'cuda:0'
def run(M, N, K, a_k, b_k, prec="tf32", reps=5):
    A = torch.randn((M, K) if a_k else (K, M), device=dev)
    B = torch.randn((N, K) if b_k else (K, N), device=dev)
    C = torch.empty(M, N, device=dev)
    lda = K if a_k else M; ldb = K if b_k else N
    for _ in range(2): curv.dev_gemm(M, N, K, A, lda, a_k, B, ldb, b_k, C, N, 1.0, precision=prec)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): curv.dev_gemm(M, N, K, A, lda, a_k, B, ldb, b_k, C, N, 1.0, precision=prec)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"M={M} N={N} K={K} a_k={a_k} b_k={b_k} {prec}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.1f} TF/s  out {M*N*4/ms/1e6:.0f} GB/s", flush=True)
for (M, N, K) in [(4096, 4096, 65536), (8192, 8192, 16384), (25472, 25472, 1000), (16384, 16384, 4096)]:
    run(M, N, K, 1, 1)
    run(M, N, K, 0, 0)
