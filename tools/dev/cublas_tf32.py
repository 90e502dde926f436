"""Dev: cuBLAS TF32 / bf16 GEMM throughput on this GPU (what a library TF32 GEMM reaches)."""
import torch, threading, time
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
torch.backends.cuda.matmul.allow_tf32 = True
for dt, name in ((torch.float32, "tf32"), (torch.bfloat16, "bf16")):
    for (M, N, K) in ((8192, 8192, 8192), (16384, 16384, 1024), (25450, 25450, 1000)):
        a = torch.randn(M, K, device="cuda", dtype=dt); b = torch.randn(K, N, device="cuda", dtype=dt)
        for _ in range(3): c = a @ b
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk = []
        e0.record()
        for i in range(20):
            c = a @ b
            if i == 10: clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{name} {M}x{N}x{K}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.0f} TF/s  sm clk {clk}")
