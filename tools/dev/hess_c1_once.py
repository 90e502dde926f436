"""Dev: one device Hessian of config c1 (TF32), timed (CUDA events), for traces / ncu."""
import sys, torch
sys.path.insert(0, '.')
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = CONFIGS[name]
params, x, y, lab = wl.draw()
dev = 'cuda:0'
p = torch.tensor(params, dtype=torch.float32, device=dev)
xx = torch.tensor(x, dtype=torch.float32, device=dev)
ll = torch.tensor(lab, dtype=torch.int32, device=dev)
spec = curv.ModelSpec(wl.widths, wl.activation)
ld = (wl.P + 31) // 32 * 32
H = torch.empty((wl.P, ld), dtype=torch.float32, device=dev)
for it in range(reps):
    if it == reps - 1: curv.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); curv.dev_assemble_hessian(spec, p, xx, ll, wl.n, H, ld, precision="tf32"); e1.record()
    torch.cuda.synchronize()
    print(name, "hessian", it, "%.3f ms" % e0.elapsed_time(e1), flush=True)
print({k: (round(v["ms"], 3), v["launches"], round(v["flops"] / v["ms"] / 1e9, 1) if v["flops"] else None) for k, v in curv.profile_end().items()})
if "--clocks" in sys.argv:  # SM clock / power while the kernel loops (pynvml)
    import threading, time, pynvml
    pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0); samp = []; stop = False
    def mon():
        while not stop:
            samp.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1e3,
                         pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
            time.sleep(0.05)
    th = threading.Thread(target=mon); th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for it in range(1000): curv.dev_assemble_hessian(spec, p, xx, ll, wl.n, H, ld, precision="tf32")
    e1.record(); torch.cuda.synchronize(); stop = True; th.join()
    print("loop ms/iter %.3f" % (e0.elapsed_time(e1) / 1000), "samples (MHz, W, reasons):", samp[len(samp) // 4: len(samp) // 4 + 12])
