"""Dev: GPU-local CPUs / NUMA node and pinned D2H bandwidth with and without binding."""
import os, time, torch, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
bus = pynvml.nvmlDeviceGetPciInfo(h).busId
bus = bus.decode() if isinstance(bus, bytes) else bus
dev = bus.lower()[-12:] if len(bus) > 12 else bus.lower()
path = f"/sys/bus/pci/devices/{dev}"
print("bus", bus, "path exists", os.path.exists(path))
for f in ("local_cpulist", "numa_node"):
    p = os.path.join(path, f)
    print(f, open(p).read().strip() if os.path.exists(p) else None)
print("allowed cpus", len(os.sched_getaffinity(0)), "nodes", os.listdir("/sys/devices/system/node") if os.path.exists("/sys/devices/system/node") else None)
P = 25450
d = torch.randn(P, P + 2, device="cuda")
def bw(hbuf):
    ts = []
    for _ in range(4):
        torch.cuda.synchronize(); t = time.perf_counter(); hbuf.copy_(d[:, :P], non_blocking=True); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    return P * P * 4 / min(ts) / 1e9, P * P * 4 / sorted(ts)[2] / 1e9
h1 = torch.empty((P, P), pin_memory=True)
print("unbound GB/s (best, median)", bw(h1))
lp = os.path.join(path, "local_cpulist")
if os.path.exists(lp):
    cpus = set()
    for part in open(lp).read().strip().split(","):
        a, _, b = part.partition("-"); cpus.update(range(int(a), int(b or a) + 1))
    os.sched_setaffinity(0, cpus & os.sched_getaffinity(0) or cpus)
    h2 = torch.empty((P, P), pin_memory=True)
    print("bound to", len(os.sched_getaffinity(0)), "cpus: GB/s", bw(h2))
