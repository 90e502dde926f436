"""Dev: device->pinned-host bandwidth, contiguous vs pitched (2D), 1 vs 4 streams."""
import time, torch
P, ld = 25450, 25472
d = torch.randn(P, ld, device="cuda")
h = torch.empty(P, P, pin_memory=True)
hc = torch.empty(P * ld, pin_memory=True)
def t(f, n=3):
    f(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / n
gb = P * P * 4 / 1e9
print("contig 1 stream  GB/s", P * ld * 4 / 1e9 / t(lambda: hc.copy_(d.view(-1), non_blocking=True)))
print("2D     1 stream  GB/s", gb / t(lambda: h.copy_(d[:, :P], non_blocking=True)))
ss = [torch.cuda.Stream() for _ in range(4)]
def multi():
    ev = torch.cuda.current_stream().record_event()
    ch = (P + 3) // 4
    for i, s in enumerate(ss):
        s.wait_event(ev)
        with torch.cuda.stream(s):
            h[i * ch:(i + 1) * ch].copy_(d[i * ch:(i + 1) * ch, :P], non_blocking=True)
    for s in ss: torch.cuda.current_stream().wait_stream(s)
print("2D     4 streams GB/s", gb / t(multi))
