"""Per-band region profile of config 3's G (or config 2's H: `band_profile.py W c2`) at W ranks, all bands run in turn on one GPU."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1905_05559_b200 import curv  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream()
cfg = sys.argv[2] if len(sys.argv) > 2 else "c3"
product = bench.PRODUCTS[cfg][0]
job = bench.Job(cfg, "tf32", dev, torch)
bench.timed(job, 2, 1, stream, torch)
curv.profile_begin()
bench.timed(job, 1, 0, stream, torch)
prof = curv.profile_end()
print("one GPU: %.2f ms  " % sum(v["ms"] for v in prof.values()) + "  ".join(f"{k} {v['ms']:.2f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1]['ms'])))
wl = job.wl
job.free()
for r in range(W):
    u0, u1, rows = curv.shard_units(job.spec, W, r)
    band = torch.empty((max(1, rows), job.ld), dtype=torch.float32, device=dev)
    f = lambda: curv.dev_assemble_band(job.spec, product, job.p_d, job.x_d, job.l_d, wl.n, W, r, band, job.ld,  # noqa: E731
                                       precision="tf32", stream=stream)
    f()
    torch.cuda.synchronize()
    curv.profile_begin()
    f()
    torch.cuda.synchronize()
    prof = curv.profile_end()
    tot = sum(v["ms"] for v in prof.values())
    print(f"rank {r}: units {list(u0)}..{list(u1)} rows {rows}: {tot:.2f} ms  " +
          "  ".join(f"{k} {v['ms']:.2f}" for k, v in sorted(prof.items(), key=lambda kv: -kv[1]['ms'])))
    del band
    torch.cuda.empty_cache()
