"""Dev: summarise the fused-Hessian pipeline trace (CURVKIT_TRACE=1 writes
gpurun_out/trace_<call>.bin: 8 x 1024 clock64 stamps of CTA 0)."""
import sys, numpy as np
TRN = 1024
for fn in [a for a in sys.argv[1:] if a.endswith(".bin")]:
    t = np.fromfile(fn, dtype=np.int64).reshape(8, TRN).astype(np.float64)
    n = int((t[3] > 0).sum())
    nt = int((t[6] > 0).sum())
    if n < 4:
        print(fn, "empty"); continue
    iss, af, td, fu = t[0, :n], t[1, :n], t[2, :n], t[3, :n]
    ok = (af > 0) & (td > 0)
    print(f"{fn}: {n} k-blocks, {nt} tiles in CTA 0")
    q = lambda x: "n/a" if len(x) == 0 else f"med {np.median(x):7.0f}  p10 {np.percentile(x, 10):7.0f}  p90 {np.percentile(x, 90):7.0f}"
    print("  TMA issue -> A landed   ", q((af - iss)[ok]))
    print("  transform (wake->arrive)", q((td - af)[ok]))
    print("  arrive -> MMA sees full ", q((fu - td)[ok]))
    print("  MMA k-block period      ", q(np.diff(fu)))
    print("  issue period            ", q(np.diff(iss)))
    if nt > 1:
        es, ee = t[6, :nt], t[7, :nt]
        print("  epilogue per tile       ", q(ee - es))
        print("  epilogue tile period    ", q(np.diff(es)))
    span = fu[-1] - fu[0]
    print(f"  total MMA span {span:.0f} clk for {n} k-blocks = {span / max(1, n - 1):.0f} clk/k-block")
# transform sub-steps (rows 4, 5 when built with the sub-step stamps)
for fn in [a for a in sys.argv[1:] if a.endswith(".bin")]:
    t = np.fromfile(fn, dtype=np.int64).reshape(8, TRN).astype(np.float64)
    n = int((t[4] > 0).sum())
    if n > 4:
        af, c, f, td = t[1, :n], t[4, :n], t[5, :n], t[2, :n]
        ok = (af > 0) & (td > 0) & (c > 0) & (f > 0)
        print("  transform: loads+math+STS", np.median((c - af)[ok]), " fence", np.median((f - c)[ok]), " syncwarp+arrive", np.median((td - f)[ok]))
# per-tile MMA spans (k-block stamps grouped by tile): shows full vs narrow tiles
if "--tiles" in sys.argv:
    nk = int(sys.argv[sys.argv.index("--tiles") + 1])
    for fn in sys.argv[1:]:
        if not fn.endswith(".bin"): continue
        t = np.fromfile(fn, dtype=np.int64).reshape(8, TRN).astype(np.float64)
        fu = t[3][t[3] > 0]
        nt = len(fu) // nk
        if nt < 2: continue
        spans = [fu[(i + 1) * nk - 1] - fu[i * nk] for i in range(nt)]
        print(fn, "per-tile MMA span (clk, nk - 1 periods):", " ".join(f"{s:.0f}" for s in spans))
