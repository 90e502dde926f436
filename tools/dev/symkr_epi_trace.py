"""Dev: epilogue sub-step times of the symmetric kernel (CURVKIT_TRACE=1 writes
gpurun_out/symkr_epi_<call>.bin): per 8-column chunk of one warp."""
import sys, numpy as np
for fn in sys.argv[1:]:
    t = np.fromfile(fn, dtype=np.int64).reshape(8, 1024).astype(np.float64)
    n = int((t[6] > 0).sum())
    if n < 4: print(fn, "empty"); continue
    t = t[:, :n]
    names = ["tmem_ld+scale", "wait_read", "bar1", "STS+fence", "bar2", "TMA issue+commit"]
    print(f"{fn}: {n} chunks")
    for i, nm in enumerate(names):
        d = t[i + 1] - t[i]
        print(f"  {nm:18s} med {np.median(d):7.0f}  p90 {np.percentile(d, 90):7.0f}")
    per = np.diff(t[0])
    print(f"  chunk period      med {np.median(per):7.0f}  p90 {np.percentile(per, 90):7.0f}")
