"""Dev: one row per captured kernel launch with the counters the design
choices are judged on (duration, DRAM traffic and bandwidth, tensor-pipe
activity, L2 hit rate)."""
import csv, io, subprocess, sys

WANT = {
    "gpu__time_duration.sum": "dur",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_mem_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
}
SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1.0,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {}
    for i, h in enumerate(hdr):
        for k, v in WANT.items():
            if h.endswith(k):
                idx[v] = i
    kn = hdr.index("Kernel Name")
    print("| # | kernel | grid | time (us) | DRAM GB/s | DRAM MB | tensor pipe % | tensor mem % |")
    print("|---|---|---|---|---|---|---|---|")
    for n, r in enumerate(rows[2:]):
        def val(key):
            if key not in idx:
                return None
            try:
                return float(r[idx[key]].replace(",", "")) * SCALE.get(units[idx[key]], 1.0)
            except ValueError:
                return None
        t = val("dur") or 0
        b = (val("dram_rd") or 0) + (val("dram_wr") or 0)
        name = r[kn].replace("void ", "").split("(")[0][:60]
        grid = r[hdr.index("Grid Size")] if "Grid Size" in hdr else ""
        tp = val("tensor_pipe_pct")
        tm = val("tensor_mem_pct")
        f = lambda x: "-" if x is None else f"{x:.1f}"  # noqa: E731
        print(f"| {n} | `{name}` | {grid} | {t * 1e6:.1f} | {b / t / 1e9 if t else 0:.0f} | {b / 1e6:.1f} | {f(tp)} | {f(tm)} |")


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(f"\n{rep}\n")
        main(rep)
