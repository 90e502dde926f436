"""Summarise an ncu report: per launch, the headline metrics (dev helper)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
want = sys.argv[2].split(",") if len(sys.argv) > 2 else [
    "Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Compute (SM) Throughput",
    "L1/TEX Cache Throughput", "L2 Cache Throughput", "Registers Per Thread", "Achieved Occupancy"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
seen = {}
for r in rows:
    key = (r["ID"], r["Kernel Name"][:60], r["Grid Size"])
    if r["Metric Name"] in want:
        seen.setdefault(key, {})[(r["Section Name"][:12], r["Metric Name"])] = r["Metric Value"] + " " + r["Metric Unit"]
for k, v in seen.items():
    print(k)
    for m, val in v.items():
        print("    ", m[1], "=", val)
