"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per kernel, launches, total and mean time, share of all GPU time.  The
per-launch times are cold-cache and serialised (ncu replays one kernel at a
time), so compare SHARES with bench.py's event-timed breakdown, not absolutes."""
import csv, collections, re, sys
path = sys.argv[1]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(lines))
agg = collections.OrderedDict()
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    short = re.sub(r"\(.*", "", name).replace("void ", "")
    short = re.sub(r"<.*", "", short)
    if "kr_kernel" in name or "tc_gemm_pair_kernel" in name or "tc_hess_fused_kernel" in name or "symkr" in name:
        m = re.search(r"<[^(]*", name)
        short += m.group(0)[:48] if m else ""
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += float(r["Metric Value"]) / 1e3
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':70s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:70]:70s} {c:8d} {t:10.1f} {t / c:9.1f} {100 * t / tot:5.1f}%")
print(f"total {sum(v[0] for v in agg.values())} launches, {tot:.1f} us")
