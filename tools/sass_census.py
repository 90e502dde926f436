"""SASS instruction census of the hot kernels in libcurvkit_b200.so: the
Blackwell-native instructions each kernel contains (tcgen05 MMA = UTC*MMA,
TMA = UTMALDG/UTMASTG, TMEM loads/stores = LDTM/STTM, FP64 tensor = DMMA) and
its static instruction count.

    python tools/sass_census.py [paper_1905_05559_b200/libcurvkit_b200.so] > profiles/r02_sass_census.txt
"""
import collections
import re
import subprocess
import sys

SO = sys.argv[1] if len(sys.argv) > 1 else "paper_1905_05559_b200/libcurvkit_b200.so"
HOT = ("symkr_kernel", "tc_gemm_pair_kernel", "tc_hess_fused_kernel", "kr_kernel", "jacobian_rows_kernel",
       "rgen_kernel", "rgen_f16_kernel", "jt_f16_kernel", "gemm_dmma_kernel", "orbit_dmma_kernel", "jacobi_kernel",
       "gram_kernel", "tc_gemm_kernel")
KEYS = ("UTCHMMA", "UTCQMMA", "UTCMMA", "UTMALDG", "UTMASTG", "UTMAPF", "LDTM", "STTM", "UTCBAR", "DMMA", "HMMA",
        "FFMA", "DFMA")

sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
func, counts, total = None, {}, {}
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        func = m.group(1)
        counts[func] = collections.Counter()
        total[func] = 0
        continue
    if func is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if not m:
        continue
    total[func] += 1
    op, mods = m.group(2), m.group(3) or ""
    for k in KEYS:
        if op == k or op.startswith(k):
            counts[func][op + mods if k in ("UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG") else op] += 1

demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"SASS census of {SO} (cuobjdump -sass; static instruction counts per kernel)\n")
for (f, c), name in zip(counts.items(), demangle):
    if not any(h in name for h in HOT):
        continue
    short = re.sub(r"\(.*", "", name)
    tags = ", ".join(f"{k} x{v}" for k, v in sorted(c.items()))
    print(f"{short}\n    {total[f]} instructions; {tags or '(no tensor/TMA instructions)'}")
