"""dev: which shapes break the fp16 J X path (one subprocess per case)."""
import subprocess
import sys

CASE = '''
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import uniform
w = {w}; n = {n}; k = {k}; os_ = {os}
spec = curv.ModelSpec(w, "sigmoid")
P = curv.param_count(spec)
rng = np.random.default_rng(0)
params = rng.standard_normal(P) * 0.3
x = rng.random((n, w[0]))
y = np.eye(w[-1])[rng.integers(0, w[-1], n)]
pairs = curv.opg_eigs(spec, params, curv.Batch(x, y), k, oversample=os_, power_iters=2, seed=3, precision="f16s")
ref = curv.opg_eigs(spec, params, curv.Batch(x, y), k, oversample=os_, power_iters=2, seed=3, precision="tf32")
print("OK", np.max(np.abs(pairs.lam - ref.lam) / np.abs(ref.lam)))
'''
cases = [([4, 8, 3], 150, 5, 10), ([8, 8, 3], 150, 5, 10), ([12, 8, 3], 150, 5, 10), ([20, 8, 3], 150, 5, 10),
         ([4, 16, 3], 150, 5, 10), ([4, 8, 3], 150, 2, 2), ([16, 8, 3], 150, 5, 10), ([64, 32, 10], 300, 5, 10)]
for w, n, k, os_ in cases:
    r = subprocess.run([sys.executable, "-c", CASE.format(w=w, n=n, k=k, os=os_)], capture_output=True, text=True)
    last = (r.stdout.strip().splitlines() or ["?"])[-1] if r.returncode == 0 else r.stderr.strip().splitlines()[-1]
    print(w, n, k, os_, "->", last[:160], flush=True)
