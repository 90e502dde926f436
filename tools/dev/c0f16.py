import sys; sys.path.insert(0, ".")
import numpy as np
from tests.conftest import load_golden
from paper_1905_05559_b200 import curv
g = load_golden("config0")
s = g["spec"]
spec = curv.ModelSpec(s["widths"], s["activation"], s["output_mode"])
pairs = curv.opg_eigs(spec, g["params"], curv.Batch(g["x"], g["y"]), 5, oversample=10, power_iters=2, seed=3, precision="f16s")
print(pairs.lam)
