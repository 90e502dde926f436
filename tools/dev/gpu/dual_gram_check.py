"""dev: accuracy of the c4 dual Gram block (fp32 SGEMM vs column-chunked fp32 -> fp64 vs fp64) on 16 pinned rows"""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import load_golden, rel_fro
from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.workloads import CONFIGS
wl = CONFIGS["c4"]; params, x, y, lab = wl.draw(); d = "cuda:0"
spec = curv.ModelSpec(wl.widths, wl.activation); P, n = wl.P, wl.n
ldj = (P + 31) // 32 * 32
J = torch.empty((n, ldj), dtype=torch.float32, device=d)
curv.dev_assemble_jacobian(spec, torch.tensor(params, dtype=torch.float32, device=d), torch.tensor(x, dtype=torch.float32, device=d),
                           torch.tensor(lab, dtype=torch.int32, device=d), n, J, ldj, precision="f32")
pins = load_golden("c4_sketch"); rows = torch.tensor(pins["rows"], device=d)
Js = J[rows, :P]
print("fp32_precision", torch.backends.cuda.matmul.fp32_precision, "allow_tf32", torch.backends.cuda.matmul.allow_tf32)
a = (Js @ Js.T).double().cpu().numpy()
b = (Js.double() @ Js.double().T).cpu().numpy()
c = np.zeros((16, 16))
for c0 in range(0, P, 16384):
    c += (Js[:, c0:c0 + 16384] @ Js[:, c0:c0 + 16384].T).double().cpu().numpy()
big = (J[:2000, :P] @ J[:, :P].T)
ridx = [int(r) for r in pins["rows"] if r < 2000]
e = big[ridx][:, rows].double().cpu().numpy()
print("sgemm16", rel_fro(a, pins["gram"]), "f64", rel_fro(b, pins["gram"]), "chunked", rel_fro(c, pins["gram"]),
      "big-sgemm", rel_fro(e, pins["gram"][:len(ridx)]))
