"""dev A/B: time curvkit_dev_assemble_{hessian,opg} of a given libcurvkit_b200.so on c1 (CUDA events)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_1905_05559_b200.workloads import CONFIGS  # noqa: E402

lib = C.CDLL(sys.argv[1])
wl = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c1"]
params, x, y, lab = wl.draw()
d = "cuda:0"
p = torch.tensor(params, dtype=torch.float32, device=d)
xx = torch.tensor(x, dtype=torch.float32, device=d)
ll = torch.tensor(lab, dtype=torch.int32, device=d)
w = (C.c_int64 * len(wl.widths))(*wl.widths)


class M(C.Structure):
    _fields_ = [("L", C.c_int32), ("w", C.POINTER(C.c_int64)), ("a", C.c_int32), ("m", C.c_int32)]


m = M(len(wl.widths), w, 1 if wl.activation == "sigmoid" else 2, 0)
P = wl.P
ld = (P + 31) // 32 * 32
H = torch.empty((P, ld), device=d)
s = torch.cuda.current_stream()
for fn in ("curvkit_dev_assemble_hessian", "curvkit_dev_assemble_opg"):
    f = getattr(lib, fn)
    call = lambda: f(C.byref(m), C.c_void_p(p.data_ptr()), C.c_void_p(xx.data_ptr()), C.c_void_p(ll.data_ptr()),  # noqa
                     C.c_int64(wl.n), C.c_int32(2), C.c_void_p(H.data_ptr()), C.c_int64(ld), C.c_void_p(s.cuda_stream))
    for _ in range(3):
        assert call() == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        call()
    e1.record()
    torch.cuda.synchronize()
    print(sys.argv[1], fn, "%.3f ms" % (e0.elapsed_time(e1) / 20))
