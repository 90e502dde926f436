"""Whole-matrix parity pins at full BASELINE sizes, produced by the reference
itself (oracle/_ref = the unmodified reference sources, TEST INFRASTRUCTURE).

For a seeded Gaussian Omega (P x k, drawn by sketch_omega below) this stores

  c1  H Omega, G Omega   (P = 25 450, k = 16, float64)
  c2  H Omega            (P = 55 050, k = 16, float32)
  c3  G Omega            (P = 109 386, k = 8, float32)

H Omega is k reference HVPs of the dataset-averaged cost (autodiff.cpp:158-244
through HvpOperator); G Omega is (1/N) J^T (J Omega) with J from the
reference's assemble_jacobian (curvature.cpp:94-100) streamed in example
blocks.  A test forms M_gpu Omega from the full GPU matrix and holds
||M_gpu Omega - M_ref Omega||_F / ||M_ref Omega||_F to the precision's
tolerance: a check over every entry of M, not a sample of rows.

  c4  16 reference per-example gradient rows (autodiff.cpp:127-143) of the
      P = 1 055 242 model, kept as their Gram J_s J_s^T (16 x 16), a sketch
      J_s Psi (16 x 8) and the row norms, float64.  They pin the GPU's J
      (and with it the dual Gram (1/N) J J^T the config-4 spectrum test uses)
      to reference data.

    python tests/golden/make_sketch_pins.py [c1 c2 c3 c4]
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref, build  # noqa: E402
from paper_1905_05559_b200.workloads import CONFIGS, normal  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
K = {"c1": 16, "c2": 16, "c3": 8}
C4_ROWS = [0, 1, 2, 777, 1999, 4096, 5000, 8191, 9999, 12345, 13000, 15000, 17777, 19000, 19998, 19999]


def sketch_omega(name: str, P: int, k: int) -> np.ndarray:
    """Seeded Gaussian test matrix (splitmix64 / Box-Muller, workloads.normal)."""
    seed = 0x5EED0000 + int(name[1:])
    return normal(seed, P * k).reshape(P, k)


def c4_psi(P: int) -> np.ndarray:
    return normal(0x5EED0C4, P * 8).reshape(P, 8)


def main(which):
    build()
    ref = Ref()
    lanes = os.cpu_count() or 1
    for name in which:
        wl = CONFIGS[name]
        params, x, y, _ = wl.draw()
        spec = dict(widths=wl.widths, activation=wl.activation)
        P = wl.P
        t = time.time()
        out = dict(widths=np.array(wl.widths), activation=np.array(wl.activation),
                   output_mode=np.array("softmax_cross_entropy"))
        if name == "c4":
            rows = np.array(C4_ROWS)
            Js = ref.jacobian(spec, params, x[rows], y[rows])
            out.update(rows=rows, gram=Js @ Js.T, sketch=Js @ c4_psi(P), norms=np.linalg.norm(Js, axis=1))
        else:
            om = sketch_omega(name, P, K[name])
            dt = np.float64 if name == "c1" else np.float32
            out["k"] = np.array(K[name])
            if wl.task in ("hessian", "hessian+opg"):
                out["h_omega"] = ref.hessian_sketch(spec, params, x, y, om, lanes).astype(dt)
            if wl.task in ("opg", "hessian+opg"):
                out["g_omega"] = ref.opg_sketch(spec, params, x, y, om).astype(dt)
        np.savez_compressed(os.path.join(OUT, f"{name}_sketch.npz"), **out)
        print(f"{name}: sketch pins in {time.time() - t:.1f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4"])
