"""Full-size OPG pins for BASELINE config 3 (P = 109 386, N = 10 000): rows of
G computed by the reference's own code (oracle/_ref: assemble_jacobian then
the rank-1 row accumulation of assemble_opg) on the seeded config-3 dataset.
Stored in float32 (the tests compare at 1e-3).  Needs /root/reference (the
compiled oracle/_ref) and ~9 GB of host memory for the reference's J.

    python tests/golden/make_c3_pins.py
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref, build  # noqa: E402
from paper_1905_05559_b200.workloads import CONFIGS  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
# first/interior/last weight rows of layer 0, its first bias, the first weight
# row of layer 1 and the last bias of the output layer
ROWS = [0, 54321, 100351, 100352, 100480, 109385]


def main():
    build()
    ref = Ref()
    wl = CONFIGS["c3"]
    params, x, y, _ = wl.draw()
    spec = dict(widths=wl.widths, activation=wl.activation)
    t = time.time()
    grows = np.concatenate([ref.opg_rows_sample(spec, params, x, y, r, r + 1, 8) for r in ROWS], axis=0)
    print(f"c3 pins: {len(ROWS)} rows in {time.time() - t:.1f} s")
    np.savez_compressed(os.path.join(OUT, "c3_pins.npz"), widths=np.array(wl.widths),
                        activation=np.array(wl.activation), output_mode=np.array("softmax_cross_entropy"),
                        rows=np.array(ROWS), grows=grows.astype(np.float32))


if __name__ == "__main__":
    main()
