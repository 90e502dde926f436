"""Golden vectors for the streaming OPG eigensolver (curv::IncrementalOpgEigs,
eigensolve.cpp:158-251), produced by the reference library itself
(oracle/_ref) on seeded inputs.  Run here, where /root/reference exists:

    python tests/golden/make_incremental_golden.py

Cases (each: J, block size, k, and the reference's q, lambda):
  c0_stream   config 0's per-example gradient rows (150 x 67, reference
              assemble_jacobian), blocks of 16 rows, k = 5: 9 update windows
              of 16 rows + one of 6 -- the truncation after every window is
              what the device solver must reproduce
  wide_stream 300 x 40 rows with a geometric column scaling, blocks of 7
              rows, k = 6 (windows of 7 rows: buffered >= k after each push)
  rank2_k4    48 x 10 rows of rank 2, one block, k = 4: the rank-deficient
              tail is completed with canonical directions
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref  # noqa: E402
from paper_1905_05559_b200.workloads import CONFIGS, normal  # noqa: E402


def main():
    ref = Ref()
    out = {}
    wl = CONFIGS["c0"]
    params, x, y, _ = wl.draw()
    J0 = ref.jacobian(dict(widths=wl.widths, activation=wl.activation), params, x, y)
    cases = [("c0_stream", J0, 16, 5),
             ("wide_stream", normal(211, 300 * 40).reshape(300, 40) * (0.8 ** np.arange(40)), 7, 6)]
    u = normal(212, 48 * 2).reshape(48, 2)
    v = normal(213, 2 * 10).reshape(2, 10)
    cases.append(("rank2_k4", u @ v, 48, 4))
    for name, J, block, k in cases:
        lam, q = ref.opg_eigs_incremental(J, block, k)
        out[f"{name}_J"] = J
        out[f"{name}_block"] = np.array(block)
        out[f"{name}_k"] = np.array(k)
        out[f"{name}_lam"] = lam
        out[f"{name}_q"] = q
    np.savez_compressed(os.path.join(HERE, "incremental_stream.npz"), **out)
    print("wrote incremental_stream.npz:", ", ".join(n for n, *_ in cases))


if __name__ == "__main__":
    main()
