"""The reference's own acceptance suite (/root/reference/proj/tests/acceptance.cpp,
criteria 1-9) run through the B200 library.

oracle/Makefile compiles the suite twice from the reference sources where
they lie (this container; the binaries travel to the GPU box):
  _ref/acceptance_ref   the unmodified reference library
  _ref/acceptance_b200  curvature.cpp replaced by integration/curvature_b200.cpp
                        (assemble_hessian / assemble_jacobian / assemble_opg on
                        the C-ABI, fp64), curv::hvp routed to
                        integration/hvp_b200.cpp and the eigenpair operators
                        (validate_eigen_pairs, low_rank_*, full_rank_*) to
                        integration/eigops_b200.cpp by link-time --wrap
Criteria 3, 4, 5, 6, 8 and 9 then exercise the GPU path through the reference's
own API; the suite's tolerances are the reference's."""
import os
import subprocess

import pytest

from conftest import ROOT

REF_BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_ref")
B200_BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


def _run(path):
    out = subprocess.run([path], capture_output=True, text=True, timeout=600)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith(("PASS", "FAIL"))]
    return out.returncode, lines, out.stdout + out.stderr


def test_reference_acceptance_suite_on_the_reference():
    if not os.path.exists(REF_BIN):
        pytest.skip("oracle/_ref/acceptance_ref not built (needs /root/reference here)")
    rc, lines, text = _run(REF_BIN)
    assert rc == 0 and len(lines) == 9 and all(ln.startswith("PASS") for ln in lines), text


@pytest.mark.gpu
def test_reference_acceptance_suite_on_b200():
    assert os.path.exists(B200_BIN), "oracle/_ref/acceptance_b200 missing: run __graft_entry__.build() where /root/reference exists"
    rc, lines, text = _run(B200_BIN)
    print(text)
    assert len(lines) == 9, text
    assert all(ln.startswith("PASS") for ln in lines), text
    assert rc == 0, text
