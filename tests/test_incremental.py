"""The streaming OPG eigensolver (curv::IncrementalOpgEigs, eigensolve.hpp:52-78,
eigensolve.cpp:158-251) through the C-ABI (curvkit_incr_opg_*).

CPU: the constructor's contract (checked before any device work).
GPU: against the reference's own streaming SVD on the golden inputs
(tests/golden/make_incremental_golden.py ran oracle/_ref): the same update
windows, truncations and rank-deficient completion, so eigenvalues agree to
fp64 rounding and eigenvectors up to sign; the reference's ContractErrors;
device-resident blocks."""
import os

import numpy as np
import pytest

from paper_1905_05559_b200 import curv
from paper_1905_05559_b200.errors import ContractError

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("p,k", [(10, 0), (10, 11), (3, -1)])
def test_constructor_contract(p, k):
    with pytest.raises(ContractError):
        curv.IncrementalOpgEigs(p, k)


def _case(name):
    g = np.load(os.path.join(GOLDEN, "incremental_stream.npz"))
    return (g[f"{name}_J"], int(g[f"{name}_block"]), int(g[f"{name}_k"]), g[f"{name}_lam"], g[f"{name}_q"])


def _signs_aligned(q, qr):
    s = np.sign(np.sum(q * qr, axis=0))
    s[s == 0] = 1.0
    return q * s


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c0_stream", "wide_stream", "rank2_k4"])
def test_streaming_matches_reference(name):
    J, block, k, lam_ref, q_ref = _case(name)
    n, p = J.shape
    acc = curv.IncrementalOpgEigs(p, k)
    windows = 0
    buffered = 0
    for r in range(0, n, block):
        acc.push_block(J[r:r + block])
        buffered += min(block, n - r)
        if buffered >= k:  # the reference's update rule (eigensolve.cpp:172)
            windows += 1
            buffered = 0
    assert acc.rows_seen() == n and acc.updates() == windows
    pairs = acc.finalize(n)
    scale = max(lam_ref.max(), 1e-300)
    assert np.max(np.abs(pairs.lam - lam_ref)) <= 1e-10 * scale, (pairs.lam, lam_ref)
    q = _signs_aligned(pairs.q, q_ref)
    assert np.max(np.abs(q - q_ref)) <= 1e-7, np.max(np.abs(q - q_ref))
    assert np.abs(pairs.q.T @ pairs.q - np.eye(k)).max() <= 1e-10


@pytest.mark.gpu
def test_single_block_is_the_exact_svd():
    """acceptance criterion 7: one block with k <= rows reproduces the SVD."""
    g = np.load(os.path.join(GOLDEN, "incremental_svd.npz"))
    J = g["J"]
    acc = curv.IncrementalOpgEigs(J.shape[1], 4)
    acc.push_block(J)
    pairs = acc.finalize(J.shape[0])
    assert np.allclose(pairs.lam, g["lam"], rtol=1e-10, atol=0)
    assert np.max(np.abs(_signs_aligned(pairs.q, g["q"]) - g["q"])) <= 1e-8


@pytest.mark.gpu
def test_reference_contract_errors():
    J = np.random.default_rng(3).standard_normal((20, 8))
    acc = curv.IncrementalOpgEigs(8, 5)
    with pytest.raises(ContractError):
        acc.push_block(J[:0])  # empty block
    acc.push_block(J[:12])
    acc.push_block(J[12:15])  # 3 rows buffered, fewer than k
    with pytest.raises(ContractError):
        acc.finalize(15)  # leftover rows
    with pytest.raises(ContractError):
        acc.finalize(14)  # row count mismatch
    fresh = curv.IncrementalOpgEigs(8, 5)
    fresh.push_block(J[:3])
    with pytest.raises(ContractError):
        fresh.finalize(3)  # no update performed


@pytest.mark.gpu
def test_device_blocks_equal_host_blocks():
    torch = pytest.importorskip("torch")
    J, block, k, lam_ref, _ = _case("wide_stream")
    n, p = J.shape
    a, b = curv.IncrementalOpgEigs(p, k), curv.IncrementalOpgEigs(p, k)
    Jd = torch.tensor(J, dtype=torch.float64, device="cuda:0")
    for r in range(0, n, block):
        a.push_block(J[r:r + block])
        b.push_block(Jd[r:r + block])
    pa, pb = a.finalize(n), b.finalize(n)
    assert np.array_equal(pa.lam, pb.lam) and np.array_equal(pa.q, pb.q)
