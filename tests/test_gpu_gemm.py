"""The tcgen05 TF32 GEMM engine against a plain PyTorch fp64 reference of the
same op.  Tolerances (relative Frobenius): TF32 single pass 2e-3 (10-bit
mantissa operands, fp32 accumulation), 3xTF32 and SIMT fp32 1e-5."""
import pytest

pytestmark = pytest.mark.gpu

TOL = {"tf32": 2e-3, "tf32x3": 1e-5, "f32": 1e-5}

SHAPES = [  # M, N, K
    (128, 256, 32), (128, 128, 64), (256, 256, 1000), (300, 200, 77), (1000, 785, 1000),
    (129, 33, 45), (5000, 300, 257), (64, 64, 8),
]


def _operand(torch, rows, k, kmajor, dev):
    # logical (rows x k) operand stored K-major ([rows][ld]) or MN-major ([k][ld])
    base = torch.randn(rows, k, dtype=torch.float32, device=dev)
    if kmajor:
        ld = (k + 3) // 4 * 4
        buf = torch.zeros(rows, ld, dtype=torch.float32, device=dev)
        buf[:, :k] = base
    else:
        ld = (rows + 3) // 4 * 4
        buf = torch.zeros(k, ld, dtype=torch.float32, device=dev)
        buf[:, :rows] = base.T
    return base, buf, ld


@pytest.mark.parametrize("prec", ["tf32", "tf32x3", "f32"])
@pytest.mark.parametrize("a_k,b_k", [(1, 1), (0, 0), (1, 0), (0, 1)])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_vs_torch(M, N, K, a_k, b_k, prec):
    torch = pytest.importorskip("torch")
    from paper_1905_05559_b200 import curv
    torch.manual_seed(M * 7 + N * 3 + K)
    dev = "cuda:0"
    A, a, lda = _operand(torch, M, K, a_k, dev)
    B, b, ldb = _operand(torch, N, K, b_k, dev)
    ldc = (N + 3) // 4 * 4
    C = torch.full((M, ldc), float("nan"), dtype=torch.float32, device=dev)
    curv.dev_gemm(M, N, K, a, lda, a_k, b, ldb, b_k, C, ldc, 0.5, precision=prec)
    torch.cuda.synchronize()
    ref = 0.5 * (A.double() @ B.double().T)
    got = C[:, :N].double()
    assert not torch.isnan(got).any()
    err = ((got - ref).norm() / ref.norm()).item()
    assert err <= TOL[prec], err
