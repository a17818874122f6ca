"""Tensor-core MLP GEMM (tcgen05 kind::tf32, 3xTF32) vs an fp64 numpy product.

Error bound: 3xTF32 keeps ~22 mantissa bits per product; with fp32 accumulation the
elementwise error is bounded by ~K * 2^-21 * (|A| |B|)_elem. We test against
1e-5 * (|A||B|) + 1e-30 (the same forward-error form as R10) which that bound satisfies
for K <= 600 and is far below what a 1-pass TF32 product (~2^-11 relative) could meet."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2412_20379_b200 import ntp
    return ntp.Context()


def _mk(rows, cols, ld, seed):
    rng = np.random.default_rng(seed)
    buf = torch.zeros(rows, ld, dtype=torch.float32, device="cuda")
    a = rng.standard_normal((rows, cols)).astype(np.float32)
    buf[:, :cols] = torch.from_numpy(a)
    return buf[:, :cols], a


@pytest.mark.parametrize("M,N,K", [(300, 256, 602), (1000, 41, 256), (256, 41, 5000), (602, 256, 3000),
                                   (129, 48, 33), (4000, 16, 20), (77, 172, 128), (128, 256, 32), (5, 7, 3)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_gemm_parity(ctx, M, N, K, ta, tb):
    ldA = ((K if not ta else M) + 3) // 4 * 4 + 4
    ldB = ((N if not tb else K) + 3) // 4 * 4
    A, a = _mk(K if ta else M, M if ta else K, ldA, 1)
    B, b = _mk(N if tb else K, K if tb else N, ldB, 2)
    C = torch.full((M, N), 7.0, device="cuda")
    ctx.gemm(A, B, C, trans_a=ta, trans_b=tb)
    torch.cuda.synchronize()
    opa = a.T if ta else a
    opb = b.T if tb else b
    ref = opa.astype(np.float64) @ opb.astype(np.float64)
    den = np.abs(opa).astype(np.float64) @ np.abs(opb).astype(np.float64)
    err = np.abs(C.cpu().numpy() - ref)
    assert (err <= 1e-5 * den + 1e-30).all(), f"max scaled err {(err / (den + 1e-300)).max():.3e}"


def test_gemm_relu_epilogue(ctx):
    A, a = _mk(500, 64, 64, 3)
    B, b = _mk(64, 96, 96, 4)
    C = torch.empty(500, 96, device="cuda")
    ctx.gemm(A, B, C, relu=True)
    torch.cuda.synchronize()
    ref = np.maximum(a.astype(np.float64) @ b.astype(np.float64), 0)
    np.testing.assert_allclose(C.cpu().numpy(), ref, rtol=1e-5, atol=1e-5)
