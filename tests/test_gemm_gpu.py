"""Direct checks of the grouped GEMM kernels (both modes, all four operand-major combinations,
ragged shapes) against float64 numpy."""
import numpy as np
import pytest

from paper_2006_11972_b200 import executor as ex

pytestmark = pytest.mark.gpu

SHAPES = [(128, 256, 784), (128, 16, 256), (256, 784, 128), (96, 256, 16), (256, 256, 96), (37, 40, 20), (128, 128, 8)]


@pytest.fixture(scope="module", params=[ex.GEMM_EXACT, ex.GEMM_TC], ids=["exact", "tc"])
def e(request):
    x = ex.Executor(n_slots=1, n_ckpts=1, max_steps=8, gemm_mode=request.param)
    yield x
    x.close()


@pytest.mark.parametrize("shape", SHAPES, ids=[f"{m}x{n}x{k}" for m, n, k in SHAPES])
@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
def test_gemm(e, shape, a_mn, b_mn):
    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    def store(X, mn):  # row-contiguous operands are stored [K][rows] with a 16-byte aligned pitch
        if not mn:
            return X
        P = np.zeros((X.shape[1], (X.shape[0] + 3) // 4 * 4), np.float32)
        P[:, :X.shape[0]] = X.T
        return P

    C = e.test_gemm(store(A, a_mn), store(B, b_mn), a_mn, b_mn, M=M, N=N)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    err = np.abs(C - ref).max() / np.abs(ref).max()
    # exact mode: one fp32 fmaf chain; tc mode: 3xTF32 products, tensor-core fp32 accumulation
    assert err < (2e-6 if e.desc.gemm_mode == ex.GEMM_EXACT else 1e-5), err
