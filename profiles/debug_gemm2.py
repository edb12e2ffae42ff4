import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2006_11972_b200 import executor as ex
e = ex.Executor(n_slots=1, n_ckpts=1, max_steps=8, gemm_mode=ex.GEMM_TC)
for (M, N, K, amn, bmn) in [(128, 16, 8, 1, 0), (128, 16, 8, 0, 1), (128, 128, 64, 1, 1)]:
    rng = np.random.default_rng(0)
    A = rng.standard_normal((M, K)).astype(np.float32); B = rng.standard_normal((N, K)).astype(np.float32)
    C = e.test_gemm(A.T.copy() if amn else A, B.T.copy() if bmn else B, bool(amn), bool(bmn))
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    print(M, N, K, amn, bmn, 'err', np.abs(C - ref).max() / np.abs(ref).max(), 'C[0,:3]', C[0, :3], C[5,:3], 'ref', ref[0, :3], ref[5,:3])
