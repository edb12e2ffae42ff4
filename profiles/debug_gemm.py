import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2006_11972_b200 import executor as ex
e = ex.Executor(n_slots=1, n_ckpts=1, max_steps=8, gemm_mode=ex.GEMM_TC)
SHAPES = [(128, 256, 784), (128, 16, 256), (256, 784, 128), (96, 256, 16), (256, 256, 96), (37, 40, 20), (128, 128, 8)]
bad = 0
for rep in range(3):
  for shape in SHAPES:
    for amn in (0, 1):
      for bmn in (0, 1):
        M, N, K = shape
        rng = np.random.default_rng(M * 7 + N * 3 + K)
        A = rng.standard_normal((M, K)).astype(np.float32); B = rng.standard_normal((N, K)).astype(np.float32)
        C = e.test_gemm(A.T.copy() if amn else A, B.T.copy() if bmn else B, bool(amn), bool(bmn))
        ref = A.astype(np.float64) @ B.astype(np.float64).T
        d = np.abs(C - ref)
        err = d.max() / np.abs(ref).max()
        if not err < 1e-5:
            bad += 1
            print(rep, shape, amn, bmn, 'err', err, 'bad cols', np.unique(np.where(~(d <= 1e-3))[1])[:20], 'rows', np.unique(np.where(~(d <= 1e-3))[0])[:10], 'C', C[0,:3], ref[0,:3])
print('bad', bad)
