
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2105_00053_b200 import _native, ops
L = _native.lib()
rng = np.random.default_rng(11)
for (n, es) in [(8, 0), (16, 1)]:
    M, K, N = 1536, 1031, 1037
    nar = 1 << (n - 1)
    A = rng.integers(0, 1 << n, (M, K)).astype(np.uint64); A[A == nar] = 0
    B = rng.integers(0, 1 << n, (K, N)).astype(np.uint64); B[B == nar] = 0
    A[5, 7] = nar  # one NaR row
    cfg = ops.PositConfig(n, es)
    want = ops.quire_gemm(cfg, torch.from_numpy(A.astype(cfg.np_code_dtype)).cuda(),
                          torch.from_numpy(B.astype(cfg.np_code_dtype)).cuda()).cpu().numpy().astype(np.uint64)
    pa = torch.from_numpy(A.view(np.int64)).pin_memory()
    pb = torch.from_numpy(B.view(np.int64)).pin_memory()
    pc = torch.full((M, N), -1, dtype=torch.int64).pin_memory()
    _native.check(L.pnn_matmul_host(n, es, pa.data_ptr(), pb.data_ptr(), pc.data_ptr(), M, K, N))
    assert (pc.numpy().view(np.uint64) == want).all(), ("pinned", n, es)
    C2 = np.full((M, N), 7, np.uint64)  # pageable: host threads only
    _native.check(L.pnn_matmul_host(n, es, A.ctypes.data, B.ctypes.data, C2.ctypes.data, M, K, N))
    assert (C2 == want).all(), ("pageable", n, es)
print('split ok')
