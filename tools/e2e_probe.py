"""Time pnn_matmul_host phases (PNN_HOST_PROFILE=1) and raw host/PCIe rates on
the GPU box: memcpy bandwidth of the pool-narrowing loop and pinned H2D/D2H."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_00053_b200 import _native  # noqa: E402

M = N = K = 4096
L = _native.lib()
for nb, es in ((8, 0), (16, 1)):
    rng = np.random.default_rng(0)
    A = torch.from_numpy(rng.integers(0, 1 << (nb - 1), (M, K)).astype(np.int64)).pin_memory()
    B = torch.from_numpy(rng.integers(0, 1 << (nb - 1), (K, N)).astype(np.int64)).pin_memory()
    Cc = torch.empty((M, N), dtype=torch.int64).pin_memory()
    for _ in range(3):
        t0 = time.perf_counter()
        _native.check(L.pnn_matmul_host(nb, es, A.data_ptr(), B.data_ptr(), Cc.data_ptr(), M, K, N))
        print(f"posit({nb},{es}) matmul_host {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
x = torch.empty(1 << 28, dtype=torch.uint8).pin_memory()
d = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(x, non_blocking=True); torch.cuda.synchronize()
    print(f"H2D 256 MiB pinned: {256 / 1024 / (time.perf_counter() - t0):.1f} GiB/s")
    torch.cuda.synchronize(); t0 = time.perf_counter(); x.copy_(d, non_blocking=True); torch.cuda.synchronize()
    print(f"D2H 256 MiB pinned: {256 / 1024 / (time.perf_counter() - t0):.1f} GiB/s")
a = np.ones(1 << 25, np.uint64); b = np.empty(1 << 25, np.uint8)
t0 = time.perf_counter(); np.copyto(b, a, casting="unsafe"); t = time.perf_counter() - t0
print(f"numpy 1-thread narrow 256 MiB -> 32 MiB: {0.25 / t:.1f} GiB/s of input; cpus={os.cpu_count()}")
