"""Device time of the config-1 posit(16,1) GEMM as one launch vs four 1024-row
panels (CUDA events, L2 flushed before each measurement)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2105_00053_b200 import ops
for (n, es) in [(8, 0), (16, 1)]:
    cfg = ops.PositConfig(n, es)
    rng = np.random.default_rng(0)
    A = torch.from_numpy(rng.integers(0, (1 << n) - 1, (4096, 4096)).astype(cfg.np_code_dtype)).cuda()
    B = torch.from_numpy(rng.integers(0, (1 << n) - 1, (4096, 4096)).astype(cfg.np_code_dtype)).cuda()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device='cuda')
    def t(fn, reps=5):
        best = 1e9
        for _ in range(reps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        return best
    full = t(lambda: ops.quire_gemm(cfg, A, B))
    for P in (2, 4, 8):
        r = 4096 // P
        pan = t(lambda: [ops.quire_gemm(cfg, A[i * r:(i + 1) * r], B) for i in range(P)])
        print(f"posit({n},{es}) full {full:.3f} ms, {P} panels {pan:.3f} ms", flush=True)
