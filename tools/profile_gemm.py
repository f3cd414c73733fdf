"""Short driver for ncu: a few warm-up GEMMs then one profiled (8,0) and one
(16,1) config-1 quire GEMM (4096^3) through the C-ABI."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import M, N, K, gen_codes  # noqa: E402
from paper_2105_00053_b200 import ops  # noqa: E402

fmts = [(8, 0), (16, 1)] if len(sys.argv) < 2 else [tuple(int(v) for v in sys.argv[1].split(","))]
for fmt in fmts:
    cfg = ops.PositConfig(*fmt)
    A, B = gen_codes(fmt, seed=2105 + fmt[0])
    dA = torch.from_numpy(A.astype(cfg.np_code_dtype)).cuda()
    dB = torch.from_numpy(B.astype(cfg.np_code_dtype)).cuda()
    for _ in range(2):
        ops.quire_gemm(cfg, dA, dB)
    torch.cuda.synchronize()
print("profile driver done")
