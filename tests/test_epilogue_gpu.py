"""The implicit-GEMM epilogue's two 64-bit quire-word roundings -- the integer
leading-one search (q_to_posit_lut) and the FP64-converter variant
(q_to_posit_lut_f64: I2F.F64 toward zero, dropped bits recovered by converting
back) -- agree on every word: powers of two, sticky bits just past the 53-bit
mantissa, ties at every rounding position, wrap-around at W bits, and random
words of every length (posit.cpp:93-132 pack_round is the reference for both)."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2105_00053_b200 import _native

pytestmark = pytest.mark.gpu


def _words(rng):
    w = [0, 1, 2, 3, (1 << 63) - 1, 1 << 62]
    for k in range(64):
        w += [1 << k, (1 << k) - 1, (1 << k) + 1]
        for s in range(1, 12):  # ties / near-ties below the leading one
            if k > s:
                w += [(1 << k) | (1 << (k - s)), (1 << k) | (1 << (k - s)) | 1,
                      (1 << k) | ((1 << (k - s)) - 1)]
    for k in range(53, 64):  # a single bit beyond the FP64 mantissa
        w += [(1 << k) | 1, ((1 << 53) - 1) << (k - 52), (((1 << 53) - 1) << (k - 52)) | 1]
    lens = rng.integers(0, 64, 200000)
    r = rng.integers(0, 1 << 62, 200000, dtype=np.int64).astype(np.uint64) | (np.uint64(1) << np.uint64(62))
    w += list((r >> (np.uint64(63) - lens.astype(np.uint64))).astype(np.uint64))
    a = np.array(w, dtype=np.uint64)
    neg = (np.uint64(0) - a)  # two's complement negatives
    return np.concatenate([a, neg, rng.integers(0, 2 ** 63 - 1, 50000, dtype=np.int64).astype(np.uint64) * np.uint64(2),
                           np.array([1 << 63], dtype=np.uint64)])


@pytest.mark.parametrize("cfg", [(8, 0), (8, 1), (8, 2), (10, 1), (12, 1), (16, 1)])
def test_round64_f64_equals_integer_path(cuda, cfg):
    n, es = cfg
    rng = np.random.default_rng(n * 7 + es)
    q = torch.from_numpy(_words(rng).view(np.int64)).cuda()
    a = torch.zeros(q.numel(), dtype=torch.int32, device="cuda")
    b = torch.ones(q.numel(), dtype=torch.int32, device="cuda")
    lib = _native.lib()
    fn = lib.pnn_internal_round64_check
    fn.restype = C.c_int
    fn.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    _native.check(fn(n, es, q.data_ptr(), q.numel(), a.data_ptr(), b.data_ptr(),
                     torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    bad = (a != b).nonzero()
    assert bad.numel() == 0, [(hex(int(q[i]) & (2 ** 64 - 1)), int(a[i]), int(b[i])) for i in bad[:8, 0].tolist()]
