"""The operand pack paths of the quire GEMM (quire_gemm_core.cuh pack_direct_kernel):
16-byte row loads, 4-byte row-group loads of column-major operands (2 rows of
16-bit codes / 4 rows of 8-bit codes per load), their scalar fallbacks for
misaligned bases and odd leading dimensions, NaR rows attributed per row inside a
row group, and every code of a format through the digitiser once.  Bit-exact
against the oracle's matmul (tensor_ops.cpp:166-185)."""
import numpy as np
import pytest
import torch

from conftest import rand_codes
from paper_2105_00053_b200 import ops

pytestmark = pytest.mark.gpu

FORMATS = [(8, 0), (8, 1), (12, 1), (16, 1)]


def dev_offset(cfg, a, off):
    """a's codes on the device in a buffer whose base is `off` elements past an
    allocation boundary (a contiguous view: data_ptr misaligned by off codes)."""
    cfg = ops._cfg(cfg)
    flat = torch.zeros(a.size + off, dtype=cfg.code_dtype, device="cuda")
    flat[off:] = torch.from_numpy(np.ascontiguousarray(a).astype(cfg.np_code_dtype)).cuda().reshape(-1)
    return flat[off:].view(*a.shape)


@pytest.mark.parametrize("cfg", FORMATS)
@pytest.mark.parametrize("offs", [(0, 0), (1, 0), (0, 1), (3, 2)])
@pytest.mark.parametrize("shape", [(64, 128, 64), (40, 72, 52), (9, 33, 10)])
def test_pack_alignment_paths(cuda, po, cfg, offs, shape):
    n, es = cfg
    m, k, nn = shape
    rng = np.random.default_rng(n * 100 + m + offs[0] * 7 + offs[1])
    A, B = rand_codes(rng, n, (m, k)), rand_codes(rng, n, (k, nn))
    got = ops.quire_gemm(cfg, dev_offset(cfg, A, offs[0]), dev_offset(cfg, B, offs[1]))
    torch.cuda.synchronize()
    assert (got.cpu().numpy().astype(np.uint64) == po.matmul(n, es, A, B)).all()


@pytest.mark.parametrize("cfg", FORMATS)
def test_pack_nar_rows_within_a_row_group(cuda, po, cfg):
    """NaR codes in neighbouring columns of B (one 4-byte load holds 2 or 4 of
    them) and in neighbouring rows of A flag exactly their own outputs."""
    n, es = cfg
    nar = 1 << (n - 1)
    rng = np.random.default_rng(n + 17)
    A, B = rand_codes(rng, n, (48, 64)), rand_codes(rng, n, (64, 64))
    B[5, 9] = nar    # column 9 only (columns 8..11 share a row group)
    B[40, 30] = nar  # column 30 (group 28..31), another k-block
    A[17, 3] = nar
    A[18, 63] = nar
    got = ops.quire_gemm(cfg, dev_offset(cfg, A, 0), dev_offset(cfg, B, 0)).cpu().numpy().astype(np.uint64)
    want = po.matmul(n, es, A, B)
    assert (got == want).all()
    nar_cols = sorted(set(np.argwhere(got[0] == nar).ravel().tolist()))
    assert nar_cols == [9, 30]
    assert (got[17] == nar).all() and (got[18] == nar).all() and not (got[16] == nar).all()


@pytest.mark.parametrize("cfg", [(8, 0), (8, 1), (12, 1), (16, 1)])
def test_every_code_through_the_digitiser(cuda, po, cfg):
    """A holds every code of the format once, B = the identity in posit 1.0:
    round(quire(a * 1)) == a for every non-NaR a, NaR rows stay NaR -- the
    branch-free decode (decode_x_bf) and the digit tables on every code."""
    n, es = cfg
    codes = np.arange(1 << n, dtype=np.uint64)
    K = 64
    A = codes.reshape(-1, K)
    one = po.from_float64(n, es, 1.0)
    B = np.zeros((K, K), np.uint64)
    B[np.arange(K), np.arange(K)] = one
    got = ops.quire_gemm(cfg, dev_offset(cfg, A, 0), dev_offset(cfg, B, 0)).cpu().numpy().astype(np.uint64)
    nar = 1 << (n - 1)
    want = A.copy()
    want[(A == nar).any(axis=1)] = nar  # the NaR code poisons its whole row
    assert (got == want).all()
