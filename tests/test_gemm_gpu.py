"""Parity of the tcgen05 quire GEMM (through the C-ABI) with the CPU oracle.

Bit-exact: every output code must equal the reference's matmul(a, b,
use_quire=true) (tensor_ops.cpp:166-185) on the same codes.
"""
import numpy as np
import pytest
import torch

from conftest import rand_codes
from paper_2105_00053_b200 import _native, ops

pytestmark = pytest.mark.gpu

FORMATS = [(8, 0), (8, 1), (8, 2), (12, 1), (16, 1)]
EXTRA = [(6, 0), (10, 1), (14, 1), (4, 0)]


def to_dev(cfg, a):
    cfg = ops._cfg(cfg)
    return torch.from_numpy(np.ascontiguousarray(a).astype(cfg.np_code_dtype)).cuda()


def gemm(cfg, A, B, **kw):
    out = ops.quire_gemm(cfg, to_dev(cfg, A), to_dev(cfg, B), **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.uint64)


def x_of(po, n, es, c):
    ls, sig, neg, nar = po.decode_fixed(n, es, c)
    if nar:
        return None
    R = (n - 2) << es
    v = sig << (ls + R) if sig else 0
    return -v if neg else v


@pytest.mark.parametrize("cfg", FORMATS + EXTRA)
def test_decode_exhaustive(cuda, po, cfg):
    n, es = cfg
    codes = torch.arange(1 << n, dtype=torch.int32, device=cuda)
    X, nar = ops.decode_x(cfg, codes)
    X, nar = X.cpu().numpy(), nar.cpu().numpy()
    for c in range(1 << n):
        want = x_of(po, n, es, c)
        if want is None:
            assert nar[c] == 1, c
        else:
            assert nar[c] == 0 and int(X[c]) == want, (c, int(X[c]), want)


@pytest.mark.parametrize("cfg", FORMATS + [(16, 2), (32, 2), (12, 2)])
def test_pack_round_random(cuda, po, cfg):
    n, es = cfg
    R = (n - 2) << es
    rng = np.random.default_rng(n * 7 + es)
    cnt = 20000
    neg = rng.integers(0, 2, cnt).astype(np.int32)
    scale = rng.integers(-R - 4, R + 4, cnt).astype(np.int32)
    sig = (rng.integers(0, 1 << 63, cnt, dtype=np.uint64) | np.uint64(1 << 63))
    # exercise exact-tie and short significands too
    sig[::7] = np.uint64(1 << 63)
    sig[1::7] = np.uint64((1 << 63) | (1 << 62))
    sticky = rng.integers(0, 2, cnt).astype(np.int32)
    got = ops.pack_round(cfg, torch.from_numpy(neg).cuda(), torch.from_numpy(scale).cuda(),
                         torch.from_numpy(sig.view(np.int64)).cuda(), torch.from_numpy(sticky).cuda())
    got = got.cpu().numpy().astype(np.uint64) & np.uint64((1 << n) - 1)
    for i in range(cnt):
        want = po.pack_round(n, es, int(neg[i]), int(scale[i]), int(sig[i]), int(sticky[i]))
        assert int(got[i]) == want, (i, int(neg[i]), int(scale[i]), hex(int(sig[i])), int(sticky[i]))


def _py_quire_round(po, n, es, q):
    """Quire::to_posit (quire.cpp:105-146) in Python over the oracle's pack_round."""
    R = (n - 2) << es
    W = 4 * R + n
    q &= (1 << W) - 1
    neg = (q >> (W - 1)) & 1
    mag = ((1 << W) - q) & ((1 << W) - 1) if neg else q
    if mag == 0:
        return 0
    top = mag.bit_length() - 1
    if top >= 63:
        sig, sticky = mag >> (top - 63), int(mag & ((1 << (top - 63)) - 1) != 0)
    else:
        sig, sticky = mag << (63 - top), 0
    return po.pack_round(n, es, neg, top - 2 * R, sig, sticky)


@pytest.mark.parametrize("cfg", FORMATS)
def test_quire_round_random(cuda, po, cfg):
    n, es = cfg
    R = (n - 2) << es
    W = 4 * R + n
    rng = np.random.default_rng(99 + n)
    qs = []
    for i in range(6000):
        bits = int(rng.integers(1, W + 1))
        v = int(rng.integers(0, 1 << 62)) | (int(rng.integers(0, 1 << 62)) << 62) | (int(rng.integers(0, 16)) << 124)
        v &= (1 << bits) - 1
        if i % 3 == 0:
            v = ((1 << W) - v) & ((1 << W) - 1)  # negative
        qs.append(v)
    qs += [0, 1, (1 << W) - 1, 1 << (W - 1), (1 << (W - 1)) - 1, 1 << (2 * R), (1 << W) - (1 << (2 * R))]
    words = np.array([[q & ((1 << 64) - 1), q >> 64] for q in qs], dtype=np.uint64)
    got = ops.quire_round(cfg, torch.from_numpy(words.view(np.int64)).cuda()).cpu().numpy()
    for q, g in zip(qs, got):
        assert (int(g) & ((1 << n) - 1)) == _py_quire_round(po, n, es, q), hex(q)


SHAPES = [(1, 1, 1), (5, 7, 6), (33, 57, 29), (128, 128, 128), (130, 300, 257), (256, 1000, 96),
          (7, 4100, 5)]


@pytest.mark.parametrize("cfg", FORMATS)
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_parity_random(cuda, po, cfg, shape):
    n, es = cfg
    m, k, nn = shape
    rng = np.random.default_rng(m * 31 + k * 7 + nn + n * 1000 + es)
    A = rand_codes(rng, n, (m, k))
    B = rand_codes(rng, n, (k, nn))
    want = po.matmul(n, es, A, B)
    got = gemm(cfg, A, B)
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:4].tolist()}"


@pytest.mark.parametrize("cfg", EXTRA)
def test_gemm_parity_other_formats(cuda, po, cfg):
    n, es = cfg
    rng = np.random.default_rng(5)
    A = rand_codes(rng, n, (70, 90))
    B = rand_codes(rng, n, (90, 40))
    assert (gemm(cfg, A, B) == po.matmul(n, es, A, B)).all()


def test_gemm_golden_vectors(cuda, golden):
    keys = sorted(k[:-2] for k in golden if k.startswith("gemm") and k.endswith("_C"))
    for key in keys:
        parts = key.split("_")
        cfg = (int(parts[1]), int(parts[2]))
        got = gemm(cfg, golden[key + "_A"], golden[key + "_B"])
        assert (got == golden[key + "_C"]).all(), key


@pytest.mark.parametrize("cfg", FORMATS)
def test_gemm_nar_propagation(cuda, po, cfg):
    n, es = cfg
    nar = 1 << (n - 1)
    rng = np.random.default_rng(3)
    A = rand_codes(rng, n, (40, 64))
    B = rand_codes(rng, n, (64, 50))
    A[3, 10] = nar
    A[5, :] = 0
    A[5, 7] = nar  # NaR times zero partners is still NaR (quire.hpp:55-56)
    B[:, 9] = 0
    B[2, 9] = nar
    got = gemm(cfg, A, B)
    want = po.matmul(n, es, A, B)
    assert (got == want).all()
    assert (got[3, :] == nar).all() and (got[5, :] == nar).all() and (got[:, 9] == nar).all()


def test_gemm_kats(cuda, po):
    one80 = po.from_float64(8, 0, 1.0)
    # test_tensor.cpp:52-62: 1x16 ones . 16x1 ones -> 16
    got = gemm((8, 0), np.full((1, 16), one80, np.uint64), np.full((16, 1), one80, np.uint64))
    assert po.to_float64(8, 0, int(got[0, 0])) == 16.0
    # test_quire.cpp:46-58: 127 ones saturate to maxpos
    got = gemm((8, 0), np.full((1, 127), one80, np.uint64), np.full((127, 1), one80, np.uint64))
    assert int(got[0, 0]) == 0x7F
    # test_tensor.cpp:64-74: cancellation keeps minpos^2 -> minpos
    a = np.array([[po.from_float64(8, 0, 64), 1, po.from_float64(8, 0, -64)]], np.uint64)
    b = np.array([[one80], [1], [one80]], np.uint64)
    assert int(gemm((8, 0), a, b)[0, 0]) == 1
    # identity
    rng = np.random.default_rng(11)
    x = rand_codes(rng, 8, (4, 4))
    eye = np.zeros((4, 4), np.uint64)
    np.fill_diagonal(eye, po.from_float64(8, 2, 1.0))
    assert (gemm((8, 2), eye, x) == x).all()
    # K = 0 -> zeros (tensor_ops.cpp:467)
    z = ops.quire_gemm((8, 0), torch.zeros((3, 0), dtype=torch.uint8, device="cuda"),
                       torch.zeros((0, 4), dtype=torch.uint8, device="cuda"))
    assert int(z.sum()) == 0


@pytest.mark.parametrize("cfg", FORMATS)
def test_splitk_is_bit_identical(cuda, cfg):
    n, es = cfg
    rng = np.random.default_rng(17)
    A = rand_codes(rng, n, (150, 700), nar_ok=True)
    B = rand_codes(rng, n, (700, 90))
    base = gemm(cfg, A, B)
    for kbs in (1, 2, 5):
        assert (gemm(cfg, A, B, max_kblocks=kbs) == base).all(), kbs


def test_int32_partials_wrap_like_the_quire(cuda, po):
    """posit(8,0): quire W=32 wraps mod 2^32 (quire.cpp:52).  K*(-2)*(-2)
    = 2^19 -> quire integer 2^31 -> negative -> saturates to -maxpos.  A
    saturating int32 MMA would give +maxpos instead."""
    m2 = po.from_float64(8, 0, -2.0)
    K = 131072
    A = np.full((1, K), m2, np.uint64)
    B = np.full((K, 1), m2, np.uint64)
    want = po.matmul(8, 0, A, B)
    assert int(want[0, 0]) == 0x81
    assert int(gemm((8, 0), A, B)[0, 0]) == 0x81


def test_long_k_chunks_exact_wide_formats(cuda, po):
    """(16,1) with K beyond one int32-exact chunk (16352) -> automatic split-K."""
    rng = np.random.default_rng(23)
    for cfg in [(16, 1), (12, 1)]:
        n, es = cfg
        K = 40000
        A = rand_codes(rng, n, (3, K))
        B = rand_codes(rng, n, (K, 5))
        # bias the magnitudes up so group sums are large
        assert (gemm(cfg, A, B) == po.matmul(n, es, A, B)).all()


@pytest.mark.parametrize("cfg", [(8, 0), (16, 1)])
def test_config1_full_size_sampled_rows(cuda, po, cfg):
    """BASELINE config 1 (4096^3): exact equality on 6 full rows (24,576
    outputs, 100M oracle MACs) plus structural properties on the rest."""
    n, es = cfg
    rng = np.random.default_rng(4096 + n)
    M = N = K = 4096
    nar = 1 << (n - 1)
    codes = np.array([c for c in range(1 << n) if c != nar], np.uint64)
    A = codes[rng.integers(0, len(codes), (M, K))]
    B = codes[rng.integers(0, len(codes), (K, N))]
    got = gemm(cfg, A, B)
    rows = rng.choice(M, 6, replace=False)
    want = po.matmul(n, es, A[rows], B)
    assert (got[rows] == want).all()
    assert not (got == nar).any()  # no NaR inputs -> no NaR outputs
    # permuting K (both operands) never changes an exact quire
    perm = rng.permutation(K)
    got2 = gemm(cfg, A[:, perm][:256], B[perm])
    assert (got2 == got[:256]).all()


def test_matmul_host_entry(cuda, po):
    rng = np.random.default_rng(8)
    for cfg in [(8, 0), (16, 1)]:
        n, es = cfg
        A = rand_codes(rng, n, (77, 300))
        B = rand_codes(rng, n, (300, 45))
        got = ops.matmul(A, B, True, cfg=cfg)
        assert got.dtype == np.uint64
        assert (got == po.matmul(n, es, A, B)).all()


def test_errors_raise(cuda):
    a = torch.zeros((4, 5), dtype=torch.uint8, device="cuda")
    b = torch.zeros((6, 3), dtype=torch.uint8, device="cuda")
    with pytest.raises(_native.PnnInvalidArgument):
        ops.quire_gemm((8, 0), a, b)
    with pytest.raises(_native.PnnError):
        ops.quire_gemm((16, 2), torch.zeros((4, 5), dtype=torch.uint16, device="cuda"),
                       torch.zeros((5, 3), dtype=torch.uint16, device="cuda"))


def test_cta_pair_kernel_parity(cuda, po):
    """The opt-in CTA-pair (tcgen05 cta_group::2) kernel is bit-identical too,
    including an odd number of m-tiles (zero-padded follower tile)."""
    import subprocess
    import sys

    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, '.');"
        "from paper_2105_00053_b200 import ops;"
        "from oracle.bind import Restatement; po = Restatement();"
        "rng = np.random.default_rng(5)\n"
        "for cfg in [(8, 0), (8, 1), (12, 1), (16, 1)]:\n"
        "    n, es = cfg\n"
        "    A = rng.integers(0, 1 << n, (3 * 128 + 5, 300)).astype(np.uint64); A[A == 1 << (n - 1)] = 0\n"
        "    B = rng.integers(0, 1 << n, (300, 70)).astype(np.uint64); B[B == 1 << (n - 1)] = 0\n"
        "    dt = ops.PositConfig(*cfg).np_code_dtype\n"
        "    got = ops.quire_gemm(cfg, torch.from_numpy(A.astype(dt)).cuda(), torch.from_numpy(B.astype(dt)).cuda())\n"
        "    assert (got.cpu().numpy().astype(np.uint64) == po.matmul(n, es, A, B)).all(), cfg\n"
        "print('pair ok')\n")
    import os
    env = dict(os.environ, PNN_B200_PAIR="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "pair ok" in r.stdout, r.stderr[-2000:]


_HOST_SPLIT_CODE = r"""
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
"""


@pytest.mark.parametrize("env", [{}, {"PNN_HOST_DMA_IN": "1", "PNN_HOST_DMA_OUT": "1", "PNN_HOST_PANELS": "3"},
                                 {"PNN_HOST_DMA_IN": "0", "PNN_HOST_DMA_OUT": "0", "PNN_HOST_PANELS": "1",
                                  "PNN_HOST_THREADS": "3"},
                                 {"PNN_HOST_DMA_IN": "0.77", "PNN_HOST_DMA_OUT": "0.13", "PNN_HOST_PANELS": "5"}])
def test_matmul_host_dma_split(cuda, po, env):
    """pnn_matmul_host with pinned Tensor storage: rows moved raw by the copy
    engines (device-narrowed / -widened) and rows narrowed / widened by host
    threads give the device GEMM's result for every split, panel count and
    thread count; pageable buffers take the host-thread path."""
    import os
    import subprocess
    import sys

    r = subprocess.run([sys.executable, "-c", _HOST_SPLIT_CODE], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, **env),
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "split ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("cfg,limit", [((8, 1), 2.0 ** 11), ((12, 1), 8.0), ((16, 1), 8.0)])
@pytest.mark.parametrize("small", [True, False])
def test_reduced_digit_gemm_variants(cuda, po, cfg, limit, small):
    """Device-selected reduced-digit variants of the explicit quire GEMM
    (posit(8,1) in 3 of 4 digits, (12,1) in 3 of 6, (16,1) in 4 of 8), forced
    on for small problems: operands within the reduced digits take the reduced
    kernel, a single wide value the full one -- both equal the oracle."""
    n, es = cfg
    lib = _native.lib()
    prev = lib.pnn_variant_min_work(0)
    try:
        rng = np.random.default_rng(n * 10 + small)
        codes = np.arange(1 << n, dtype=np.uint64)
        vals = np.array([po.to_float64(n, es, int(c)) for c in codes])
        ok = codes[(np.abs(vals) < limit) & np.isfinite(vals)] if small else codes[codes != (1 << (n - 1))]
        A = rng.choice(ok, (300, 200)).astype(np.uint64)
        B = rng.choice(ok, (200, 140)).astype(np.uint64)
        A[7, 3] = 1 << (n - 1)  # a NaR row
        got = gemm(cfg, A, B)
        assert (got == po.matmul(n, es, A, B)).all()
    finally:
        lib.pnn_variant_min_work(prev)
