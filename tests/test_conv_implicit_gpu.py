"""Implicit-GEMM conv path (TMA tile gathers from digitised activations,
igemm_core.cuh) against the CPU oracle, forced on with pnn_conv_algo(2) so an
ineligible shape fails instead of silently taking the explicit path.  Shapes
are the CIFAR-CNN family (C, F multiples of 32, 3x3 pad 1) plus the edges the
tiling has: partial last tile along N, sub-128-pixel images (several images
per tile), 1x1 taps, valid (pad 0) convs, F not a multiple of the N tile,
128-channel wgrad slots."""
import numpy as np
import pytest
import torch

from conftest import rand_codes
from paper_2105_00053_b200 import ops

pytestmark = pytest.mark.gpu

FORMATS = [(8, 0), (8, 1), (8, 2), (12, 1), (16, 1)]

# (N, C, H, W, F, K, pad, passes that are implicit-eligible)
SHAPES = [
    (2, 32, 8, 8, 32, 3, 1, "fdw"),      # 2 images per 128-row tile
    (3, 32, 8, 8, 64, 3, 1, "fdw"),      # odd N: last tile half out of range
    (2, 64, 16, 16, 32, 3, 1, "fdw"),    # 2 tiles per image; wgrad 2 taps per m-tile
    (1, 32, 32, 32, 32, 3, 1, "fdw"),    # CIFAR conv2 geometry, 8 tiles per image
    (2, 32, 4, 16, 32, 3, 1, "fdw"),     # wide rows: 16-wide K blocks of 2 rows
    (2, 32, 16, 16, 32, 1, 0, "fdw"),    # 1x1 taps
    (2, 32, 10, 10, 32, 3, 0, "fw"),     # valid conv: fwd 8x8 tiles, box reads inside 10x10
    (2, 32, 8, 8, 40, 3, 1, "fw"),       # F = 40: partial N tile / padded dy digits
    (2, 128, 8, 8, 32, 3, 1, "fdw"),     # 128-channel wgrad slot (128B swizzle)
    (2, 3, 32, 32, 32, 3, 1, "fdw"),     # first layer: taps folded into 27 of 32 channels
    (2, 1, 16, 16, 8, 5, 2, "fw"),       # folded 5x5, C = 1 (25 taps), pad 2
    (4, 2, 10, 10, 32, 3, 0, "fw"),      # folded valid conv
    (4, 64, 1, 1, 32, 1, 0, "fd"),       # Linear as 1x1 conv: elementwise digitiser
    (130, 32, 1, 1, 64, 1, 0, "fd"),     # Linear, 128 rows per tile + a partial tile
]


def dev(cfg, a):
    return torch.from_numpy(np.ascontiguousarray(a).astype(ops._cfg(cfg).np_code_dtype)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.int64).astype(np.uint64)


@pytest.fixture
def implicit_only():
    prev = ops.conv_algo(2)
    yield
    ops.conv_algo(prev)


def _algo_for(passes, which):
    return 2 if which in passes else 0


@pytest.mark.parametrize("cfg", FORMATS)
@pytest.mark.parametrize("shape", SHAPES)
def test_implicit_conv_passes(cuda, po, cfg, shape):
    n, es = cfg
    N, Cc, H, W, F, K, p, passes = shape
    rng = np.random.default_rng(N * 7919 + Cc * 31 + H * 7 + F + K + p + n * 3 + es)
    x = rand_codes(rng, n, (N, Cc, H, W))
    w = rand_codes(rng, n, (F, Cc, K, K))
    b = rand_codes(rng, n, (F,))
    prev = ops.conv_algo(_algo_for(passes, "f"))
    try:
        y = host(ops.conv2d(cfg, dev(cfg, x), dev(cfg, w), dev(cfg, b), 1, p))
        y_want = po.conv2d(n, es, x, w, b, 1, p)
        assert (y == y_want).all()
        y_nb = host(ops.conv2d(cfg, dev(cfg, x), dev(cfg, w), None, 1, p))
        assert (y_nb == po.conv2d(n, es, x, w, None, 1, p)).all()
        dy = rand_codes(rng, n, y_want.shape)
        ops.conv_algo(_algo_for(passes, "d"))
        dx = host(ops.conv2d_input_grad(cfg, dev(cfg, dy), dev(cfg, w), x.shape, 1, p))
        assert (dx == po.conv2d_input_grad(n, es, dy, w, x.shape, 1, p)).all()
        ops.conv_algo(_algo_for(passes, "w"))
        dw = host(ops.conv2d_weight_grad(cfg, dev(cfg, dy), dev(cfg, x), w.shape, 1, p))
        assert (dw == po.conv2d_weight_grad(n, es, dy, x, w.shape, 1, p)).all()
    finally:
        ops.conv_algo(prev)


@pytest.mark.parametrize("cfg", FORMATS)
def test_implicit_conv_nar(cuda, po, cfg, implicit_only):
    """NaR reaches exactly the outputs whose terms include it: the fix-up
    kernels rebuild the explicit path's row flags from the digitiser's maps."""
    n, es = cfg
    nar = 1 << (n - 1)
    rng = np.random.default_rng(5 + n + es)
    N, Cc, H, W, F, K, p = 2, 32, 8, 8, 32, 3, 1
    x = rand_codes(rng, n, (N, Cc, H, W))
    w = rand_codes(rng, n, (F, Cc, K, K))
    b = rand_codes(rng, n, (F,))
    x[0, 5, 0, 7] = nar      # corner pixel: only some taps / outputs see it
    w[3, 1, 2, 0] = nar
    b[7] = nar
    y = host(ops.conv2d(cfg, dev(cfg, x), dev(cfg, w), dev(cfg, b), 1, p))
    want = po.conv2d(n, es, x, w, b, 1, p)
    assert (y == want).all()
    assert (want != nar).any()
    dy = rand_codes(rng, n, want.shape)
    dy[1, 4, 7, 7] = nar
    dx = host(ops.conv2d_input_grad(cfg, dev(cfg, dy), dev(cfg, w), x.shape, 1, p))
    want = po.conv2d_input_grad(n, es, dy, w, x.shape, 1, p)
    assert (dx == want).all() and (want != nar).any()
    dw = host(ops.conv2d_weight_grad(cfg, dev(cfg, dy), dev(cfg, x), w.shape, 1, p))
    want = po.conv2d_weight_grad(n, es, dy, x, w.shape, 1, p)
    assert (dw == want).all()
    # NaR only in x (no dy NaR): exactly the taps whose window covers the pixel
    dy2 = rand_codes(rng, n, dy.shape)
    dw2 = host(ops.conv2d_weight_grad(cfg, dev(cfg, dy2), dev(cfg, x), w.shape, 1, p))
    want2 = po.conv2d_weight_grad(n, es, dy2, x, w.shape, 1, p)
    assert (dw2 == want2).all() and (want2 != nar).any()


@pytest.mark.parametrize("cfg", FORMATS)
def test_folded_first_layer_nar(cuda, po, cfg, implicit_only):
    """Tap-folded first layer: NaR rows rebuilt from the folded receptive fields."""
    n, es = cfg
    nar = 1 << (n - 1)
    rng = np.random.default_rng(21 + n + es)
    x = rand_codes(rng, n, (2, 3, 16, 16))
    w = rand_codes(rng, n, (32, 3, 3, 3))
    b = rand_codes(rng, n, (32,))
    x[1, 2, 15, 0] = nar  # corner: only taps reaching it see it
    w[4, 1, 0, 2] = nar
    y = host(ops.conv2d(cfg, dev(cfg, x), dev(cfg, w), dev(cfg, b), 1, 1))
    want = po.conv2d(n, es, x, w, b, 1, 1)
    assert (y == want).all() and (want != nar).any()
    dy = rand_codes(rng, n, want.shape)
    dw = host(ops.conv2d_weight_grad(cfg, dev(cfg, dy), dev(cfg, x), w.shape, 1, 1))
    want = po.conv2d_weight_grad(n, es, dy, x, w.shape, 1, 1)
    assert (dw == want).all() and (want != nar).any()


@pytest.mark.parametrize("cfg", FORMATS)
def test_implicit_linear_nar(cuda, po, cfg, implicit_only):
    n, es = cfg
    nar = 1 << (n - 1)
    rng = np.random.default_rng(11 + n + es)
    x = rand_codes(rng, n, (6, 64, 1, 1))
    w = rand_codes(rng, n, (32, 64, 1, 1))
    b = rand_codes(rng, n, (32,))
    x[2, 17, 0, 0] = nar
    w[5, 3, 0, 0] = nar
    y = host(ops.conv2d(cfg, dev(cfg, x), dev(cfg, w), dev(cfg, b), 1, 0))
    want = po.conv2d(n, es, x, w, b, 1, 0)
    assert (y == want).all() and (want != nar).any()
    dy = rand_codes(rng, n, want.shape)
    dy[4, 9, 0, 0] = nar
    dx = host(ops.conv2d_input_grad(cfg, dev(cfg, dy), dev(cfg, w), x.shape, 1, 0))
    assert (dx == po.conv2d_input_grad(n, es, dy, w, x.shape, 1, 0)).all()


@pytest.mark.parametrize("cfg", [(8, 1), (12, 1), (16, 1)])
def test_implicit_wgrad_long_k_raw_words(cuda, po, cfg, implicit_only):
    """Batch-16 CIFAR conv weight grad (K = 16,384 pixels > the 16,383-term
    int32 chunk of D = 8): split-K partials,
    raw quire words (the data-parallel reduction input) round to the codes."""
    n, es = cfg
    rng = np.random.default_rng(640 + n)
    x = rand_codes(rng, n, (16, 32, 32, 32))
    dy = rand_codes(rng, n, (16, 32, 32, 32))
    want = po.conv2d_weight_grad(n, es, dy, x, (32, 32, 3, 3), 1, 1)
    dw, words, nar = ops.conv2d_weight_grad(cfg, dev(cfg, dy), dev(cfg, x), (32, 32, 3, 3), 1, 1,
                                            raw=True)
    assert (host(dw) == want).all()
    q = ops.quire_round(cfg, words.view(-1, 2))
    assert (host(q).reshape(want.shape) & np.uint64((1 << n) - 1) == want).all()
    assert int(nar.sum()) == 0


def test_ineligible_shape_fails_loudly_when_forced(cuda, implicit_only):
    cfg = (8, 0)
    x = torch.zeros((1, 32, 8, 8), dtype=torch.uint8, device="cuda")
    w = torch.zeros((32, 32, 3, 3), dtype=torch.uint8, device="cuda")
    with pytest.raises(Exception):
        ops.conv2d(cfg, x, w, None, 2, 1)  # stride 2: no implicit tiling


def test_auto_matches_explicit_on_cifar_layer(cuda):
    """Auto (implicit) and explicit paths agree bit for bit on a CIFAR layer."""
    cfg = (12, 1)
    rng = np.random.default_rng(3)
    x = dev(cfg, rand_codes(rng, 12, (16, 32, 32, 32)))
    w = dev(cfg, rand_codes(rng, 12, (64, 32, 3, 3)))
    b = dev(cfg, rand_codes(rng, 12, (64,)))
    dy = dev(cfg, rand_codes(rng, 12, (16, 64, 32, 32)))
    outs = []
    for algo in (1, 0):
        prev = ops.conv_algo(algo)
        try:
            outs.append((host(ops.conv2d(cfg, x, w, b, 1, 1)),
                         host(ops.conv2d_input_grad(cfg, dy, w, x.shape, 1, 1)),
                         host(ops.conv2d_weight_grad(cfg, dy, x, w.shape, 1, 1))))
        finally:
            ops.conv_algo(prev)
    for a, b_ in zip(*outs):
        assert (a == b_).all()
