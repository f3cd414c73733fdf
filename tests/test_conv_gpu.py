"""Parity of the conv2d / linear passes (implicit GEMMs on the tcgen05 quire
core, through the C-ABI) with the CPU oracle and the golden reference vectors."""
import numpy as np
import pytest
import torch

from conftest import rand_codes
from paper_2105_00053_b200 import ops

pytestmark = pytest.mark.gpu

FORMATS = [(8, 0), (8, 1), (12, 1), (16, 1)]


def dev(cfg, a):
    cfg = ops._cfg(cfg)
    return torch.from_numpy(np.ascontiguousarray(a).astype(cfg.np_code_dtype)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.uint64)


# (N, C, H, W, F, K, stride, pad): LeNet conv1/conv2, CIFAR-style 3x3 pad 1, strided, 1x1 (Linear)
SHAPES = [(2, 1, 32, 32, 6, 5, 1, 0), (3, 6, 14, 14, 16, 5, 1, 0), (2, 3, 16, 16, 8, 3, 1, 1),
          (2, 4, 9, 7, 5, 3, 2, 1), (2, 3, 11, 10, 4, 4, 3, 2), (5, 40, 1, 1, 12, 1, 1, 0)]


@pytest.mark.parametrize("cfg", FORMATS)
@pytest.mark.parametrize("shape", SHAPES)
def test_conv_passes_random(cuda, po, cfg, shape):
    n, es = cfg
    N, Cc, H, W, F, K, s, p = shape
    rng = np.random.default_rng(N * 1000 + Cc * 100 + H + F + K + s + p + n)
    x = rand_codes(rng, n, (N, Cc, H, W))
    w = rand_codes(rng, n, (F, Cc, K, K))
    b = rand_codes(rng, n, (F,))
    y_want = po.conv2d(n, es, x, w, b, s, p)
    y = host(ops.conv2d(cfg, dev(cfg, x), dev(cfg, w), dev(cfg, b), s, p))
    assert (y == y_want).all()
    y_nb = host(ops.conv2d(cfg, dev(cfg, x), dev(cfg, w), None, s, p))
    assert (y_nb == po.conv2d(n, es, x, w, None, s, p)).all()
    dy = rand_codes(rng, n, y_want.shape)
    dx = host(ops.conv2d_input_grad(cfg, dev(cfg, dy), dev(cfg, w), x.shape, s, p))
    assert (dx == po.conv2d_input_grad(n, es, dy, w, x.shape, s, p)).all()
    dw = host(ops.conv2d_weight_grad(cfg, dev(cfg, dy), dev(cfg, x), w.shape, s, p))
    assert (dw == po.conv2d_weight_grad(n, es, dy, x, w.shape, s, p)).all()
    db = host(ops.conv2d_bias_grad(cfg, dev(cfg, dy)))
    assert (db == po.conv2d_bias_grad(n, es, dy)).all()


@pytest.mark.parametrize("cfg", FORMATS)
def test_conv_nar_semantics(cuda, po, cfg):
    """NaR poisons exactly the outputs whose term set contains it
    (quire.hpp:55): strided/edge input-grad taps must not leak a NaR weight."""
    n, es = cfg
    nar = 1 << (n - 1)
    rng = np.random.default_rng(77 + n)
    for (N, Cc, H, W, F, K, s, p) in [(2, 3, 9, 9, 4, 3, 2, 0), (1, 2, 14, 14, 3, 5, 1, 0),
                                      (2, 2, 8, 8, 3, 3, 1, 1)]:
        x = rand_codes(rng, n, (N, Cc, H, W))
        w = rand_codes(rng, n, (F, Cc, K, K))
        b = rand_codes(rng, n, (F,))
        x[0, 1, 2, 3] = nar
        w[1, 0, K - 1, K - 1] = nar
        b[2] = nar
        y = host(ops.conv2d(cfg, dev(cfg, x), dev(cfg, w), dev(cfg, b), s, p))
        assert (y == po.conv2d(n, es, x, w, b, s, p)).all()
        dy = rand_codes(rng, n, y.shape)
        dy[-1, 0, 0, 1] = nar
        dx = host(ops.conv2d_input_grad(cfg, dev(cfg, dy), dev(cfg, w), x.shape, s, p))
        want = po.conv2d_input_grad(n, es, dy, w, x.shape, s, p)
        assert (dx == want).all()
        assert (want != nar).any()  # the NaR weight must not poison every output
        dw = host(ops.conv2d_weight_grad(cfg, dev(cfg, dy), dev(cfg, x), w.shape, s, p))
        assert (dw == po.conv2d_weight_grad(n, es, dy, x, w.shape, s, p)).all()
        db = host(ops.conv2d_bias_grad(cfg, dev(cfg, dy)))
        assert (db == po.conv2d_bias_grad(n, es, dy)).all()


def test_conv_golden_vectors(cuda, golden):
    keys = sorted(k[:-2] for k in golden if k.startswith("conv_") and k.endswith("_y"))
    for key in keys:
        parts = key.split("_")
        cfg = (int(parts[1]), int(parts[2]))
        s, p = (int(v) for v in parts[5][1:].split("p"))
        x, w, b, dy = (golden[key + t] for t in ("_x", "_w", "_b", "_dy"))
        assert (host(ops.conv2d(cfg, dev(cfg, x), dev(cfg, w), dev(cfg, b), s, p)) == golden[key + "_y"]).all(), key
        assert (host(ops.conv2d_input_grad(cfg, dev(cfg, dy), dev(cfg, w), x.shape, s, p)) ==
                golden[key + "_dx"]).all(), key
        assert (host(ops.conv2d_weight_grad(cfg, dev(cfg, dy), dev(cfg, x), w.shape, s, p)) ==
                golden[key + "_dw"]).all(), key
        assert (host(ops.conv2d_bias_grad(cfg, dev(cfg, dy))) == golden[key + "_db"]).all(), key


@pytest.mark.parametrize("cfg", [(12, 1), (16, 1)])
def test_weight_grad_long_k_and_raw_words(cuda, po, cfg):
    """Batch-64 LeNet conv1 weight grad (K = 50,176 terms per weight): split-K
    partials must be exact; the raw quire words must round to the same codes."""
    n, es = cfg
    rng = np.random.default_rng(64)
    x = rand_codes(rng, n, (64, 1, 32, 32))
    dy = rand_codes(rng, n, (64, 6, 28, 28))
    want = po.conv2d_weight_grad(n, es, dy, x, (6, 1, 5, 5), 1, 0)
    dw, words, nar = ops.conv2d_weight_grad(cfg, dev(cfg, dy), dev(cfg, x), (6, 1, 5, 5), 1, 0, raw=True)
    assert (host(dw) == want).all()
    q = ops.quire_round(cfg, words.view(-1, 2))
    assert (host(q).reshape(want.shape) & np.uint64((1 << n) - 1) == want).all()
    assert int(nar.sum()) == 0


def test_column_sum(cuda, po):
    rng = np.random.default_rng(9)
    for cfg in FORMATS:
        n, es = cfg
        x = rand_codes(rng, n, (64, 84))
        assert (host(ops.column_sum(cfg, dev(cfg, x))) == po.column_sum(n, es, x)).all()
