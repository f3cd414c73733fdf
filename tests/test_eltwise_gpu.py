"""Parity of the device scalar ALU and the elementwise training-step kernels
(convert, ReLU, max-pool, softmax cross-entropy, SGD) with the CPU oracle."""
import numpy as np
import pytest
import torch

from conftest import rand_codes
from paper_2105_00053_b200 import ops

pytestmark = pytest.mark.gpu

FORMATS = [(8, 0), (8, 1), (12, 1), (16, 1)]


def dev(cfg, a):
    return torch.from_numpy(np.ascontiguousarray(a).astype(ops._cfg(cfg).np_code_dtype)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.int64).astype(np.uint64)


def mask(n):
    return np.uint64((1 << n) - 1)


@pytest.mark.parametrize("cfg", [(8, 0), (8, 1), (8, 2)])
def test_scalar_ops_exhaustive_8bit(cuda, po, cfg):
    n, es = cfg
    a = np.repeat(np.arange(256), 256).astype(np.int64)
    b = np.tile(np.arange(256), 256).astype(np.int64)
    for op in range(4):
        got = host(ops.scalar_eval(cfg, op, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())) & mask(n)
        want = po.ew(n, es, op, a.astype(np.uint64), b.astype(np.uint64))
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (op, a[bad[:3]], b[bad[:3]], got[bad[:3]], want[bad[:3]])


@pytest.mark.parametrize("cfg", [(12, 1), (16, 1), (10, 1)])
def test_scalar_ops_random(cuda, po, cfg):
    n, es = cfg
    rng = np.random.default_rng(n)
    a = rng.integers(0, 1 << n, 200000).astype(np.int64)
    b = rng.integers(0, 1 << n, 200000).astype(np.int64)
    for op in range(4):
        got = host(ops.scalar_eval(cfg, op, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())) & mask(n)
        want = po.ew(n, es, op, a.astype(np.uint64), b.astype(np.uint64))
        assert (got == want).all(), op


@pytest.mark.parametrize("cfg", [(10, 2), (12, 2)])
def test_scalar_ops_wide_formats(cuda, po, cfg):
    """The posit(8,2)* optimizer / loss formats (2R > 56: 128-bit images and
    significand products): every op on random pairs plus the corner codes."""
    n, es = cfg
    rng = np.random.default_rng(n * 7 + es)
    corners = np.array([0, 1, 2, 3, (1 << (n - 1)) - 1, (1 << (n - 1)) - 2, 1 << (n - 1),
                        (1 << (n - 1)) + 1, (1 << n) - 1, (1 << n) - 2, 1 << (n - 2)], np.int64)
    a = np.concatenate([rng.integers(0, 1 << n, 300000), np.repeat(corners, corners.size)])
    b = np.concatenate([rng.integers(0, 1 << n, 300000), np.tile(corners, corners.size)])
    a, b = a.astype(np.int64), b.astype(np.int64)
    for op in range(4):
        got = host(ops.scalar_eval(cfg, op, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())) & mask(n)
        want = po.ew(n, es, op, a.astype(np.uint64), b.astype(np.uint64))
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (op, a[bad[:3]], b[bad[:3]], got[bad[:3]], want[bad[:3]])


@pytest.mark.parametrize("cfg", [(8, 0), (8, 1), (12, 1), (16, 1), (10, 2), (12, 2)])
def test_exp_log_all_codes(cuda, po, cfg):
    n, es = cfg
    codes = np.arange(1 << n, dtype=np.int64)
    step = 1 if n <= 12 else 7  # every 7th 16-bit code keeps the oracle loop short
    codes = codes[::step]
    e = host(ops.scalar_eval(cfg, 4, torch.from_numpy(codes).cuda())) & mask(n)
    l = host(ops.scalar_eval(cfg, 5, torch.from_numpy(codes).cuda())) & mask(n)
    r = host(ops.scalar_eval(cfg, 6, torch.from_numpy(codes).cuda())) & mask(n)
    for i, c in enumerate(codes):
        assert int(e[i]) == po.exp(n, es, int(c)), ("exp", int(c))
        assert int(l[i]) == po.log(n, es, int(c)), ("log", int(c))
        assert int(r[i]) == po.round_to_int(n, es, int(c)), ("round_to_int", int(c))


@pytest.mark.parametrize("pair", [((16, 1), (12, 1)), ((12, 1), (8, 1)), ((12, 1), (8, 0)),
                                  ((8, 0), (12, 1)), ((16, 1), (8, 0)), ((8, 1), (16, 1))])
def test_convert_all_codes(cuda, po, golden, pair):
    (sn, se), (dn, de) = pair
    x = np.arange(1 << sn, dtype=np.uint64)
    got = host(ops.convert_tensor(dev((sn, se), x), (sn, se), (dn, de)))
    assert (got == golden[f"convert_{sn}_{se}_{dn}_{de}"]).all()
    assert (got == po.convert_tensor(sn, se, dn, de, x)).all()


@pytest.mark.parametrize("cfg", FORMATS)
def test_relu(cuda, po, cfg):
    n, es = cfg
    rng = np.random.default_rng(1)
    x = rng.integers(0, 1 << n, 5000).astype(np.uint64)  # includes NaR
    assert (host(ops.relu_fwd(cfg, dev(cfg, x))) == po.relu_fwd(n, es, x)).all()
    g = (12, 1)
    dy = rng.integers(0, 1 << 12, 5000).astype(np.uint64)
    assert (host(ops.relu_bwd(cfg, dev(cfg, x), g, dev(g, dy))) == po.relu_bwd(n, es, x, dy)).all()


@pytest.mark.parametrize("pair", [((8, 1), (12, 1)), ((12, 1), (16, 1)), ((16, 1), (8, 0))])
def test_vector_paths_tails_and_unaligned(cuda, po, pair):
    """16-byte vector paths: lengths that are not multiples of 8 (scalar tail)
    and unaligned views (scalar fallback) give the same codes."""
    (sn, se), (dn, de) = pair
    rng = np.random.default_rng(sn + dn)
    x = rng.integers(0, 1 << sn, 5003).astype(np.uint64)
    dy = rng.integers(0, 1 << dn, 5003).astype(np.uint64)
    xt, dyt = dev((sn, se), x), dev((dn, de), dy)
    for sl in (slice(0, 5003), slice(1, 5003), slice(3, 4000)):
        got = host(ops.convert_tensor(xt[sl], (sn, se), (dn, de)))
        assert (got == po.convert_tensor(sn, se, dn, de, x[sl])).all(), sl
        assert (host(ops.relu_fwd((sn, se), xt[sl])) == po.relu_fwd(sn, se, x[sl])).all(), sl
        got = host(ops.relu_bwd((sn, se), xt[sl], (dn, de), dyt[sl]))
        assert (got == po.relu_bwd(sn, se, x[sl], dy[sl])).all(), sl


@pytest.mark.parametrize("cfg", FORMATS)
@pytest.mark.parametrize("geom", [(2, 2), (3, 2), (3, 1), (2, 1)])
def test_maxpool(cuda, po, cfg, geom):
    """Includes overlapping windows (k > stride): the backward accumulates with
    posit adds in output order like maxpool2d_backward (tensor_ops.cpp:665-668)."""
    n, es = cfg
    k, s = geom
    rng = np.random.default_rng(k * 10 + s + n)
    x = rand_codes(rng, n, (2, 3, 9, 8), nar_ok=True)
    x[0, 0, 0:3, 0:3] = x[0, 0, 0, 0]  # ties: first strict max wins
    y, am = ops.maxpool2d(cfg, dev(cfg, x), k, s)
    yw, amw = po.maxpool2d(n, es, x, k, s)
    assert (host(y) == yw).all() and (am.cpu().numpy() == amw).all()
    dy = rand_codes(rng, n, yw.shape)
    dx = ops.maxpool2d_backward(cfg, dev(cfg, dy), am, x.shape, k, s)
    want = po.maxpool2d_backward(n, es, dy, amw, x.shape)
    assert (host(dx) == want).all()
    # reference signature: window-independent scatter
    dx = ops.maxpool2d_backward(cfg, dev(cfg, dy), am, x.shape)
    assert (host(dx) == want).all()


@pytest.mark.parametrize("cfg", FORMATS + [(12, 2)])
@pytest.mark.parametrize("shape", [(1, 1, 5, 8), (3, 7, 33, 17), (1, 1, 1, 1)])
def test_maxpool_backward_scatter_any_argmax(cuda, po, cfg, shape):
    """maxpool2d_backward(dy, argmax, x_shape) for an arbitrary argmax (not
    produced by a window): collisions add in increasing output order
    (tensor_ops.cpp:665-668), untouched targets stay 0, NaR is sticky."""
    n, es = cfg
    rng = np.random.default_rng(n * 7 + es + shape[1])
    n_in = int(np.prod(shape))
    for n_out in (0, 1, 37, 5000):
        am = rng.integers(0, max(1, n_in // 3), n_out).astype(np.int64)
        dy = rand_codes(rng, n, (n_out,), nar_ok=True)
        dx = ops.maxpool2d_backward(cfg, dev(cfg, dy), torch.from_numpy(am).cuda(), shape)
        assert (host(dx).ravel() == po.maxpool2d_backward(n, es, dy, am, shape).ravel()).all(), n_out


def test_maxpool_backward_rejects_bad_window_and_index(cuda):
    """The window-specialised form checks dy against (N, C, OH, OW) instead of
    reading past it (k=3, s=3 on 6x6 has 4 outputs per plane, not 9); the
    scatter rejects indices outside the input."""
    cfg = (8, 0)
    x = torch.randint(0, 255, (1, 2, 6, 6), dtype=torch.uint8).cuda()
    y, am = ops.maxpool2d(cfg, x, 3, 3)
    with pytest.raises(ops._native.PnnInvalidArgument):
        ops.maxpool2d_backward(cfg, y, am, x.shape, 2, 2)
    with pytest.raises(ops._native.PnnInvalidArgument):
        ops.maxpool2d_backward(cfg, y, am + 72, x.shape)
    with pytest.raises(ops._native.PnnInvalidArgument):
        ops.maxpool2d_backward(cfg, y, am - 100, x.shape)


@pytest.mark.parametrize("cfg", [(16, 1), (12, 1), (8, 0), (10, 2), (12, 2)])
def test_softmax_xent(cuda, po, cfg):
    n, es = cfg
    rng = np.random.default_rng(n + 3)
    B, Cn = 64, 10
    z = np.array([[po.from_float64(n, es, v) for v in row] for row in rng.normal(0, 3, (B, Cn))], np.uint64)
    labels = rng.integers(0, Cn, B).astype(np.int32)
    loss, d, rows = ops.softmax_xent(cfg, dev(cfg, z), torch.from_numpy(labels).cuda(), 6)
    lw, dw, rw = po.softmax_xent(n, es, z, labels, 6)
    assert (host(rows) == rw).all()
    assert (host(d) == dw).all()
    assert int(host(loss)[0]) == lw


@pytest.mark.parametrize("fmts", [((16, 1), (16, 1)), ((16, 1), (12, 1))])
def test_sgd_step(cuda, po, fmts):
    (on, oe), (gn, ge) = fmts
    rng = np.random.default_rng(5)
    w = rand_codes(rng, on, (3000,))
    g = rand_codes(rng, gn, (3000,))
    lr = po.from_float64(on, oe, 1.0 / 16)
    m = dev((on, oe), w)
    c1 = torch.empty(3000, dtype=torch.uint8, device="cuda")
    c2 = torch.empty(3000, dtype=torch.uint16, device="cuda")
    ops.sgd_step((on, oe), m, (gn, ge), dev((gn, ge), g), lr, copies=[((8, 0), c1), ((12, 1), c2)])
    want = po.sgd(on, oe, w, gn, ge, g, lr)
    assert (host(m) == want).all()
    assert (host(c1) == po.convert_tensor(on, oe, 8, 0, want)).all()
    assert (host(c2) == po.convert_tensor(on, oe, 12, 1, want)).all()


@pytest.mark.parametrize("cfg", [(16, 1), (10, 2), (8, 2)])
@pytest.mark.parametrize("scale", [0, 3, 10, -2])
def test_softmax_xent_loss_scaled(cuda, po, cfg, scale):
    """Loss scaling (SPEC scale_gradients): dlogits carry 2^s, the loss does not."""
    n, es = cfg
    rng = np.random.default_rng(n + 11 + scale)
    B, Cn = 32, 10
    z = np.array([[po.from_float64(n, es, v) for v in row] for row in rng.normal(0, 3, (B, Cn))], np.uint64)
    labels = rng.integers(0, Cn, B).astype(np.int32)
    loss, d, rows = ops.softmax_xent(cfg, dev(cfg, z), torch.from_numpy(labels).cuda(), 5,
                                     grad_scale_log2=scale)
    lw, dw, rw = po.softmax_xent(n, es, z, labels, 5, scale)
    assert (host(d) == dw).all() and (host(rows) == rw).all() and int(host(loss)[0]) == lw
    l0, _, r0 = po.softmax_xent(n, es, z, labels, 5, 0)
    assert lw == l0 and (rw == r0).all()  # the loss itself is not scaled


@pytest.mark.parametrize("fmts", [((12, 2), (8, 2)), ((16, 1), (12, 1))])
@pytest.mark.parametrize("scale", [0, 4, -3])
def test_sgd_step_scaled(cuda, po, fmts, scale):
    (on, oe), (gn, ge) = fmts
    rng = np.random.default_rng(17 + scale)
    w = rand_codes(rng, on, (5000,))
    g = rand_codes(rng, gn, (5000,))
    lr = po.from_float64(on, oe, 1.0 / 16)
    m = dev((on, oe), w)
    c1 = torch.empty(5000, dtype=torch.uint8, device="cuda")
    ops.sgd_step((on, oe), m, (gn, ge), dev((gn, ge), g), lr, copies=[((8, 2), c1)], grad_scale_log2=scale)
    want = po.sgd(on, oe, w, gn, ge, g, lr, scale)
    assert (host(m) == want).all()
    assert (host(c1) == po.convert_tensor(on, oe, 8, 2, want)).all()


def test_softmax_raw_word_needs_narrow_quire(cuda):
    z = torch.zeros((4, 10), dtype=torch.uint16, device="cuda")
    lab = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(Exception, match="128 bits"):
        ops.softmax_xent((10, 2), z, lab, 2, raw=True)
