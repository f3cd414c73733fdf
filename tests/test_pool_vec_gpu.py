"""2x2 / stride-2 pooling of the training layers: forward without argmax and
the backward that recomputes the first strict max from x
(pnn_maxpool2d_bwd_x) equal the reference-shaped argmax pair
(maxpool2d / maxpool2d_backward, tensor_ops.cpp:620-670), which
test_eltwise_gpu pins to the oracle -- with ties (low-entropy codes) and NaR."""
import numpy as np
import pytest
import torch

from conftest import rand_codes
from paper_2105_00053_b200 import ops

pytestmark = pytest.mark.gpu


def dev(cfg, a):
    return torch.from_numpy(np.ascontiguousarray(a).astype(ops._cfg(cfg).np_code_dtype)).cuda()


@pytest.mark.parametrize("xf,gf", [((8, 1), (12, 1)), ((8, 0), (8, 0)), ((12, 1), (12, 1)),
                                   ((16, 1), (16, 1)), ((12, 1), (8, 1))])
@pytest.mark.parametrize("shape", [(2, 3, 8, 16), (4, 32, 32, 32), (1, 5, 16, 32)])
@pytest.mark.parametrize("ties", [False, True])
def test_pool_recompute_equals_argmax(cuda, xf, gf, shape, ties):
    rng = np.random.default_rng(hash((xf, gf, shape, ties)) & 0xFFFF)
    xa = rand_codes(rng, xf[0], shape, nar_ok=True)
    if ties:  # few distinct values: many equal maxima, NaR windows
        xa = rng.choice(np.array([0, 1, 2, 1 << (xf[0] - 1), (1 << xf[0]) - 1], np.uint64), shape)
    x = dev(xf, xa)
    N, C, H, W = shape
    wpt = 8 if xf[0] <= 8 else 4
    if W % (2 * wpt):
        assert ops.maxpool2d_noidx(xf, x, 2, 2) is None
        return
    y = ops.maxpool2d_noidx(xf, x, 2, 2)
    y_ref, am = ops.maxpool2d(xf, x, 2, 2)
    assert torch.equal(y, y_ref)
    dy = dev(gf, rand_codes(rng, gf[0], (N, C, H // 2, W // 2), nar_ok=True))
    dx = ops.maxpool2d_backward_x(xf, x, gf, dy, 2, 2)
    dx_ref = ops.maxpool2d_backward(gf, dy, am, shape, 2, 2)
    assert torch.equal(dx, dx_ref)


@pytest.mark.parametrize("opt,grad,copies", [((16, 1), (12, 1), [(8, 1), (12, 1)]),
                                             ((16, 1), (16, 1), []),
                                             ((12, 2), (8, 2), [(8, 2)]),
                                             ((16, 1), (8, 0), [(8, 0)]),
                                             ((16, 1), (12, 1), [(8, 1), (8, 0)]),
                                             ((16, 1), (16, 1), [(12, 1), (16, 1)])])
@pytest.mark.parametrize("scale", [0, 1])
def test_sgd_multi_equals_per_tensor(cuda, opt, grad, copies, scale):
    """The whole-model optimizer launch == pnn_sgd_step_scaled per tensor."""
    rng = np.random.default_rng(5)
    sizes = [150, 6, 2400, 16, 48000, 120, 10081, 84, 1, 10]
    lr = (1 << (opt[0] - 2)) >> 2  # a positive code below 1.0
    masters = [dev(opt, rand_codes(rng, opt[0], (n,), nar_ok=True)) for n in sizes]
    grads = [dev(grad, rand_codes(rng, grad[0], (n,), nar_ok=True)) for n in sizes]
    ref_m = [m.clone() for m in masters]
    ref_c = [tuple(torch.zeros(n, dtype=ops._cfg(c).code_dtype, device="cuda") for c in copies) for n in sizes]
    got_c = [tuple(torch.zeros(n, dtype=ops._cfg(c).code_dtype, device="cuda") for c in copies) for n in sizes]
    for m, g, cs in zip(ref_m, grads, ref_c):
        ops.sgd_step(opt, m, grad, g, lr, list(zip(copies, cs)), grad_scale_log2=scale)
    ops.sgd_step_multi(opt, grad, lr, masters, grads, copies, got_c, grad_scale_log2=scale)
    for a, b in zip(masters, ref_m):
        assert torch.equal(a, b)
    for a, b in zip(got_c, ref_c):
        for x, y in zip(a, b):
            assert torch.equal(x, y)


@pytest.mark.parametrize("cfg", [(8, 0), (8, 1), (12, 1), (10, 1)])
@pytest.mark.parametrize("shape", [(64, 32, 32, 32), (7, 64, 16, 16), (3, 5, 8, 16), (1, 3, 4, 4)])
def test_bias_grad_single_launch_vs_oracle(cuda, po, cfg, shape):
    """conv2d_bias_grad (tensor_ops.cpp:605-618) through the one-launch
    shared-table kernel (and the general path for rows that are not 16-byte
    multiples), NaR included, raw words too."""
    rng = np.random.default_rng(hash((cfg, shape)) & 0xFFFF)
    dy = rand_codes(rng, cfg[0], shape, nar_ok=True)
    if shape[0] > 3:
        dy[dy == (1 << (cfg[0] - 1))] = 0
        dy[1, 2, 0, 3] = 1 << (cfg[0] - 1)
    want = po.conv2d_bias_grad(cfg[0], cfg[1], dy)
    got = ops.conv2d_bias_grad(cfg, dev(cfg, dy))
    torch.cuda.synchronize()
    assert (got.cpu().numpy().astype(np.uint64) == want).all()
    db, words, nar = ops.conv2d_bias_grad(cfg, dev(cfg, dy), raw=True)
    assert torch.equal(db, got)


@pytest.mark.parametrize("cfg,gcfg", [((12, 1), (8, 1)), ((8, 0), (8, 0)), ((12, 1), (12, 1)), ((8, 1), (8, 1))])
@pytest.mark.parametrize("shape", [(64, 32, 32, 32), (7, 64, 16, 16), (3, 5, 4, 4)])
def test_bias_grad_gated(cuda, cfg, gcfg, shape):
    """bias grad of relu_bwd(gate, dy) without materialising it == the two-step path."""
    rng = np.random.default_rng(hash((cfg, gcfg, shape)) & 0xFFFF)
    dy = dev(cfg, rand_codes(rng, cfg[0], shape, nar_ok=True))
    gate = dev(gcfg, rand_codes(rng, gcfg[0], shape, nar_ok=True))
    got = ops.conv2d_bias_grad_gated(cfg, dy, gcfg, gate)
    want = ops.conv2d_bias_grad(cfg, ops.relu_bwd(gcfg, gate, cfg, dy))
    if shape[2] * shape[3] % (16 if cfg[0] <= 8 else 8) or (cfg[0] <= 8 and gcfg[0] > 8):
        assert got is None
        return
    assert torch.equal(got, want)
    g2 = ops.conv2d_bias_grad_gated(cfg, dy, gcfg, gate, raw=True)
    w2 = ops.conv2d_bias_grad(cfg, ops.relu_bwd(gcfg, gate, cfg, dy), raw=True)
    assert all(torch.equal(a, b) for a, b in zip(g2, w2))


@pytest.mark.parametrize("opt,grad,copies", [((16, 1), (12, 1), [(8, 1), (12, 1)]),
                                             ((12, 1), (8, 0), [(8, 0)]),
                                             ((16, 1), (16, 1), [(8, 0), (16, 1)])])
def test_sgd_table_path_exhaustive_master_codes(cuda, opt, grad, copies):
    """The table-driven SGD launch (m = lr * convert(g) by table, w - m exact on
    integer images, copies by table) == the scalar-op SGD for every master code
    against a spread of gradient codes (incl. NaR, 0, extremes) and several lr."""
    rng = np.random.default_rng(17)
    n_o = 1 << opt[0]
    gsel = np.concatenate([[0, 1, (1 << grad[0]) - 1, 1 << (grad[0] - 1), (1 << (grad[0] - 1)) - 1,
                            (1 << (grad[0] - 1)) + 1], rng.integers(0, 1 << grad[0], 10)])
    w = np.tile(np.arange(n_o, dtype=np.uint64), len(gsel))
    g = np.repeat(gsel.astype(np.uint64), n_o)
    one = 1 << (opt[0] - 2)
    for lr in (one >> 4, one, rng.integers(1, 1 << (opt[0] - 1))):
        ms = [dev(opt, w[:len(w) // 2]), dev(opt, w[len(w) // 2:])]
        gs = [dev(grad, g[:len(g) // 2]), dev(grad, g[len(g) // 2:])]
        ref_m = [m.clone() for m in ms]
        ref_c = [tuple(torch.zeros(m.numel(), dtype=ops._cfg(c).code_dtype, device="cuda") for c in copies)
                 for m in ms]
        got_c = [tuple(torch.zeros(m.numel(), dtype=ops._cfg(c).code_dtype, device="cuda") for c in copies)
                 for m in ms]
        for m, gg, cs in zip(ref_m, gs, ref_c):
            ops.sgd_step(opt, m, grad, gg, int(lr), list(zip(copies, cs)))
        ops.sgd_step_multi(opt, grad, int(lr), ms, gs, copies, got_c)
        for a, b in zip(ms, ref_m):
            assert torch.equal(a, b), lr
        for a, b in zip(got_c, ref_c):
            for x, y in zip(a, b):
                assert torch.equal(x, y), lr
