"""Non-quire (use_quire=false) device kernels vs the oracle: one correctly
rounded posit multiply and add per term in the reference's order
(tensor_ops.cpp:145-164, 232-264, 302-335)."""
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


@pytest.mark.parametrize("cfg", FORMATS)
def test_seq_matmul_and_conv(cuda, po, cfg):
    n, es = cfg
    rng = np.random.default_rng(60 + n)
    A = rand_codes(rng, n, (37, 45), nar_ok=True)
    B = rand_codes(rng, n, (45, 21), nar_ok=True)
    assert (host(ops.matmul(dev(cfg, A), dev(cfg, B), False, cfg=cfg)) == po.matmul_seq(n, es, A, B)).all()
    assert (ops.matmul(A, B, False, cfg=cfg) == po.matmul_seq(n, es, A, B)).all()  # host arrays
    for (N, Cc, H, W, F, K, s, p) in [(2, 3, 9, 8, 4, 3, 1, 1), (2, 1, 12, 12, 3, 5, 1, 0), (1, 2, 9, 7, 3, 3, 2, 1)]:
        x = rand_codes(rng, n, (N, Cc, H, W), nar_ok=True)
        w = rand_codes(rng, n, (F, Cc, K, K))
        b = rand_codes(rng, n, (F,))
        y = host(ops.conv2d(cfg, dev(cfg, x), dev(cfg, w), dev(cfg, b), s, p, use_quire=False))
        assert (y == po.conv2d_seq(n, es, x, w, b, s, p)).all()
        dy = rand_codes(rng, n, y.shape)
        assert (host(ops.conv2d_input_grad(cfg, dev(cfg, dy), dev(cfg, w), x.shape, s, p, use_quire=False)) ==
                po.conv2d_input_grad_seq(n, es, dy, w, x.shape, s, p)).all()
        assert (host(ops.conv2d_weight_grad(cfg, dev(cfg, dy), dev(cfg, x), w.shape, s, p, use_quire=False)) ==
                po.conv2d_weight_grad_seq(n, es, dy, x, w.shape, s, p)).all()
        assert (host(ops.conv2d_bias_grad(cfg, dev(cfg, dy), use_quire=False)) ==
                po.bias_grad_seq(n, es, dy.reshape(N, F, -1))).all()


def test_seq_kat_and_column_sum(cuda, po):
    a = np.array([[po.from_float64(8, 0, 64), 1, po.from_float64(8, 0, -64)]], np.uint64)
    b = np.array([[po.from_float64(8, 0, 1)], [1], [po.from_float64(8, 0, 1)]], np.uint64)
    assert int(host(ops.matmul(dev((8, 0), a), dev((8, 0), b), False, cfg=(8, 0)))[0, 0]) == 0
    rng = np.random.default_rng(2)
    for cfg in FORMATS:
        x = rand_codes(rng, cfg[0], (64, 84))
        assert (host(ops.column_sum(cfg, dev(cfg, x), use_quire=False)) ==
                po.bias_grad_seq(*cfg, x.reshape(64, 84, 1))).all()
