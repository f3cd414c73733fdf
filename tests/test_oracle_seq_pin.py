"""Pin the oracle's non-quire sequential kernels (use_quire=false) to the
unmodified reference library (no GPU) and to the reference's own KAT
(test_tensor.cpp:64-74: the sequential path loses minpos^2 -> 0)."""
import numpy as np
import pytest

from conftest import rand_codes

FORMATS = [(8, 0), (8, 1), (8, 2), (12, 1), (16, 1)]


def test_seq_kat_cancellation(po):
    a = np.array([[po.from_float64(8, 0, 64), 1, po.from_float64(8, 0, -64)]], np.uint64)
    b = np.array([[po.from_float64(8, 0, 1)], [1], [po.from_float64(8, 0, 1)]], np.uint64)
    assert int(po.matmul_seq(8, 0, a, b)[0, 0]) == 0
    assert int(po.matmul(8, 0, a, b)[0, 0]) == 1


@pytest.mark.parametrize("cfg", FORMATS)
def test_seq_kernels_vs_reference(po, ref, cfg):
    n, es = cfg
    rng = np.random.default_rng(40 + n + es)
    A = rand_codes(rng, n, (13, 29), nar_ok=True)
    B = rand_codes(rng, n, (29, 11), nar_ok=True)
    assert (po.matmul_seq(n, es, A, B) == ref.matmul(n, es, A, B, use_quire=False)).all()
    x = rand_codes(rng, n, (2, 3, 9, 8), nar_ok=True)
    w = rand_codes(rng, n, (4, 3, 3, 3))
    b = rand_codes(rng, n, (4,))
    for s, p in [(1, 1), (2, 0), (1, 0)]:
        y = po.conv2d_seq(n, es, x, w, b, s, p)
        assert (y == ref.conv2d(n, es, x, w, b, s, p, use_quire=False)).all()
        dy = rand_codes(rng, n, y.shape)
        assert (po.conv2d_input_grad_seq(n, es, dy, w, x.shape, s, p) ==
                ref.conv2d_input_grad(n, es, dy, w, x.shape, s, p, use_quire=False)).all()
        assert (po.conv2d_weight_grad_seq(n, es, dy, x, w.shape, s, p) ==
                ref.conv2d_weight_grad(n, es, dy, x, w.shape, s, p, use_quire=False)).all()
        N, F, OH, OW = dy.shape
        assert (po.bias_grad_seq(n, es, dy.reshape(N, F, OH * OW)) ==
                ref.conv2d_bias_grad(n, es, dy, use_quire=False)).all()
    xs = rand_codes(rng, n, (9, 13))
    assert (po.bias_grad_seq(n, es, xs.reshape(9, 13, 1)) == ref.column_sum(n, es, xs, use_quire=False)).all()
