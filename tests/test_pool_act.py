"""avg-pool (tensor_ops.cpp:672-720) and tanh / sigmoid
(posit_math.cpp:109-130).  CPU: the oracle restatement pinned to the
reference library; GPU: the device kernels pinned to the oracle."""
import numpy as np
import pytest
import torch

from conftest import rand_codes

FORMATS = [(8, 0), (8, 1), (8, 2), (12, 1), (16, 1)]


@pytest.mark.parametrize("cfg", FORMATS)
def test_oracle_avgpool_tanh_sigmoid_vs_reference(po, ref, cfg):
    n, es = cfg
    rng = np.random.default_rng(n * 3 + es)
    for c in rng.integers(0, 1 << n, 800):
        assert po.tanh(n, es, c) == ref.tanh(n, es, c), c
        assert po.sigmoid(n, es, c) == ref.sigmoid(n, es, c), c
    x = rand_codes(rng, n, (2, 3, 8, 9), nar_ok=True)
    r = po.from_float64(n, es, 0.25)
    for k, s in [(2, 2), (3, 1), (2, 1)]:
        for q in (False, True):
            assert (po.avgpool2d(n, es, x, k, s, q, r) == ref.avgpool2d(n, es, x, k, s, q, r)).all()
        OH, OW = (8 - k) // s + 1, (9 - k) // s + 1
        dy = rand_codes(rng, n, (2, 3, OH, OW))
        assert (po.avgpool2d_backward(n, es, dy, k, s, (2, 3, 8, 9), r) ==
                ref.avgpool2d_backward(n, es, dy, k, s, (2, 3, 8, 9), r)).all()


def test_kat_avgpool_constant_and_exact_mean(po):
    # test_tensor.cpp:188-210: mean of a constant is the constant; {1,2,3,4} -> 2.5 in (8,2)
    f = (8, 2)
    c = np.full((1, 1, 4, 4), po.from_float64(*f, 0.75), np.uint64)
    r = po.from_float64(*f, 0.25)
    assert all(po.to_float64(*f, int(v)) == 0.75 for v in po.avgpool2d(*f, c, 2, 2, True, r).ravel())
    x = np.array([po.from_float64(*f, v) for v in (1, 2, 3, 4)], np.uint64).reshape(1, 1, 2, 2)
    assert po.to_float64(*f, int(po.avgpool2d(*f, x, 2, 2, True, r)[0, 0, 0, 0])) == 2.5


def _dev(cfg, a):
    from paper_2105_00053_b200 import ops

    return torch.from_numpy(np.ascontiguousarray(a).astype(ops._cfg(cfg).np_code_dtype)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.int64).astype(np.uint64)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(8, 0), (8, 1), (12, 1), (16, 1)])
def test_gpu_tanh_sigmoid_all_codes(cuda, po, cfg):
    from paper_2105_00053_b200 import ops

    n, es = cfg
    codes = np.arange(1 << n, dtype=np.int64)[:: 1 if n <= 12 else 5]
    t = _host(ops.scalar_eval(cfg, 10, torch.from_numpy(codes).cuda())) & np.uint64((1 << n) - 1)
    s = _host(ops.scalar_eval(cfg, 11, torch.from_numpy(codes).cuda())) & np.uint64((1 << n) - 1)
    for i, c in enumerate(codes):
        assert int(t[i]) == po.tanh(n, es, int(c)), ("tanh", int(c))
        assert int(s[i]) == po.sigmoid(n, es, int(c)), ("sigmoid", int(c))


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(8, 0), (8, 1), (12, 1), (16, 1)])
def test_gpu_avgpool(cuda, po, cfg):
    from paper_2105_00053_b200 import ops

    n, es = cfg
    rng = np.random.default_rng(n)
    x = rand_codes(rng, n, (2, 3, 10, 9), nar_ok=True)
    r = po.from_float64(n, es, 0.25)
    for k, s in [(2, 2), (3, 1), (2, 1)]:
        for q in (False, True):
            got = _host(ops.avgpool2d(cfg, _dev(cfg, x), k, s, q, r))
            assert (got == po.avgpool2d(n, es, x, k, s, q, r)).all(), (k, s, q)
        OH, OW = (10 - k) // s + 1, (9 - k) // s + 1
        dy = rand_codes(rng, n, (2, 3, OH, OW))
        got = _host(ops.avgpool2d_backward(cfg, _dev(cfg, dy), k, s, x.shape, r))
        assert (got == po.avgpool2d_backward(n, es, dy, k, s, x.shape, r)).all(), (k, s)
