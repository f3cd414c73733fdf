"""Pin the CPU oracle (no GPU).

1. The reference's own known-answer tests (proj/tests/test_quire.cpp,
   test_tensor.cpp, test_posit.cpp), re-asserted against our plain-C
   restatement (oracle/posit_oracle.c).
2. The committed golden fixtures (tests/golden/reference_vectors.npz, made by
   tests/golden/make_golden.py from the unmodified reference).
3. The reference library itself (oracle/_ref/libpnn_ref.so) on random inputs,
   and the reference's own unit-test binary (43 doctest cases).
"""
import os
import subprocess

import numpy as np
import pytest

from conftest import rand_codes

P80, P81, P82, P121, P161 = (8, 0), (8, 1), (8, 2), (12, 1), (16, 1)
FORMATS = [P80, P81, P82, P121, P161]


def f64(lib, cfg, x):
    return lib.from_float64(*cfg, x)


# ---------------------------------------------------------------- 1. KATs


def test_kat_quire_sums_of_ones(po):
    # test_quire.cpp:46-58
    one = f64(po, P80, 1.0)
    q = po.quire(*P80)
    for _ in range(16):
        q.add_product(one, one)
    assert po.to_float64(*P80, q.to_posit()) == 16.0
    q.clear()
    for _ in range(127):
        q.add_product(one, one)
    assert q.to_posit() == 0x7F  # saturates to maxpos = 64
    q2 = po.quire(*P82)
    q2.add_posit(f64(po, P82, 2.0))
    assert q2.to_posit() == f64(po, P82, 2.0)


def test_kat_quire_nar_sticky(po):
    # test_quire.cpp:32-44
    q = po.quire(*P80)
    assert q.to_posit() == 0
    q.add_product(0x80, f64(po, P80, 1.0))
    assert q.to_posit() == 0x80
    q.add_product(f64(po, P80, 1.0), f64(po, P80, 1.0))
    assert q.to_posit() == 0x80
    q.clear()
    assert q.to_posit() == 0


def test_kat_quire_cancellation(po):
    # test_quire.cpp:71-83: 64 + minpos^2 - 64 -> minpos (quire) vs 0 (sequential)
    q = po.quire(*P80)
    q.add_posit(f64(po, P80, 64))
    q.add_product(1, 1)
    q.add_posit(f64(po, P80, -64))
    assert q.to_posit() == 1
    seq = po.op(*P80, 0, f64(po, P80, 64), po.op(*P80, 2, 1, 1))
    seq = po.op(*P80, 0, seq, f64(po, P80, -64))
    assert seq == 0


def test_kat_quire_sub_product(po):
    # test_quire.cpp:85-94
    q = po.quire(*P82)
    q.add_product(f64(po, P82, 3), f64(po, P82, 5))
    q.sub_product(f64(po, P82, 3), f64(po, P82, 5))
    assert q.to_posit() == 0
    q.clear()
    q.sub_product(f64(po, P82, 2), f64(po, P82, 4))
    assert po.to_float64(*P82, q.to_posit()) == -8.0


def test_kat_quire_two_is_0x60(po):
    # test_quire.cpp:150-154
    q = po.quire(*P80)
    q.add_product(f64(po, P80, 1), f64(po, P80, 2))
    assert q.to_posit() == 0x60


def test_kat_quire_widths(po):
    # test_quire.cpp:136-142 / test_posit.cpp:264-279 (Table 1)
    from oracle.bind import Restatement  # noqa: F401

    lib = po.lib
    assert lib.po_quire_bits(8, 0) == 32
    assert lib.po_quire_bits(16, 1) == 128
    assert lib.po_quire_bits(32, 2) == 512
    assert lib.po_quire_bits(64, 3) == 2048
    assert lib.po_quire_bits(8, 2) == 104
    assert lib.po_max_scale(8, 0) == 6 and lib.po_max_scale(16, 1) == 28


def test_kat_matmul_ones_and_identity(po):
    # test_tensor.cpp:52-62
    one = f64(po, P80, 1.0)
    A = np.full((1, 16), one, np.uint64)
    B = np.full((16, 1), one, np.uint64)
    assert po.to_float64(*P80, int(po.matmul(*P80, A, B)[0, 0])) == 16.0
    rng = np.random.default_rng(11)
    a = rand_codes(rng, 8, (4, 4))
    eye = np.zeros((4, 4), np.uint64)
    np.fill_diagonal(eye, f64(po, P82, 1.0))
    assert (po.matmul(*P82, eye, a) == a).all()


def test_kat_matmul_cancellation(po):
    # test_tensor.cpp:64-74
    a = np.array([[f64(po, P80, 64), 1, f64(po, P80, -64)]], np.uint64)
    b = np.array([[f64(po, P80, 1)], [1], [f64(po, P80, 1)]], np.uint64)
    assert int(po.matmul(*P80, a, b)[0, 0]) == 1


def test_kat_conv_all_ones(po):
    # test_tensor.cpp:127-146: 5x5 all-ones over 8x8 all-ones -> 25 -> rounds to 24
    one = f64(po, P80, 1.0)
    x = np.full((1, 1, 8, 8), one, np.uint64)
    w = np.full((1, 1, 5, 5), one, np.uint64)
    y = po.conv2d(*P80, x, w, None, 1, 0)
    assert y.shape == (1, 1, 4, 4)
    assert all(po.to_float64(*P80, int(c)) == 24.0 for c in y.ravel())


def test_kat_maxpool(po):
    # test_tensor.cpp:188-210
    x = np.array([f64(po, P82, v) for v in (1, 2, 3, 4)], np.uint64).reshape(1, 1, 2, 2)
    y, am = po.maxpool2d(*P82, x, 2, 2)
    assert po.to_float64(*P82, int(y.ravel()[0])) == 4.0 and am.ravel()[0] == 3
    dy = np.array([f64(po, P82, 1.0)], np.uint64)
    dx = po.maxpool2d_backward(*P82, dy, am, (1, 1, 2, 2)).ravel()
    assert po.to_float64(*P82, int(dx[3])) == 1.0 and dx[0] == 0


def test_kat_scalar_basics(po):
    # test_posit.cpp:24-75
    assert f64(po, P80, 1.0) == 0x40
    assert f64(po, P80, 128.0) == 0x7F
    assert f64(po, P80, -1e9) == 0x81
    assert f64(po, P161, 2.0 ** -28) == 1
    assert f64(po, P161, 1e-300) == 1
    assert po.to_float64(*P80, 0x7F) == 64.0
    two = po.op(*P80, 0, 0x40, 0x40)
    assert two == 0x60
    assert po.op(*P80, 0, 0x7F, 0x7F) == 0x7F
    assert po.op(*P80, 2, 0x80, two) == 0x80
    assert po.op(*P80, 3, two, 0) == 0x80
    assert po.op(*P80, 3, 0, two) == 0


def test_kat_convert(po):
    # test_posit.cpp:180-221
    assert po.convert(16, 1, 8, 0, 0x7FFF) == 0x7F
    assert po.convert(12, 2, 8, 2, 1) == 1
    assert po.convert(16, 1, 8, 0, 0x8000) == 0x80
    assert po.convert(16, 1, 8, 0, 0) == 0
    for b in range(256):
        assert po.convert(12, 2, 8, 2, po.convert(8, 2, 12, 2, b)) == b


def test_kat_round_to_int(po):
    # test_posit.cpp:306-318
    cfg = (12, 2)

    def ri(x):
        return po.to_int64(*cfg, po.round_to_int(*cfg, f64(po, cfg, x)))

    assert [ri(v) for v in (0.4, 0.5, 0.75, 1.5, 2.5, -3.5, 17.0, -0.25)] == [0, 0, 1, 2, 2, -4, 17, 0]


def test_kat_exp_log_identities(po):
    # test_posit.cpp:326-342 (the exp/log subset the CE loss uses)
    for cfg in [P82, P121, P161]:
        assert po.to_float64(*cfg, po.exp(*cfg, 0)) == 1.0
        nar = 1 << (cfg[0] - 1)
        assert po.log(*cfg, 0) == nar
        assert po.log(*cfg, f64(po, cfg, -1.0)) == nar
        assert po.exp(*cfg, nar) == nar
        assert po.to_float64(*cfg, po.log(*cfg, f64(po, cfg, 1.0))) == 0.0


# ------------------------------------------------------------ 2. golden


def test_golden_gemm(po, golden):
    keys = sorted(k[:-2] for k in golden if k.startswith("gemm") and k.endswith("_C"))
    assert len(keys) >= 20
    for key in keys:
        parts = key.split("_")
        n, es = int(parts[1]), int(parts[2])
        got = po.matmul(n, es, golden[key + "_A"], golden[key + "_B"])
        assert (got == golden[key + "_C"]).all(), key


def test_golden_conv_family(po, golden):
    keys = sorted(k[:-2] for k in golden if k.startswith("conv_") and k.endswith("_y"))
    assert len(keys) >= 15
    for key in keys:
        parts = key.split("_")
        n, es = int(parts[1]), int(parts[2])
        s, p = (int(v) for v in parts[5][1:].split("p"))
        x, w, b = golden[key + "_x"], golden[key + "_w"], golden[key + "_b"]
        dy = golden[key + "_dy"]
        assert (po.conv2d(n, es, x, w, b, s, p) == golden[key + "_y"]).all(), key
        assert (po.conv2d_input_grad(n, es, dy, w, x.shape, s, p) == golden[key + "_dx"]).all(), key
        assert (po.conv2d_weight_grad(n, es, dy, x, w.shape, s, p) == golden[key + "_dw"]).all(), key
        assert (po.conv2d_bias_grad(n, es, dy) == golden[key + "_db"]).all(), key


def test_golden_convert_exhaustive(po, golden):
    for key in [k for k in golden if k.startswith("convert_")]:
        sn, se, dn, de = (int(v) for v in key.split("_")[1:])
        x = np.arange(1 << sn, dtype=np.uint64)
        assert (po.convert_tensor(sn, se, dn, de, x) == golden[key]).all(), key


# --------------------------------------------------- 3. the reference itself


def test_reference_unit_suite_passes():
    from oracle import bind

    if not os.path.exists(bind.REF_UNIT_TESTS):
        pytest.skip("reference unit tests not built on this host")
    r = subprocess.run([bind.REF_UNIT_TESTS], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "43 passed | 0 failed" in r.stdout


@pytest.mark.parametrize("cfg", FORMATS + [(10, 1), (6, 0), (16, 2)])
def test_decode_exhaustive_vs_reference(po, ref, cfg):
    n, es = cfg
    for c in range(1 << n):
        assert po.decode_fixed(n, es, c) == ref.decode_fixed(n, es, c), c


@pytest.mark.parametrize("cfg", FORMATS)
def test_scalar_ops_random_vs_reference(po, ref, cfg):
    n, es = cfg
    rng = np.random.default_rng(n * 10 + es)
    for _ in range(3000):
        a, b, op = int(rng.integers(1 << n)), int(rng.integers(1 << n)), int(rng.integers(4))
        assert po.op(n, es, op, a, b) == ref.op(n, es, op, a, b), (op, a, b)
    for _ in range(3000):
        neg, sc = int(rng.integers(2)), int(rng.integers(-70, 70))
        sig, st = int(rng.integers(0, 1 << 63)) | (1 << 63), int(rng.integers(2))
        assert po.pack_round(n, es, neg, sc, sig, st) == ref.pack_round(n, es, neg, sc, sig, st)
    for _ in range(200):
        a = int(rng.integers(1 << n))
        assert po.exp(n, es, a) == ref.exp(n, es, a), a
        assert po.log(n, es, a) == ref.log(n, es, a), a


@pytest.mark.parametrize("cfg", FORMATS)
def test_tensor_ops_random_vs_reference(po, ref, cfg):
    n, es = cfg
    rng = np.random.default_rng(7 + n + es)
    A = rand_codes(rng, n, (23, 41), nar_ok=True)
    B = rand_codes(rng, n, (41, 17), nar_ok=True)
    assert (po.matmul(n, es, A, B) == ref.matmul(n, es, A, B)).all()
    x = rand_codes(rng, n, (2, 3, 10, 9), nar_ok=True)
    w = rand_codes(rng, n, (5, 3, 3, 3))
    for s, p in [(1, 1), (2, 0)]:
        y = po.conv2d(n, es, x, w, None, s, p)
        assert (y == ref.conv2d(n, es, x, w, None, s, p)).all()
        dy = rand_codes(rng, n, y.shape, nar_ok=True)
        assert (po.conv2d_input_grad(n, es, dy, w, x.shape, s, p) ==
                ref.conv2d_input_grad(n, es, dy, w, x.shape, s, p)).all()
        assert (po.conv2d_weight_grad(n, es, dy, x, w.shape, s, p) ==
                ref.conv2d_weight_grad(n, es, dy, x, w.shape, s, p)).all()
    xs = rand_codes(rng, n, (9, 13))
    assert (po.column_sum(n, es, xs) == ref.column_sum(n, es, xs)).all()
    y1, a1 = po.maxpool2d(n, es, x, 2, 2)
    y2, a2 = ref.maxpool2d(n, es, x, 2, 2)
    assert (y1 == y2).all() and (a1 == a2).all()
    dy = rand_codes(rng, n, y1.shape)
    assert (po.maxpool2d_backward(n, es, dy, a1, x.shape) ==
            ref.maxpool2d_backward(n, es, dy, a2, x.shape)).all()
