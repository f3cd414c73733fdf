"""ctypes bindings for the two CPU oracles (TEST INFRASTRUCTURE ONLY).

* ``Restatement`` -> oracle/_build/libposit_oracle.so (our plain-C restatement)
* ``Reference``   -> oracle/_ref/libpnn_ref.so (the unmodified reference library
  built from /root/reference by oracle/Makefile, plus our C-ABI shim)

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) import this module.  The product package
(paper_2105_00053_b200/) never does.

All tensors are numpy uint64 arrays of posit codes (one code per element, the
reference's own Tensor storage, tensor.hpp:10-14).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "_build", "libposit_oracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libpnn_ref.so")
REF_UNIT_TESTS = os.path.join(HERE, "_ref", "ref_unit_tests")

_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
i64 = C.c_int64


def build(reference: bool = True) -> None:
    """Compile the restatement (always) and the reference (when its sources exist)."""
    targets = ["restatement"]
    if reference and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    if a.dtype == np.int64:
        return a.ctypes.data_as(_i64p)
    assert a.dtype == np.uint64, a.dtype
    return a.ctypes.data_as(_u64p)


def _codes(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


class _Base:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run oracle/Makefile)")
        self.lib = C.CDLL(path)
        self.path = path
        L, p = self.lib, self.prefix
        self._f = lambda name: getattr(L, p + name)
        for name, res, args in [
            ("pack_round", C.c_uint64, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int]),
            ("convert", C.c_uint64, [C.c_int] * 4 + [C.c_uint64]),
            ("scalar_op", C.c_uint64, [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64]),
            ("compare", C.c_int, [C.c_int, C.c_int, C.c_uint64, C.c_uint64]),
            ("from_float64", C.c_uint64, [C.c_int, C.c_int, C.c_double]),
            ("to_float64", C.c_double, [C.c_int, C.c_int, C.c_uint64]),
            ("ldexp", C.c_uint64, [C.c_int, C.c_int, C.c_uint64, C.c_int]),
            ("round_to_int", C.c_uint64, [C.c_int, C.c_int, C.c_uint64]),
            ("to_int64", C.c_int64, [C.c_int, C.c_int, C.c_uint64]),
            ("from_int64", C.c_uint64, [C.c_int, C.c_int, C.c_int64]),
            ("exp", C.c_uint64, [C.c_int, C.c_int, C.c_uint64]),
            ("log", C.c_uint64, [C.c_int, C.c_int, C.c_uint64]),
            ("tanh", C.c_uint64, [C.c_int, C.c_int, C.c_uint64]),
            ("sigmoid", C.c_uint64, [C.c_int, C.c_int, C.c_uint64]),
            ("sqrt", C.c_uint64, [C.c_int, C.c_int, C.c_uint64]),
            ("quire_new", C.c_void_p, [C.c_int, C.c_int]),
            ("quire_free", None, [C.c_void_p]),
            ("quire_clear", None, [C.c_void_p]),
            ("quire_add_posit", None, [C.c_void_p, C.c_uint64]),
            ("quire_add_product", None, [C.c_void_p, C.c_uint64, C.c_uint64]),
            ("quire_sub_product", None, [C.c_void_p, C.c_uint64, C.c_uint64]),
            ("quire_to_posit", C.c_uint64, [C.c_void_p]),
        ]:
            fn = self._f(name)
            fn.restype = res
            fn.argtypes = args

    # -- scalar ---------------------------------------------------------
    def pack_round(self, n, es, neg, scale, sig, sticky):
        return self._f("pack_round")(n, es, int(neg), int(scale), int(sig), int(sticky))

    def convert(self, sn, se, dn, de, code):
        return self._f("convert")(sn, se, dn, de, int(code))

    def op(self, n, es, op, a, b):
        return self._f("scalar_op")(n, es, op, int(a), int(b))

    def compare(self, n, es, a, b):
        return self._f("compare")(n, es, int(a), int(b))

    def from_float64(self, n, es, x):
        return self._f("from_float64")(n, es, float(x))

    def to_float64(self, n, es, code):
        return self._f("to_float64")(n, es, int(code))

    def ldexp(self, n, es, code, k):
        return self._f("ldexp")(n, es, int(code), int(k))

    def round_to_int(self, n, es, code):
        return self._f("round_to_int")(n, es, int(code))

    def to_int64(self, n, es, code):
        return self._f("to_int64")(n, es, int(code))

    def from_int64(self, n, es, v):
        return self._f("from_int64")(n, es, int(v))

    def exp(self, n, es, code):
        return self._f("exp")(n, es, int(code))

    def log(self, n, es, code):
        return self._f("log")(n, es, int(code))

    def tanh(self, n, es, code):
        return self._f("tanh")(n, es, int(code))

    def sigmoid(self, n, es, code):
        return self._f("sigmoid")(n, es, int(code))

    def sqrt(self, n, es, code):
        return self._f("sqrt")(n, es, int(code))

    def avgpool2d(self, n, es, x, k, stride, use_quire, recip):
        x = _codes(x)
        N, Cc, H, W = x.shape
        OH, OW = (H - k) // stride + 1, (W - k) // stride + 1
        y = np.zeros((N, Cc, OH, OW), np.uint64)
        rc = self._f("avgpool2d")(n, es, _p(x), i64(N), i64(Cc), i64(H), i64(W), k, stride, int(use_quire),
                                  C.c_uint64(int(recip)), _p(y))
        if rc:
            raise ValueError("avgpool2d rejected its arguments")
        return y

    def avgpool2d_backward(self, n, es, dy, k, stride, x_shape, recip):
        dy = _codes(dy)
        N, Cc, H, W = x_shape
        dx = np.zeros(tuple(x_shape), np.uint64)
        rc = self._f("avgpool2d_backward")(n, es, _p(dy), i64(N), i64(Cc), i64(H), i64(W), k, stride,
                                           C.c_uint64(int(recip)), _p(dx))
        if rc:
            raise ValueError("avgpool2d_backward rejected its arguments")
        return dx

    def quire(self, n, es):
        return _Quire(self, n, es)

    def fused_dot(self, n, es, a, b):
        q = self.quire(n, es)
        for x, y in zip(a, b):
            q.add_product(x, y)
        return q.to_posit()


class _Quire:
    def __init__(self, lib: _Base, n: int, es: int):
        self.lib = lib
        self.h = lib._f("quire_new")(n, es)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib._f("quire_free")(self.h)
            self.h = None

    def clear(self):
        self.lib._f("quire_clear")(self.h)

    def add_posit(self, a):
        self.lib._f("quire_add_posit")(self.h, int(a))

    def add_product(self, a, b):
        self.lib._f("quire_add_product")(self.h, int(a), int(b))

    def sub_product(self, a, b):
        self.lib._f("quire_sub_product")(self.h, int(a), int(b))

    def to_posit(self):
        return self.lib._f("quire_to_posit")(self.h)


class Restatement(_Base):
    """Our plain-C restatement (oracle/posit_oracle.c)."""

    prefix = "po_"

    def __init__(self, path: str = RESTATEMENT_SO):
        super().__init__(path)

    def _chk(self, rc, what):
        if rc != 0:
            raise ValueError(f"oracle {what} rejected its arguments")

    def decode_fixed(self, n, es, code):
        ls, sg, ng, nr = C.c_int32(), C.c_uint32(), C.c_uint8(), C.c_uint8()
        self.lib.po_decode_fixed(n, es, C.c_uint64(int(code)), C.byref(ls), C.byref(sg),
                                 C.byref(ng), C.byref(nr))
        return ls.value, sg.value, ng.value, nr.value

    def matmul(self, n, es, A, B):
        A, B = _codes(A), _codes(B)
        m, k = A.shape
        k2, nn = B.shape
        assert k == k2
        Cm = np.zeros((m, nn), np.uint64)
        self._chk(self.lib.po_matmul(n, es, _p(A), _p(B), _p(Cm), i64(m), i64(k), i64(nn)), "matmul")
        return Cm

    def conv2d(self, n, es, x, w, bias, stride, pad):
        x, w = _codes(x), _codes(w)
        N, Cc, H, W = x.shape
        F, C2, KH, KW = w.shape
        OH, OW = (H + 2 * pad - KH) // stride + 1, (W + 2 * pad - KW) // stride + 1
        y = np.zeros((N, F, OH, OW), np.uint64)
        b = _codes(bias) if bias is not None else None
        self._chk(self.lib.po_conv2d(n, es, _p(x), i64(N), i64(Cc), i64(H), i64(W), _p(w), i64(F),
                                     i64(KH), i64(KW), _p(b), stride, pad, _p(y)), "conv2d")
        return y

    def conv2d_input_grad(self, n, es, dy, w, x_shape, stride, pad):
        dy, w = _codes(dy), _codes(w)
        N, F, OH, OW = dy.shape
        _, Cc, KH, KW = w.shape
        H, W = x_shape[2], x_shape[3]
        dx = np.zeros((N, Cc, H, W), np.uint64)
        self._chk(self.lib.po_conv2d_input_grad(n, es, _p(dy), i64(N), i64(F), i64(OH), i64(OW),
                                                _p(w), i64(Cc), i64(KH), i64(KW), i64(H), i64(W),
                                                stride, pad, _p(dx)), "conv2d_input_grad")
        return dx

    def conv2d_weight_grad(self, n, es, dy, x, w_shape, stride, pad):
        dy, x = _codes(dy), _codes(x)
        N, F, OH, OW = dy.shape
        _, Cc, H, W = x.shape
        KH, KW = w_shape[2], w_shape[3]
        dw = np.zeros((F, Cc, KH, KW), np.uint64)
        self._chk(self.lib.po_conv2d_weight_grad(n, es, _p(dy), i64(N), i64(F), i64(OH), i64(OW),
                                                 _p(x), i64(Cc), i64(H), i64(W), i64(KH), i64(KW),
                                                 stride, pad, _p(dw)), "conv2d_weight_grad")
        return dw

    def conv2d_bias_grad(self, n, es, dy):
        dy = _codes(dy)
        N, F, OH, OW = dy.shape
        db = np.zeros((F,), np.uint64)
        self._chk(self.lib.po_conv2d_bias_grad(n, es, _p(dy), i64(N), i64(F), i64(OH), i64(OW),
                                               _p(db)), "conv2d_bias_grad")
        return db

    def column_sum(self, n, es, x):
        x = _codes(x)
        B, N = x.shape
        out = np.zeros((N,), np.uint64)
        self._chk(self.lib.po_column_sum(n, es, _p(x), i64(B), i64(N), _p(out)), "column_sum")
        return out

    def maxpool2d(self, n, es, x, k, stride):
        x = _codes(x)
        N, Cc, H, W = x.shape
        OH, OW = (H - k) // stride + 1, (W - k) // stride + 1
        y = np.zeros((N, Cc, OH, OW), np.uint64)
        am = np.zeros((N, Cc, OH, OW), np.int64)
        self._chk(self.lib.po_maxpool2d(n, es, _p(x), i64(N), i64(Cc), i64(H), i64(W), k, stride,
                                        _p(y), _p(am)), "maxpool2d")
        return y, am

    def maxpool2d_backward(self, n, es, dy, argmax, x_shape):
        dy = _codes(dy).ravel()
        am = np.ascontiguousarray(np.asarray(argmax, np.int64)).ravel()
        nx = int(np.prod(x_shape))
        dx = np.zeros((nx,), np.uint64)
        self._chk(self.lib.po_maxpool2d_backward(n, es, _p(dy), i64(dy.size), _p(am), i64(nx),
                                                 _p(dx)), "maxpool2d_backward")
        return dx.reshape(x_shape)

    # -- non-quire sequential kernels (use_quire=false) --
    def matmul_seq(self, n, es, A, B):
        A, B = _codes(A), _codes(B)
        m, k = A.shape
        nn = B.shape[1]
        Cm = np.zeros((m, nn), np.uint64)
        self._chk(self.lib.po_matmul_seq(n, es, _p(A), _p(B), _p(Cm), i64(m), i64(k), i64(nn)), "matmul_seq")
        return Cm

    def conv2d_seq(self, n, es, x, w, bias, stride, pad):
        x, w = _codes(x), _codes(w)
        N, Cc, H, W = x.shape
        F, _, KH, KW = w.shape
        OH, OW = (H + 2 * pad - KH) // stride + 1, (W + 2 * pad - KW) // stride + 1
        y = np.zeros((N, F, OH, OW), np.uint64)
        b = _codes(bias) if bias is not None else None
        self._chk(self.lib.po_conv2d_seq(n, es, _p(x), i64(N), i64(Cc), i64(H), i64(W), _p(w), i64(F),
                                         i64(KH), i64(KW), _p(b), stride, pad, _p(y)), "conv2d_seq")
        return y

    def conv2d_input_grad_seq(self, n, es, dy, w, x_shape, stride, pad):
        dy, w = _codes(dy), _codes(w)
        N, F, OH, OW = dy.shape
        _, Cc, KH, KW = w.shape
        H, W = x_shape[2], x_shape[3]
        dx = np.zeros((N, Cc, H, W), np.uint64)
        self._chk(self.lib.po_conv2d_input_grad_seq(n, es, _p(dy), i64(N), i64(F), i64(OH), i64(OW), _p(w),
                                                    i64(Cc), i64(KH), i64(KW), i64(H), i64(W), stride, pad,
                                                    _p(dx)), "conv2d_input_grad_seq")
        return dx

    def conv2d_weight_grad_seq(self, n, es, dy, x, w_shape, stride, pad):
        dy, x = _codes(dy), _codes(x)
        N, F, OH, OW = dy.shape
        _, Cc, H, W = x.shape
        KH, KW = w_shape[2], w_shape[3]
        dw = np.zeros((F, Cc, KH, KW), np.uint64)
        self._chk(self.lib.po_conv2d_weight_grad_seq(n, es, _p(dy), i64(N), i64(F), i64(OH), i64(OW), _p(x),
                                                     i64(Cc), i64(H), i64(W), i64(KH), i64(KW), stride, pad,
                                                     _p(dw)), "conv2d_weight_grad_seq")
        return dw

    def bias_grad_seq(self, n, es, dy3):
        dy3 = _codes(dy3)
        N, F, P = dy3.shape
        db = np.zeros((F,), np.uint64)
        self._chk(self.lib.po_bias_grad_seq(n, es, _p(dy3), i64(N), i64(F), i64(P), _p(db)), "bias_grad_seq")
        return db

    def quire_words(self, q) -> tuple[int, bool]:
        """(W-bit quire value as a Python int, NaR flag) of a restatement quire."""
        buf = (C.c_uint64 * 16)()
        nar = C.c_int()
        self.lib.po_quire_words.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_int, C.POINTER(C.c_int)]
        nw = self.lib.po_quire_words(q.h, buf, 16, C.byref(nar))
        return sum(int(buf[i]) << (64 * i) for i in range(nw)), bool(nar.value)

    def round_words(self, n, es, value: int) -> int:
        """Round a W-bit quire value (Python int, taken mod 2^W) once."""
        W = 4 * ((n - 2) << es) + n
        value &= (1 << W) - 1
        nw = (W + 63) // 64
        arr = (C.c_uint64 * nw)(*[(value >> (64 * i)) & ((1 << 64) - 1) for i in range(nw)])
        self.lib.po_round_words.restype = C.c_uint64
        return int(self.lib.po_round_words(n, es, arr, nw))

    def ew(self, n, es, op, a, b):
        a, b = _codes(a), _codes(b)
        out = np.zeros(a.shape, np.uint64)
        self.lib.po_ew(n, es, op, _p(a), _p(b), _p(out), i64(a.size))
        return out

    def relu_fwd(self, n, es, x):
        x = _codes(x)
        y = np.zeros(x.shape, np.uint64)
        self.lib.po_relu_fwd(n, es, _p(x), _p(y), i64(x.size))
        return y

    def relu_bwd(self, xn, xes, x, dy):
        x, dy = _codes(x), _codes(dy)
        dx = np.zeros(dy.shape, np.uint64)
        self.lib.po_relu_bwd(xn, xes, _p(x), _p(dy), _p(dx), i64(x.size))
        return dx

    def softmax_xent(self, n, es, logits, labels, log2_batch, grad_scale_log2=0):
        z = _codes(logits)
        B, Cn = z.shape
        lab = np.ascontiguousarray(np.asarray(labels, np.int32))
        d = np.zeros(z.shape, np.uint64)
        rows = np.zeros((B,), np.uint64)
        self.lib.po_softmax_xent_scaled.restype = C.c_uint64
        loss = self.lib.po_softmax_xent_scaled(n, es, _p(z), lab.ctypes.data_as(C.POINTER(C.c_int32)),
                                               i64(B), i64(Cn), int(log2_batch), int(grad_scale_log2),
                                               _p(d), _p(rows))
        return int(loss), d, rows

    def sgd(self, on, oes, w, gn, ges, g, lr, grad_scale_log2=0):
        w = _codes(w).copy()
        g = _codes(g)
        self.lib.po_sgd_scaled(on, oes, _p(w), gn, ges, _p(g), i64(w.size), C.c_uint64(int(lr)),
                               int(grad_scale_log2))
        return w

    def convert_tensor(self, sn, se, dn, de, x):
        x = _codes(x)
        y = np.zeros(x.shape, np.uint64)
        flat = np.ascontiguousarray(x.ravel())
        yf = np.zeros(flat.shape, np.uint64)
        self._chk(self.lib.po_convert_tensor(sn, se, dn, de, _p(flat), i64(flat.size), _p(yf)),
                  "convert_tensor")
        y[...] = yf.reshape(x.shape)
        return y


    # ---- remaining SPEC layers (layers_oracle.c) ----
    def act_fwd(self, kind, n, es, x):
        x = _codes(x)
        y = np.zeros(x.shape, np.uint64)
        self.lib.po_act_fwd(int(kind), n, es, _p(x), _p(y), i64(x.size))
        return y

    def act_bwd(self, kind, f, y, b, dy):
        y, dy = _codes(y), _codes(dy)
        dx = np.zeros(dy.shape, np.uint64)
        self.lib.po_act_bwd(int(kind), *f, _p(y), *b, _p(dy), _p(dx), i64(dy.size))
        return dx

    def dropout_bits(self, seed, i):
        self.lib.po_dropout_bits.restype = C.c_uint64
        return self.lib.po_dropout_bits(C.c_uint64(int(seed)), i64(int(i)))

    def dropout(self, n, es, x, seed, thresh, scale):
        x = _codes(x)
        y = np.zeros(x.shape, np.uint64)
        self.lib.po_dropout(n, es, _p(x), _p(y), i64(x.size), C.c_uint64(int(seed)),
                            C.c_uint32(int(thresh)), C.c_uint64(int(scale)))
        return y

    def mse(self, n, es, y, t, global_count, grad_scale_log2=0):
        y, t = _codes(y), _codes(t)
        g = np.zeros(y.shape, np.uint64)
        self.lib.po_mse.restype = C.c_uint64
        loss = self.lib.po_mse(n, es, _p(y), _p(t), i64(y.size), i64(int(global_count)),
                               int(grad_scale_log2), _p(g))
        return int(loss), g

    def batchnorm_fwd(self, f, x, gamma, beta, eps, training, o, run_mean, run_var, mom):
        x = _codes(x)
        N, Cc = x.shape[:2]
        HW = int(np.prod(x.shape[2:], dtype=np.int64)) if x.ndim > 2 else 1
        rm, rv = _codes(run_mean).copy(), _codes(run_var).copy()
        y, xh = np.zeros(x.shape, np.uint64), np.zeros(x.shape, np.uint64)
        inv = np.zeros(Cc, np.uint64)
        self.lib.po_batchnorm_fwd(*f, _p(x), i64(N), i64(Cc), i64(HW), _p(_codes(gamma)), _p(_codes(beta)),
                                  C.c_uint64(int(eps)), int(training), *o, _p(rm), _p(rv),
                                  C.c_uint64(int(mom)), _p(y), _p(xh), _p(inv))
        return y, xh, inv, rm, rv

    def batchnorm_bwd(self, f, xhat, inv, b, dy, gamma_b, g):
        xhat, dy = _codes(xhat), _codes(dy)
        N, Cc = dy.shape[:2]
        HW = int(np.prod(dy.shape[2:], dtype=np.int64)) if dy.ndim > 2 else 1
        dx = np.zeros(dy.shape, np.uint64)
        dgm, dbt = np.zeros(Cc, np.uint64), np.zeros(Cc, np.uint64)
        self.lib.po_batchnorm_bwd(*f, _p(xhat), _p(_codes(inv)), *b, _p(dy), i64(N), i64(Cc), i64(HW),
                                  _p(_codes(gamma_b)), *g, _p(dx), _p(dgm), _p(dbt))
        return dx, dgm, dbt

    def sgd_momentum(self, o, w, v, g_fmt, g, lr, mu, grad_scale_log2=0):
        w, v, g = _codes(w).copy(), _codes(v).copy(), _codes(g)
        self.lib.po_sgd_momentum(*o, _p(w), _p(v), *g_fmt, _p(g), i64(w.size), C.c_uint64(int(lr)),
                                 C.c_uint64(int(mu)), int(grad_scale_log2))
        return w, v


class Reference(_Base):
    """The unmodified reference library (oracle/_ref/libpnn_ref.so)."""

    prefix = "ref_"

    def __init__(self, path: str = REFERENCE_SO):
        super().__init__(path)
        self.lib.ref_last_error.restype = C.c_char_p
        self.lib.ref_time_matmul.restype = C.c_double

    def _chk(self, rc):
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())

    def decode_fixed(self, n, es, code):
        ls, sg, ng, nr = C.c_int32(), C.c_uint32(), C.c_uint8(), C.c_uint8()
        self._chk(self.lib.ref_decode_fixed(n, es, C.c_uint64(int(code)), C.byref(ls), C.byref(sg),
                                            C.byref(ng), C.byref(nr)))
        return ls.value, sg.value, ng.value, nr.value

    def matmul(self, n, es, A, B, threads: int = 1, use_quire: bool = True):
        A, B = _codes(A), _codes(B)
        m, k = A.shape
        k2, nn = B.shape
        assert k == k2
        Cm = np.zeros((m, nn), np.uint64)
        self._chk(self.lib.ref_matmul(n, es, _p(A), _p(B), _p(Cm), i64(m), i64(k), i64(nn),
                                      int(use_quire), threads))
        return Cm

    def time_matmul(self, n, es, A, B, threads: int):
        """(seconds, C) for one reference quire matmul, timed inside the library."""
        A, B = _codes(A), _codes(B)
        m, k = A.shape
        nn = B.shape[1]
        Cm = np.zeros((m, nn), np.uint64)
        t = self.lib.ref_time_matmul(n, es, _p(A), _p(B), _p(Cm), i64(m), i64(k), i64(nn), threads)
        return t, Cm

    def conv2d(self, n, es, x, w, bias, stride, pad, threads: int = 1, use_quire: bool = True):
        x, w = _codes(x), _codes(w)
        N, Cc, H, W = x.shape
        F, _, KH, KW = w.shape
        OH, OW = (H + 2 * pad - KH) // stride + 1, (W + 2 * pad - KW) // stride + 1
        y = np.zeros((N, F, OH, OW), np.uint64)
        b = _codes(bias) if bias is not None else None
        self._chk(self.lib.ref_conv2d(n, es, _p(x), i64(N), i64(Cc), i64(H), i64(W), _p(w), i64(F),
                                      i64(KH), i64(KW), _p(b), stride, pad, int(use_quire), threads, _p(y)))
        return y

    def conv2d_input_grad(self, n, es, dy, w, x_shape, stride, pad, threads: int = 1, use_quire: bool = True):
        dy, w = _codes(dy), _codes(w)
        N, F, OH, OW = dy.shape
        _, Cc, KH, KW = w.shape
        H, W = x_shape[2], x_shape[3]
        dx = np.zeros((N, Cc, H, W), np.uint64)
        self._chk(self.lib.ref_conv2d_input_grad(n, es, _p(dy), i64(N), i64(F), i64(OH), i64(OW),
                                                 _p(w), i64(Cc), i64(KH), i64(KW), i64(H), i64(W),
                                                 stride, pad, int(use_quire), threads, _p(dx)))
        return dx

    def conv2d_weight_grad(self, n, es, dy, x, w_shape, stride, pad, threads: int = 1, use_quire: bool = True):
        dy, x = _codes(dy), _codes(x)
        N, F, OH, OW = dy.shape
        _, Cc, H, W = x.shape
        KH, KW = w_shape[2], w_shape[3]
        dw = np.zeros((F, Cc, KH, KW), np.uint64)
        self._chk(self.lib.ref_conv2d_weight_grad(n, es, _p(dy), i64(N), i64(F), i64(OH), i64(OW),
                                                  _p(x), i64(Cc), i64(H), i64(W), i64(KH), i64(KW),
                                                  stride, pad, int(use_quire), threads, _p(dw)))
        return dw

    def conv2d_bias_grad(self, n, es, dy, use_quire: bool = True):
        dy = _codes(dy)
        N, F, OH, OW = dy.shape
        db = np.zeros((F,), np.uint64)
        self._chk(self.lib.ref_conv2d_bias_grad(n, es, _p(dy), i64(N), i64(F), i64(OH), i64(OW), int(use_quire),
                                                _p(db)))
        return db

    def column_sum(self, n, es, x, use_quire: bool = True):
        x = _codes(x)
        B, N = x.shape
        out = np.zeros((N,), np.uint64)
        self._chk(self.lib.ref_column_sum(n, es, _p(x), i64(B), i64(N), int(use_quire), _p(out)))
        return out

    def maxpool2d(self, n, es, x, k, stride):
        x = _codes(x)
        N, Cc, H, W = x.shape
        OH, OW = (H - k) // stride + 1, (W - k) // stride + 1
        y = np.zeros((N, Cc, OH, OW), np.uint64)
        am = np.zeros((N, Cc, OH, OW), np.int64)
        self._chk(self.lib.ref_maxpool2d(n, es, _p(x), i64(N), i64(Cc), i64(H), i64(W), k, stride,
                                         _p(y), _p(am)))
        return y, am

    def maxpool2d_backward(self, n, es, dy, argmax, x_shape):
        dy = _codes(dy).ravel()
        am = np.ascontiguousarray(np.asarray(argmax, np.int64)).ravel()
        N, Cc, H, W = x_shape
        dx = np.zeros(tuple(x_shape), np.uint64)
        self._chk(self.lib.ref_maxpool2d_backward(n, es, _p(dy), i64(dy.size), _p(am), i64(N),
                                                  i64(Cc), i64(H), i64(W), _p(dx)))
        return dx

    def convert_tensor(self, sn, se, dn, de, x):
        x = _codes(x)
        flat = np.ascontiguousarray(x.ravel())
        yf = np.zeros(flat.shape, np.uint64)
        self._chk(self.lib.ref_convert_tensor(sn, se, dn, de, _p(flat), i64(flat.size), _p(yf)))
        return yf.reshape(x.shape)


def reference_available() -> bool:
    return os.path.exists(REFERENCE_SO)
