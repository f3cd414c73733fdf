"""Host-side mirror of the reference operator API for the quire hot path.

Mirrors /root/reference/proj/include/pnn/tensor_ops.hpp (names, argument
meaning and error behaviour): ``matmul(a, b, use_quire, pool=None)`` etc.
Two tensor kinds are accepted:

* numpy ``uint64`` arrays -- the reference's Tensor storage (one code per
  64-bit slot, tensor.hpp:10-14); routed through the synchronous ``*_host``
  C-ABI entry points (H2D copy, device kernels, D2H copy);
* torch CUDA tensors of packed codes (uint8 for nbits <= 8, uint16 up to 16)
  -- the device-resident path, asynchronous on the current torch stream.

Every call lands in libpnn_b200.so; nothing here computes posit arithmetic.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native

try:  # torch is plumbing (device memory, streams), not the product
    import torch
except Exception:  # pragma: no cover - torch is present in this image
    torch = None


@dataclass(frozen=True)
class PositConfig:
    """posit.hpp:17-42 (nbits, es) with the derived constants."""

    nbits: int
    es: int

    @property
    def max_scale(self) -> int:
        return (self.nbits - 2) << self.es

    @property
    def quire_bits(self) -> int:
        return 4 * self.max_scale + self.nbits

    @property
    def nar_pattern(self) -> int:
        return 1 << (self.nbits - 1)

    @property
    def maxpos_pattern(self) -> int:
        return self.nar_pattern - 1

    @property
    def code_dtype(self):
        return torch.uint8 if self.nbits <= 8 else torch.uint16

    @property
    def np_code_dtype(self):
        return np.uint8 if self.nbits <= 8 else np.uint16


P80, P81, P82 = PositConfig(8, 0), PositConfig(8, 1), PositConfig(8, 2)
P121, P161 = PositConfig(12, 1), PositConfig(16, 1)
# optimizer / loss formats of the posit(8,2)* preset (O12L10);
# elementwise-only (convert, softmax cross-entropy, SGD), no quire GEMMs
P102, P122 = PositConfig(10, 2), PositConfig(12, 2)


def _cfg(cfg) -> PositConfig:
    return cfg if isinstance(cfg, PositConfig) else PositConfig(*cfg)


def _stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class _Workspace:
    """Grow-only device workspace per device (digit planes, NaR flags, partials)."""

    def __init__(self):
        self.buf = {}

    def get(self, device, nbytes: int):
        key = torch.device(device).index
        t = self.buf.get(key)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)
            self.buf[key] = t
        return t


_ws = _Workspace()


def quire_gemm_workspace(cfg, M: int, N: int, K: int) -> int:
    cfg = _cfg(cfg)
    n = C.c_size_t()
    _native.check(_native.lib().pnn_quire_gemm_workspace(cfg.nbits, cfg.es, M, N, K, C.byref(n)))
    return n.value


def quire_gemm(cfg, A, B, out=None, max_kblocks: int | None = None):
    """Device quire GEMM on packed codes: C = round(A . B) (tensor_ops.cpp:166-185)."""
    cfg = _cfg(cfg)
    if A.dim() != 2 or B.dim() != 2:
        raise _native.PnnInvalidArgument(1, "matmul: rank-2 tensors required")
    if A.shape[1] != B.shape[0]:
        raise _native.PnnInvalidArgument(1, "matmul: inner dimensions disagree")
    if A.dtype != cfg.code_dtype or B.dtype != cfg.code_dtype:
        raise _native.PnnInvalidArgument(1, "matmul: dtype mismatch")
    A, B = A.contiguous(), B.contiguous()
    M, K = A.shape
    N = B.shape[1]
    if out is None:
        out = torch.empty((M, N), dtype=cfg.code_dtype, device=A.device)
    ws_bytes = quire_gemm_workspace(cfg, M, N, K)
    if max_kblocks is not None:  # forced split-K can need more partial space
        ws_bytes = max(ws_bytes, ws_bytes + 16 * M * N * (K // 32 + 2))
    ws = _ws.get(A.device, ws_bytes)
    L = _native.lib()
    if max_kblocks is None:
        rc = L.pnn_quire_gemm(cfg.nbits, cfg.es, A.data_ptr(), B.data_ptr(), out.data_ptr(), M, N, K,
                              ws.data_ptr(), ws.numel(), _stream_ptr(A.device))
    else:
        rc = L.pnn_quire_gemm_splitk(cfg.nbits, cfg.es, A.data_ptr(), B.data_ptr(), out.data_ptr(), M,
                                     N, K, int(max_kblocks), ws.data_ptr(), ws.numel(),
                                     _stream_ptr(A.device))
    _native.check(rc)
    return out


def matmul(a, b, use_quire: bool = True, pool=None, cfg=None):
    """tensor_ops.hpp:28-29.  ``pool`` is accepted and ignored (results are
    worker-count invariant in the reference, tensor_ops.hpp:12-13)."""
    if cfg is None:
        raise _native.PnnInvalidArgument(1, "matmul: posit config required")
    cfg = _cfg(cfg)
    if not use_quire:  # sequential rounding per term (tensor_ops.cpp:145-164)
        if isinstance(a, np.ndarray):
            d = matmul_seq(cfg, torch.from_numpy(np.ascontiguousarray(a).astype(cfg.np_code_dtype)).cuda(),
                           torch.from_numpy(np.ascontiguousarray(b).astype(cfg.np_code_dtype)).cuda())
            return d.cpu().numpy().astype(np.int64).astype(np.uint64)
        return matmul_seq(cfg, a, b)
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        if a.ndim != 2 or b.ndim != 2:
            raise _native.PnnInvalidArgument(1, "matmul: rank-2 tensors required")
        if a.shape[1] != b.shape[0]:
            raise _native.PnnInvalidArgument(1, "matmul: inner dimensions disagree")
        M, K = a.shape
        N = b.shape[1]
        c = np.zeros((M, N), np.uint64)
        _native.check(_native.lib().pnn_matmul_host(cfg.nbits, cfg.es, a.ctypes.data, b.ctypes.data,
                                                    c.ctypes.data, M, K, N))
        return c
    return quire_gemm(cfg, a, b)


def matmul_seq(cfg, A, B):
    """Non-quire posit matmul (matmul_seq, tensor_ops.cpp:145-164) on device codes."""
    cfg = _cfg(cfg)
    if A.dim() != 2 or B.dim() != 2 or A.shape[1] != B.shape[0]:
        raise _native.PnnInvalidArgument(1, "matmul: bad shapes")
    _check_codes(cfg, A, B)
    A, B = A.contiguous(), B.contiguous()
    M, K = A.shape
    N = B.shape[1]
    out = torch.empty((M, N), dtype=cfg.code_dtype, device=A.device)
    _native.check(_native.lib().pnn_matmul_seq(cfg.nbits, cfg.es, A.data_ptr(), B.data_ptr(), out.data_ptr(),
                                               M, N, K, _stream_ptr(A.device)))
    return out


def par_matmul(a, b, use_quire: bool, workers: int, cfg=None):
    """tensor_ops.hpp:30-31 -- identical to matmul for every worker count."""
    return matmul(a, b, use_quire, None, cfg=cfg)


# ---- device posit core (parity / diagnostics) ------------------------------

def decode_x(cfg, codes):
    """codes (CUDA int32/uint32 tensor) -> (X int64, nar uint8)."""
    cfg = _cfg(cfg)
    codes = codes.to(torch.int32).contiguous()
    X = torch.empty(codes.shape, dtype=torch.int64, device=codes.device)
    nar = torch.empty(codes.shape, dtype=torch.uint8, device=codes.device)
    _native.check(_native.lib().pnn_decode_x(cfg.nbits, cfg.es, codes.data_ptr(), codes.numel(),
                                             X.data_ptr(), nar.data_ptr(), _stream_ptr(codes.device)))
    return X, nar


def quire_round(cfg, q_words):
    """q_words: CUDA int64 tensor [n, 2] (lo, hi) -> int32 codes [n]."""
    cfg = _cfg(cfg)
    q_words = q_words.contiguous()
    n = q_words.shape[0]
    out = torch.empty((n,), dtype=torch.int32, device=q_words.device)
    _native.check(_native.lib().pnn_quire_round(cfg.nbits, cfg.es, q_words.data_ptr(), n,
                                                out.data_ptr(), _stream_ptr(q_words.device)))
    return out


def pack_round(cfg, neg, scale, sig, sticky):
    """Elementwise detail::pack_round on CUDA tensors (int32, int32, int64, int32)."""
    cfg = _cfg(cfg)
    n = neg.numel()
    out = torch.empty((n,), dtype=torch.int32, device=neg.device)
    _native.check(_native.lib().pnn_pack_round(cfg.nbits, cfg.es, neg.contiguous().data_ptr(),
                                               scale.contiguous().data_ptr(),
                                               sig.contiguous().data_ptr(),
                                               sticky.contiguous().data_ptr(), n, out.data_ptr(),
                                               _stream_ptr(neg.device)))
    return out


# ---- Conv2d / Linear passes (tensor_ops.hpp:34-42, 61) ----------------------

def conv_algo(algo: int) -> int:
    """Select the conv implementation (pnn_conv_algo): 0 auto (implicit GEMM
    where eligible), 1 explicit im2col pack, 2 implicit only.  Returns the
    previous setting.  Results are bit-identical either way."""
    prev = _native.lib().pnn_conv_algo(int(algo))
    if prev < 0:
        raise _native.PnnInvalidArgument(1, "conv_algo: 0, 1 or 2")
    return prev


def _conv_ws(pass_, cfg, N, Cc, H, W, F, KH, KW, stride, pad, has_bias):
    n = C.c_size_t()
    _native.check(_native.lib().pnn_conv2d_workspace(pass_, cfg.nbits, cfg.es, N, Cc, H, W, F, KH, KW,
                                                      stride, pad, int(has_bias), C.byref(n)))
    return n.value


def _check_codes(cfg, *ts):
    for t in ts:
        if t is not None and t.dtype != cfg.code_dtype:
            raise _native.PnnInvalidArgument(1, "dtype mismatch")


def conv2d(cfg, x, w, bias, stride: int, pad: int, use_quire: bool = True, pool=None):
    """tensor_ops.hpp:34-35: y = round(conv(x_pad, w) + bias), bias inside the quire."""
    cfg = _cfg(cfg)
    if x.dim() != 4 or w.dim() != 4:
        raise _native.PnnInvalidArgument(1, "conv2d: NCHW/FCKK tensors required")
    if x.shape[1] != w.shape[1]:
        raise _native.PnnInvalidArgument(1, "conv2d: channel mismatch")
    _check_codes(cfg, x, w, bias)
    x, w = x.contiguous(), w.contiguous()
    bias = bias.contiguous() if bias is not None else None
    N, Cc, H, W = x.shape
    F, _, KH, KW = w.shape
    OH, OW = (H + 2 * pad - KH) // stride + 1, (W + 2 * pad - KW) // stride + 1
    y = torch.empty((N, F, OH, OW), dtype=cfg.code_dtype, device=x.device)
    if not use_quire:  # conv_seq, tensor_ops.cpp:232-264
        _native.check(_native.lib().pnn_conv2d_fwd_seq(
            cfg.nbits, cfg.es, x.data_ptr(), N, Cc, H, W, w.data_ptr(), F, KH, KW,
            bias.data_ptr() if bias is not None else None, stride, pad, y.data_ptr(), _stream_ptr(x.device)))
        return y
    ws = _ws.get(x.device, _conv_ws(0, cfg, N, Cc, H, W, F, KH, KW, stride, pad, bias is not None))
    _native.check(_native.lib().pnn_conv2d_fwd(
        cfg.nbits, cfg.es, x.data_ptr(), N, Cc, H, W, w.data_ptr(), F, KH, KW,
        bias.data_ptr() if bias is not None else None, stride, pad, y.data_ptr(), ws.data_ptr(),
        ws.numel(), _stream_ptr(x.device)))
    return y


def conv2d_input_grad(cfg, dy, w, x_shape, stride: int, pad: int, use_quire: bool = True, pool=None):
    """tensor_ops.hpp:36-38."""
    cfg = _cfg(cfg)
    _check_codes(cfg, dy, w)
    dy, w = dy.contiguous(), w.contiguous()
    N, Cc, H, W = (int(v) for v in x_shape)
    _, F, OH, OW = dy.shape
    _, _, KH, KW = w.shape
    dx = torch.empty((N, Cc, H, W), dtype=cfg.code_dtype, device=dy.device)
    if not use_quire:  # gather_seq over the valid taps, tensor_ops.cpp:302-318, 539-560
        _native.check(_native.lib().pnn_conv2d_dgrad_seq(
            cfg.nbits, cfg.es, dy.data_ptr(), N, F, OH, OW, w.data_ptr(), Cc, KH, KW, H, W, stride, pad,
            dx.data_ptr(), _stream_ptr(dy.device)))
        return dx
    ws = _ws.get(dy.device, _conv_ws(1, cfg, N, Cc, H, W, F, KH, KW, stride, pad, False))
    _native.check(_native.lib().pnn_conv2d_dgrad(
        cfg.nbits, cfg.es, dy.data_ptr(), N, F, OH, OW, w.data_ptr(), Cc, KH, KW, H, W, stride, pad,
        dx.data_ptr(), ws.data_ptr(), ws.numel(), _stream_ptr(dy.device)))
    return dx


def conv2d_weight_grad(cfg, dy, x, w_shape, stride: int, pad: int, use_quire: bool = True, pool=None,
                       raw: bool = False):
    """tensor_ops.hpp:39-41.  raw=True also returns the exact unrounded quire
    words (int64 [..., 2]: lo, hi) and NaR mask -- the data-parallel reduction input."""
    cfg = _cfg(cfg)
    _check_codes(cfg, dy, x)
    dy, x = dy.contiguous(), x.contiguous()
    N, F, OH, OW = dy.shape
    _, Cc, H, W = x.shape
    KH, KW = int(w_shape[2]), int(w_shape[3])
    dw = torch.empty((F, Cc, KH, KW), dtype=cfg.code_dtype, device=dy.device)
    if not use_quire:  # gather_seq over (n, oy, ox), tensor_ops.cpp:302-318, 586-600
        if raw:
            raise _native.PnnInvalidArgument(1, "raw quire words need use_quire=True")
        _native.check(_native.lib().pnn_conv2d_wgrad_seq(
            cfg.nbits, cfg.es, dy.data_ptr(), N, F, OH, OW, x.data_ptr(), Cc, H, W, KH, KW, stride, pad,
            dw.data_ptr(), _stream_ptr(dy.device)))
        return dw
    words = nar = None
    if raw:
        words = torch.empty((F, Cc, KH, KW, 2), dtype=torch.int64, device=dy.device)
        nar = torch.empty((F, Cc, KH, KW), dtype=torch.uint8, device=dy.device)
    ws = _ws.get(dy.device, _conv_ws(2, cfg, N, Cc, H, W, F, KH, KW, stride, pad, False))
    _native.check(_native.lib().pnn_conv2d_wgrad(
        cfg.nbits, cfg.es, dy.data_ptr(), N, F, OH, OW, x.data_ptr(), Cc, H, W, KH, KW, stride, pad,
        dw.data_ptr(), words.data_ptr() if raw else None, nar.data_ptr() if raw else None,
        ws.data_ptr(), ws.numel(), _stream_ptr(dy.device)))
    return (dw, words, nar) if raw else dw


def conv2d_saved_bytes(cfg, x_shape, w_shape, stride: int, pad: int) -> int:
    """Bytes of the forward's saved activation digits (0: no implicit
    forward / weight-gradient pair for this geometry)."""
    cfg = _cfg(cfg)
    N, Cc, H, W = (int(v) for v in x_shape)
    F, _, KH, KW = (int(v) for v in w_shape)
    n = C.c_size_t()
    _native.check(_native.lib().pnn_conv2d_saved_bytes(cfg.nbits, cfg.es, N, Cc, H, W, F, KH, KW, stride,
                                                       pad, C.byref(n)))
    return n.value


def conv2d_fwd_save(cfg, x, w, bias, stride: int, pad: int, saved):
    """conv2d that also leaves x's digit planes in `saved` (uint8 device tensor
    of conv2d_saved_bytes) for conv2d_backward's weight gradient."""
    cfg = _cfg(cfg)
    _check_codes(cfg, x, w, bias)
    x, w = x.contiguous(), w.contiguous()
    bias = bias.contiguous() if bias is not None else None
    N, Cc, H, W = x.shape
    F, _, KH, KW = w.shape
    OH, OW = (H + 2 * pad - KH) // stride + 1, (W + 2 * pad - KW) // stride + 1
    y = torch.empty((N, F, OH, OW), dtype=cfg.code_dtype, device=x.device)
    ws = _ws.get(x.device, _conv_ws(0, cfg, N, Cc, H, W, F, KH, KW, stride, pad, bias is not None))
    _native.check(_native.lib().pnn_conv2d_fwd_save(
        cfg.nbits, cfg.es, x.data_ptr(), N, Cc, H, W, w.data_ptr(), F, KH, KW,
        bias.data_ptr() if bias is not None else None, stride, pad, y.data_ptr(), saved.data_ptr(),
        saved.numel(), ws.data_ptr(), ws.numel(), _stream_ptr(x.device)))
    return y


def conv2d_fwd_layer(cfg, x, w, bias, stride: int, pad: int, saved=None, relu: bool = False,
                     want_pre: bool = False):
    """Forward of a Conv2d layer (optionally keeping x's digits in `saved`) with
    the following ReLU fused: returns (relu(y), y or None).  None when the
    geometry has no implicit forward (use conv2d + relu_fwd)."""
    cfg = _cfg(cfg)
    _check_codes(cfg, x, w, bias)
    x, w = x.contiguous(), w.contiguous()
    bias = bias.contiguous() if bias is not None else None
    N, Cc, H, W = x.shape
    F, _, KH, KW = w.shape
    OH, OW = (H + 2 * pad - KH) // stride + 1, (W + 2 * pad - KW) // stride + 1
    nb = C.c_size_t()
    rc = _native.lib().pnn_conv2d_workspace(0, cfg.nbits, cfg.es, N, Cc, H, W, F, KH, KW, stride, pad,
                                            int(bias is not None), C.byref(nb))
    if rc != 0:
        return None
    y = torch.empty((N, F, OH, OW), dtype=cfg.code_dtype, device=x.device)
    pre = torch.empty_like(y) if want_pre else None
    ws = _ws.get(x.device, nb.value)
    rc = _native.lib().pnn_conv2d_fwd_layer(
        cfg.nbits, cfg.es, x.data_ptr(), N, Cc, H, W, w.data_ptr(), F, KH, KW,
        bias.data_ptr() if bias is not None else None, stride, pad, int(relu), y.data_ptr(),
        pre.data_ptr() if pre is not None else None, saved.data_ptr() if saved is not None else None,
        saved.numel() if saved is not None else 0, ws.data_ptr(), ws.numel(), _stream_ptr(x.device))
    if rc == 2:  # PNN_EUNSUPPORTED: not an implicit-path geometry
        return None
    _native.check(rc)
    return y, pre


def conv2d_backward_eligible(f_cfg, b_cfg, g_cfg, x_shape, w_shape, stride, pad, raw, has_dx, has_saved):
    f, b, g = _cfg(f_cfg), _cfg(b_cfg), _cfg(g_cfg)
    N, Cc, H, W = (int(v) for v in x_shape)
    F, _, KH, KW = (int(v) for v in w_shape)
    n = C.c_size_t()
    rc = _native.lib().pnn_conv2d_backward_workspace(f.nbits, f.es, b.nbits, b.es, g.nbits, g.es, N, Cc, H, W,
                                                     F, KH, KW, stride, pad, int(raw), int(has_dx),
                                                     int(has_saved), C.byref(n))
    return n.value if rc == 0 else None


def conv2d_backward(f_cfg, b_cfg, g_cfg, dy, x, saved, w_bwd, x_shape, w_shape, stride: int, pad: int,
                    need_dx: bool, raw: bool = False):
    """Fused Conv2d layer backward:
      dw = conv2d_weight_grad(p_g, convert(dy, p_b->p_g), convert(x, p_f->p_g))
      dx = conv2d_input_grad(p_b, dy, w_bwd)           (need_dx)
    reading the forward's saved digits (conv2d_fwd_save) when usable; dy digitised
    once for both passes when p_b == p_g.  Returns (dx | None, dw) or, raw,
    (dx | None, (None, words, nar)); None when the geometry / formats are not
    eligible (use the per-pass calls)."""
    f, b, g = _cfg(f_cfg), _cfg(b_cfg), _cfg(g_cfg)
    nbytes = conv2d_backward_eligible(f, b, g, x_shape, w_shape, stride, pad, raw, need_dx, saved is not None)
    if nbytes is None:
        return None
    _check_codes(b, dy, w_bwd if need_dx else None)
    if x is not None:
        _check_codes(f, x)
        x = x.contiguous()
    dy = dy.contiguous()
    w_bwd = w_bwd.contiguous() if need_dx else None
    N, Cc, H, W = (int(v) for v in x_shape)
    F, _, KH, KW = (int(v) for v in w_shape)
    dev = dy.device
    dx = torch.empty((N, Cc, H, W), dtype=b.code_dtype, device=dev) if need_dx else None
    dw = words = nar = None
    if raw:
        words = torch.empty((F, Cc, KH, KW, 2), dtype=torch.int64, device=dev)
        nar = torch.empty((F, Cc, KH, KW), dtype=torch.uint8, device=dev)
    else:
        dw = torch.empty((F, Cc, KH, KW), dtype=g.code_dtype, device=dev)
    ws = _ws.get(dev, nbytes)
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    _native.check(_native.lib().pnn_conv2d_backward(
        f.nbits, f.es, b.nbits, b.es, g.nbits, g.es, dy.data_ptr(), ptr(x), ptr(saved),
        saved.numel() if saved is not None else 0, ptr(w_bwd),
        N, Cc, H, W, F, KH, KW, stride, pad, ptr(dx), ptr(dw), ptr(words), ptr(nar), ws.data_ptr(),
        ws.numel(), _stream_ptr(dev)))
    return dx, ((None, words, nar) if raw else dw)


def conv2d_backward_gated(f_cfg, b_cfg, g_cfg, dy, gate, x, saved, w_bwd, x_shape, w_shape, stride: int,
                          pad: int, need_dx: bool, raw: bool = False, want_gated: bool = True):
    """conv2d_backward of a Conv2d followed by a ReLU: dy is the ReLU's output
    gradient, gate its saved forward output (p_f); the ReLU backward is applied
    inside the digitisers.  Returns (dx | None, dw | (None, words, nar), gated dy)
    or None when not eligible.  want_gated=False skips the gated dy (None)."""
    f, b, g = _cfg(f_cfg), _cfg(b_cfg), _cfg(g_cfg)
    nbytes = conv2d_backward_eligible(f, b, g, x_shape, w_shape, stride, pad, raw, need_dx, saved is not None)
    if nbytes is None:
        return None
    _check_codes(b, dy, w_bwd if need_dx else None)
    _check_codes(f, gate)
    if x is not None:
        _check_codes(f, x)
        x = x.contiguous()
    dy, gate = dy.contiguous(), gate.contiguous()
    w_bwd = w_bwd.contiguous() if need_dx else None
    N, Cc, H, W = (int(v) for v in x_shape)
    F, _, KH, KW = (int(v) for v in w_shape)
    dev = dy.device
    dx = torch.empty((N, Cc, H, W), dtype=b.code_dtype, device=dev) if need_dx else None
    dw = words = nar = None
    if raw:
        words = torch.empty((F, Cc, KH, KW, 2), dtype=torch.int64, device=dev)
        nar = torch.empty((F, Cc, KH, KW), dtype=torch.uint8, device=dev)
    else:
        dw = torch.empty((F, Cc, KH, KW), dtype=g.code_dtype, device=dev)
    dyg = torch.empty_like(dy) if want_gated else None
    ws = _ws.get(dev, nbytes)
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    _native.check(_native.lib().pnn_conv2d_backward_gated(
        f.nbits, f.es, b.nbits, b.es, g.nbits, g.es, dy.data_ptr(), gate.data_ptr(), ptr(dyg), ptr(x),
        ptr(saved), saved.numel() if saved is not None else 0, ptr(w_bwd), N, Cc, H, W, F, KH, KW, stride,
        pad, ptr(dx), ptr(dw), ptr(words), ptr(nar), ws.data_ptr(), ws.numel(), _stream_ptr(dev)))
    return dx, ((None, words, nar) if raw else dw), dyg


def _bias_grad(cfg, dy3, raw=False, use_quire=True):
    N, F, P = dy3.shape
    db = torch.empty((F,), dtype=cfg.code_dtype, device=dy3.device)
    if not use_quire:  # gather_seq_sum, tensor_ops.cpp:320-335
        _native.check(_native.lib().pnn_bias_grad_seq(cfg.nbits, cfg.es, dy3.data_ptr(), N, F, P, db.data_ptr(),
                                                      _stream_ptr(dy3.device)))
        return db
    words = nar = None
    if raw:
        words = torch.empty((F, 2), dtype=torch.int64, device=dy3.device)
        nar = torch.empty((F,), dtype=torch.uint8, device=dy3.device)
    n = C.c_size_t()
    _native.check(_native.lib().pnn_bias_grad_workspace(F, C.byref(n)))
    ws = _ws.get(dy3.device, n.value)
    _native.check(_native.lib().pnn_bias_grad(cfg.nbits, cfg.es, dy3.data_ptr(), N, F, P, db.data_ptr(),
                                              words.data_ptr() if raw else None,
                                              nar.data_ptr() if raw else None, ws.data_ptr(), ws.numel(),
                                              _stream_ptr(dy3.device)))
    return (db, words, nar) if raw else db


def conv2d_bias_grad(cfg, dy, use_quire: bool = True, raw: bool = False):
    """tensor_ops.hpp:42: db[f] = round(quire sum over (n, oy, ox) of dy)."""
    cfg = _cfg(cfg)
    _check_codes(cfg, dy)
    if dy.dim() != 4:
        raise _native.PnnInvalidArgument(1, "conv2d_bias_grad: bad rank")
    N, F, OH, OW = dy.shape
    return _bias_grad(cfg, dy.contiguous().view(N, F, OH * OW), raw, use_quire)


def conv2d_bias_grad_gated(cfg, dy, gate_cfg, gate, raw: bool = False):
    """conv2d_bias_grad of relu_bwd(gate, dy) without materialising it; None
    when the kernel does not cover the format / row length."""
    cfg, gc = _cfg(cfg), _cfg(gate_cfg)
    _check_codes(cfg, dy)
    _check_codes(gc, gate)
    N, F, OH, OW = dy.shape
    dy, gate = dy.contiguous(), gate.contiguous()
    db = torch.empty((F,), dtype=cfg.code_dtype, device=dy.device)
    words = torch.empty((F, 2), dtype=torch.int64, device=dy.device) if raw else None
    nar = torch.empty((F,), dtype=torch.uint8, device=dy.device) if raw else None
    n = C.c_size_t()
    _native.check(_native.lib().pnn_bias_grad_workspace(F, C.byref(n)))
    ws = _ws.get(dy.device, n.value)
    rc = _native.lib().pnn_bias_grad_gated(cfg.nbits, cfg.es, dy.data_ptr(), gc.nbits, gate.data_ptr(), N, F,
                                           OH * OW, db.data_ptr(), words.data_ptr() if raw else None,
                                           nar.data_ptr() if raw else None, ws.data_ptr(), ws.numel(),
                                           _stream_ptr(dy.device))
    if rc == 2:
        return None
    _native.check(rc)
    return (db, words, nar) if raw else db


def column_sum(cfg, x, use_quire: bool = True, raw: bool = False):
    """tensor_ops.hpp:61: [B,N] -> [N] quire column sums."""
    cfg = _cfg(cfg)
    _check_codes(cfg, x)
    if x.dim() != 2:
        raise _native.PnnInvalidArgument(1, "column_sum: rank-2 tensor required")
    B, N = x.shape
    return _bias_grad(cfg, x.contiguous().view(B, N, 1), raw, use_quire)


# ---- elementwise kernels of the training step -------------------------------

def convert_tensor(t, src_cfg, dst_cfg):
    """tensor_ops.hpp:26 convert_tensor (same dtype returns the input, :808)."""
    s, d = _cfg(src_cfg), _cfg(dst_cfg)
    if s == d:
        return t
    t = t.contiguous()
    out = torch.empty(t.shape, dtype=d.code_dtype, device=t.device)
    _native.check(_native.lib().pnn_convert(s.nbits, s.es, d.nbits, d.es, t.data_ptr(), out.data_ptr(),
                                            t.numel(), _stream_ptr(t.device)))
    return out


def relu_fwd(cfg, x):
    cfg = _cfg(cfg)
    x = x.contiguous()
    y = torch.empty_like(x)
    _native.check(_native.lib().pnn_relu_fwd(cfg.nbits, cfg.es, x.data_ptr(), y.data_ptr(), x.numel(),
                                             _stream_ptr(x.device)))
    return y


def relu_bwd(x_cfg, x, g_cfg, dy):
    xc, gc = _cfg(x_cfg), _cfg(g_cfg)
    x, dy = x.contiguous(), dy.contiguous()
    if x.numel() != dy.numel():
        raise _native.PnnInvalidArgument(1, "relu_bwd: shape mismatch")
    dx = torch.empty_like(dy)
    _native.check(_native.lib().pnn_relu_bwd(xc.nbits, xc.es, x.data_ptr(), gc.nbits, gc.es, dy.data_ptr(),
                                             dx.data_ptr(), x.numel(), _stream_ptr(x.device)))
    return dx


def maxpool2d(cfg, x, k: int, stride: int, pool=None):
    """tensor_ops.hpp:44-49: (out, argmax as flat input indices)."""
    cfg = _cfg(cfg)
    x = x.contiguous()
    N, Cc, H, W = x.shape
    if H < k or W < k:
        raise _native.PnnInvalidArgument(1, "maxpool2d: window larger than input")
    OH, OW = (H - k) // stride + 1, (W - k) // stride + 1
    y = torch.empty((N, Cc, OH, OW), dtype=x.dtype, device=x.device)
    am = torch.empty((N, Cc, OH, OW), dtype=torch.int64, device=x.device)
    _native.check(_native.lib().pnn_maxpool2d_fwd(cfg.nbits, cfg.es, x.data_ptr(), N, Cc, H, W, k, stride,
                                                  y.data_ptr(), am.data_ptr(), _stream_ptr(x.device)))
    return y, am


def maxpool2d_backward(cfg, dy, argmax, x_shape, k=None, stride=None):
    """tensor_ops.hpp:50-51 / tensor_ops.cpp:658-670.

    Reference signature (k, stride omitted): window-independent scatter,
    dx[argmax[i]] = add(dx[argmax[i]], dy[i]) for i in increasing order, for any
    argmax.  Indices outside [0, numel(x_shape)) raise PnnInvalidArgument (the
    reference has undefined behaviour there).  With k and stride given, dy and
    argmax must be the (N, C, OH, OW) result of maxpool2d(x, k, stride): the
    window-specialised kernel runs after a shape check."""
    cfg = _cfg(cfg)
    N, Cc, H, W = (int(v) for v in x_shape)
    dy, argmax = dy.contiguous(), argmax.contiguous()
    if dy.numel() != argmax.numel():
        raise _native.PnnInvalidArgument(1, "maxpool2d_backward: argmax mismatch")
    dx = torch.empty((N, Cc, H, W), dtype=cfg.code_dtype, device=dy.device)
    if (k is None) != (stride is None):
        raise _native.PnnInvalidArgument(1, "maxpool2d_backward: give both k and stride, or neither")
    if k is not None:
        if H < k or W < k or k < 1 or stride < 1:
            raise _native.PnnInvalidArgument(1, "maxpool2d_backward: bad window")
        OH, OW = (H - k) // stride + 1, (W - k) // stride + 1
        if tuple(dy.shape) != (N, Cc, OH, OW):
            raise _native.PnnInvalidArgument(
                1, f"maxpool2d_backward: dy shape {tuple(dy.shape)} is not {(N, Cc, OH, OW)}")
        _native.check(_native.lib().pnn_maxpool2d_bwd(cfg.nbits, cfg.es, dy.data_ptr(), argmax.data_ptr(),
                                                      N, Cc, H, W, k, stride, dx.data_ptr(),
                                                      _stream_ptr(dy.device)))
        return dx
    n_in = N * Cc * H * W
    if argmax.numel() and (int(argmax.min()) < 0 or int(argmax.max()) >= n_in):
        raise _native.PnnInvalidArgument(1, "maxpool2d_backward: argmax index out of range")
    n = C.c_size_t()
    _native.check(_native.lib().pnn_maxpool2d_bwd_scatter_workspace(dy.numel(), n_in, C.byref(n)))
    ws = _ws.get(dy.device, n.value)
    _native.check(_native.lib().pnn_maxpool2d_bwd_scatter(cfg.nbits, cfg.es, dy.data_ptr(),
                                                          argmax.to(torch.int64).data_ptr(), dy.numel(),
                                                          dx.data_ptr(), n_in, ws.data_ptr(), ws.numel(),
                                                          _stream_ptr(dy.device)))
    return dx


def softmax_xent_grad(cfg, logits, labels, log2_batch: int, grad_scale_log2: int = 0):
    """First half of softmax_xent: (dlogits, S row sums) -- the loss half is
    softmax_xent_loss, which may run on another stream."""
    cfg = _cfg(cfg)
    logits = logits.contiguous()
    B, Cn = logits.shape
    labels = labels.to(torch.int32).contiguous()
    d = torch.empty_like(logits)
    srows = torch.empty((B,), dtype=logits.dtype, device=logits.device)
    _native.check(_native.lib().pnn_softmax_xent_grad(cfg.nbits, cfg.es, logits.data_ptr(), labels.data_ptr(),
                                                      B, Cn, int(log2_batch), int(grad_scale_log2),
                                                      d.data_ptr(), srows.data_ptr(), _stream_ptr(logits.device)))
    return d, srows


def softmax_xent_loss(cfg, logits, labels, srows, log2_batch: int, raw: bool = False):
    """Second half: (loss [1], loss rows[, raw word, raw nar]) from softmax_xent_grad's S rows."""
    cfg = _cfg(cfg)
    logits = logits.contiguous()
    B, Cn = logits.shape
    labels = labels.to(torch.int32).contiguous()
    rows = torch.empty((B,), dtype=logits.dtype, device=logits.device)
    loss = torch.empty((1,), dtype=logits.dtype, device=logits.device)
    word = torch.empty((2,), dtype=torch.int64, device=logits.device) if raw else None
    nar = torch.empty((1,), dtype=torch.uint8, device=logits.device) if raw else None
    _native.check(_native.lib().pnn_softmax_xent_loss(cfg.nbits, cfg.es, logits.data_ptr(), labels.data_ptr(),
                                                      srows.data_ptr(), B, Cn, int(log2_batch), rows.data_ptr(),
                                                      loss.data_ptr(), word.data_ptr() if raw else None,
                                                      nar.data_ptr() if raw else None,
                                                      _stream_ptr(logits.device)))
    return (loss, rows, word, nar) if raw else (loss, rows)


def maxpool2d_noidx(cfg, x, k: int, stride: int):
    """maxpool2d output only (2x2 / stride-2 tiled; None when not eligible):
    the layer recomputes the argmax in maxpool2d_backward_x."""
    cfg = _cfg(cfg)
    x = x.contiguous()
    N, Cc, H, W = x.shape
    wpt = 8 if cfg.nbits <= 8 else 4
    if not (k == 2 and stride == 2 and H % 2 == 0 and W % (2 * wpt) == 0):
        return None
    y = torch.empty((N, Cc, H // 2, W // 2), dtype=x.dtype, device=x.device)
    _native.check(_native.lib().pnn_maxpool2d_fwd(cfg.nbits, cfg.es, x.data_ptr(), N, Cc, H, W, k, stride,
                                                  y.data_ptr(), None, _stream_ptr(x.device)))
    return y


def maxpool2d_backward_x(x_cfg, x, g_cfg, dy, k: int = 2, stride: int = 2, relu_gate: bool = False):
    """maxpool2d_backward(dy, argmax(maxpool2d(x))) with the argmax recomputed from x;
    relu_gate: x is a ReLU's output and the ReLU's backward is applied too."""
    xc, gc = _cfg(x_cfg), _cfg(g_cfg)
    x = x.contiguous()
    N, Cc, H, W = x.shape
    dx = torch.empty((N, Cc, H, W), dtype=gc.code_dtype, device=dy.device)
    _native.check(_native.lib().pnn_maxpool2d_relu_bwd_x(xc.nbits, xc.es, x.data_ptr(), gc.nbits, gc.es,
                                                         dy.contiguous().data_ptr(), N, Cc, H, W, k, stride,
                                                         int(relu_gate), dx.data_ptr(), _stream_ptr(dy.device)))
    return dx


def softmax_xent(cfg, logits, labels, log2_batch: int, raw: bool = False, grad_scale_log2: int = 0):
    """SURVEY.md Appendix A.5 -> (loss code tensor [1], dlogits, loss_rows[, raw word, raw nar]).
    grad_scale_log2 = s multiplies dlogits by 2^s (loss scaling)."""
    cfg = _cfg(cfg)
    logits = logits.contiguous()
    B, Cn = logits.shape
    labels = labels.to(torch.int32).contiguous()
    d = torch.empty_like(logits)
    rows = torch.empty((B,), dtype=logits.dtype, device=logits.device)
    loss = torch.empty((1,), dtype=logits.dtype, device=logits.device)
    word = torch.empty((2,), dtype=torch.int64, device=logits.device) if raw else None
    nar = torch.empty((1,), dtype=torch.uint8, device=logits.device) if raw else None
    _native.check(_native.lib().pnn_softmax_xent_scaled(cfg.nbits, cfg.es, logits.data_ptr(), labels.data_ptr(),
                                                 B, Cn, int(log2_batch), int(grad_scale_log2),
                                                 d.data_ptr(), rows.data_ptr(),
                                                 loss.data_ptr(), word.data_ptr() if raw else None,
                                                 nar.data_ptr() if raw else None, _stream_ptr(logits.device)))
    return (loss, d, rows, word, nar) if raw else (loss, d, rows)


def loss_reduce(cfg, loss_rows, log2_batch: int):
    """Batch loss from per-sample loss rows: ldexp(round(quire sum), -log2_batch)."""
    cfg = _cfg(cfg)
    rows = loss_rows.contiguous()
    out = torch.empty((1,), dtype=rows.dtype, device=rows.device)
    _native.check(_native.lib().pnn_loss_reduce(cfg.nbits, cfg.es, rows.data_ptr(), rows.numel(),
                                                int(log2_batch), out.data_ptr(), _stream_ptr(rows.device)))
    return out


def quire_bits(cfg) -> int:
    """W = 4R + nbits, R = (nbits - 2) << es."""
    cfg = _cfg(cfg)
    return 4 * ((cfg.nbits - 2) << cfg.es) + cfg.nbits


def sgd_step(opt_cfg, master, g_cfg, grad, lr_code: int, copies=(), grad_scale_log2: int = 0):
    """SURVEY.md Appendix A.7, in place on master; copies = [(cfg, tensor), ...] (<= 2).
    grad_scale_log2 = s unscales the gradient by 2^-s in the optimizer format."""
    oc, gc = _cfg(opt_cfg), _cfg(g_cfg)
    cps = [(_cfg(c), t) for c, t in copies] + [(oc, None)] * (2 - len(copies))
    (c1, t1), (c2, t2) = cps[0], cps[1]
    _native.check(_native.lib().pnn_sgd_step_scaled(oc.nbits, oc.es, master.data_ptr(), gc.nbits, gc.es,
                                                    grad.contiguous().data_ptr(), master.numel(),
                                                    int(lr_code), c1.nbits, c1.es,
                                                    t1.data_ptr() if t1 is not None else None,
                                                    c2.nbits, c2.es, t2.data_ptr() if t2 is not None else None,
                                                    int(grad_scale_log2), _stream_ptr(master.device)))
    return master


def sgd_step_multi(opt_cfg, g_cfg, lr_code: int, masters, grads, copy_cfgs=(), copies=(),
                   grad_scale_log2: int = 0):
    """sgd_step over several tensors in one launch; copies[i] = tuple of up to
    two stage-copy tensors of masters[i] in the formats copy_cfgs."""
    oc, gc = _cfg(opt_cfg), _cfg(g_cfg)
    n = len(masters)
    if n == 0:
        return
    cfgs = [_cfg(c) for c in copy_cfgs] + [oc] * (2 - len(copy_cfgs))
    P = C.c_void_p * n
    ms = P(*[m.data_ptr() for m in masters])
    gs = [g.contiguous() for g in grads]
    gp = P(*[g.data_ptr() for g in gs])
    c1 = P(*[c[0].data_ptr() for c in copies]) if len(copy_cfgs) > 0 else None
    c2 = P(*[c[1].data_ptr() for c in copies]) if len(copy_cfgs) > 1 else None
    ns = (C.c_int64 * n)(*[m.numel() for m in masters])
    _native.check(_native.lib().pnn_sgd_step_multi(oc.nbits, oc.es, gc.nbits, gc.es, int(lr_code),
                                                   cfgs[0].nbits, cfgs[0].es, cfgs[1].nbits, cfgs[1].es,
                                                   int(grad_scale_log2), n, ms, gp, c1, c2, ns,
                                                   _stream_ptr(masters[0].device)))


def scalar_eval(cfg, op: int, a, b=None):
    """Device scalar ALU (parity): a, b CUDA int32 code tensors."""
    cfg = _cfg(cfg)
    a = a.to(torch.int32).contiguous()
    b = b.to(torch.int32).contiguous() if b is not None else None
    out = torch.empty_like(a)
    _native.check(_native.lib().pnn_scalar_eval(cfg.nbits, cfg.es, op, a.data_ptr(),
                                                b.data_ptr() if b is not None else None, out.data_ptr(),
                                                a.numel(), _stream_ptr(a.device)))
    return out


# ---- data-parallel lane encoding (csrc/dp.cu) --------------------------------

def quire_to_lanes(cfg, words, nar):
    """Raw quire words (int64 [..., 2]) + NaR bytes -> int64 lanes [n, L+1]."""
    cfg = _cfg(cfg)
    L = _native.lib().pnn_quire_lanes(cfg.nbits, cfg.es)
    n = nar.numel()
    lanes = torch.empty((n, L + 1), dtype=torch.int64, device=words.device)
    _native.check(_native.lib().pnn_quire_to_lanes(cfg.nbits, cfg.es, words.contiguous().data_ptr(),
                                                   nar.contiguous().data_ptr(), n, lanes.data_ptr(),
                                                   _stream_ptr(words.device)))
    return lanes


def lanes_to_posit(cfg, lanes):
    cfg = _cfg(cfg)
    n = lanes.shape[0]
    out = torch.empty((n,), dtype=cfg.code_dtype, device=lanes.device)
    _native.check(_native.lib().pnn_lanes_to_posit(cfg.nbits, cfg.es, lanes.contiguous().data_ptr(), n,
                                                   out.data_ptr(), None, _stream_ptr(lanes.device)))
    return out


# ---- avg-pool (tensor_ops.hpp:53-58) ------------------------------------------

def avgpool2d(cfg, x, k: int, stride: int, use_quire: bool, recip_bits: int, pool=None):
    """Window sum (quire or add chain) times the caller-quantized 1/count."""
    cfg = _cfg(cfg)
    x = x.contiguous()
    N, Cc, H, W = x.shape
    if H < k or W < k:
        raise _native.PnnInvalidArgument(1, "avgpool2d: window larger than input")
    OH, OW = (H - k) // stride + 1, (W - k) // stride + 1
    y = torch.empty((N, Cc, OH, OW), dtype=x.dtype, device=x.device)
    _native.check(_native.lib().pnn_avgpool2d_fwd(cfg.nbits, cfg.es, x.data_ptr(), N, Cc, H, W, k, stride,
                                                  int(use_quire), int(recip_bits), y.data_ptr(),
                                                  _stream_ptr(x.device)))
    return y


def avgpool2d_backward(cfg, dy, k: int, stride: int, x_shape, recip_bits: int, pool=None):
    cfg = _cfg(cfg)
    N, Cc, H, W = (int(v) for v in x_shape)
    dx = torch.empty((N, Cc, H, W), dtype=cfg.code_dtype, device=dy.device)
    _native.check(_native.lib().pnn_avgpool2d_bwd(cfg.nbits, cfg.es, dy.contiguous().data_ptr(), N, Cc, H, W, k,
                                                  stride, int(recip_bits), dx.data_ptr(), _stream_ptr(dy.device)))
    return dx


# ---- remaining SPEC layers (csrc/layers.cu) ---------------

ACT_TANH, ACT_SIGMOID = 1, 2


def act_fwd(kind: int, cfg, x):
    """y = tanh_posit / sigmoid_posit (x) elementwise (posit_math.cpp:109-130)."""
    cfg = _cfg(cfg)
    x = x.contiguous()
    y = torch.empty_like(x)
    _native.check(_native.lib().pnn_act_fwd(int(kind), cfg.nbits, cfg.es, x.data_ptr(), y.data_ptr(),
                                            x.numel(), _stream_ptr(x.device)))
    return y


def act_bwd(kind: int, f_cfg, y, b_cfg, dy):
    """dx from the forward output y: tanh dy*(1-y*y), sigmoid dy*(y*(1-y)), in b."""
    fc, bc = _cfg(f_cfg), _cfg(b_cfg)
    y, dy = y.contiguous(), dy.contiguous()
    if y.numel() != dy.numel():
        raise _native.PnnInvalidArgument(1, "act_bwd: shape mismatch")
    dx = torch.empty_like(dy)
    _native.check(_native.lib().pnn_act_bwd(int(kind), fc.nbits, fc.es, y.data_ptr(), bc.nbits, bc.es,
                                            dy.data_ptr(), dx.data_ptr(), dy.numel(), _stream_ptr(dy.device)))
    return dx


def dropout_threshold(p: float) -> int:
    """floor(p * 2^32): element kept iff its 32 mask bits are >= this."""
    if not (0.0 <= p < 1.0):
        raise ValueError("dropout probability must be in [0, 1)")
    return int(p * 4294967296.0)


def dropout(cfg, x, seed: int, thresh: int, scale_code: int, seed_offset=None):
    """y = keep(seed [+ *seed_offset], i) ? x * scale : 0 (the backward: same call
    on dy).  seed_offset: optional device int64 [1] step counter."""
    cfg = _cfg(cfg)
    x = x.contiguous()
    y = torch.empty_like(x)
    _native.check(_native.lib().pnn_dropout(cfg.nbits, cfg.es, x.data_ptr(), y.data_ptr(), x.numel(),
                                            int(seed) & ((1 << 64) - 1),
                                            seed_offset.data_ptr() if seed_offset is not None else None,
                                            int(thresh), int(scale_code), _stream_ptr(x.device)))
    return y


def mse(cfg, y, t, global_count: int, grad_scale_log2: int = 0):
    """-> (loss code tensor [1], grad): loss = sum (y-t)^2 / G, grad = ldexp((y-t)*(2/G), s)."""
    cfg = _cfg(cfg)
    y, t = y.contiguous(), t.contiguous()
    if y.numel() != t.numel():
        raise _native.PnnInvalidArgument(1, "mse: shape mismatch")
    g = torch.empty_like(y)
    loss = torch.empty((1,), dtype=y.dtype, device=y.device)
    _native.check(_native.lib().pnn_mse(cfg.nbits, cfg.es, y.data_ptr(), t.data_ptr(), y.numel(),
                                        int(global_count), int(grad_scale_log2), g.data_ptr(),
                                        loss.data_ptr(), _stream_ptr(y.device)))
    return loss, g


def _bn_shape(x):
    N, Cc = int(x.shape[0]), int(x.shape[1])
    HW = int(x.numel() // max(N * Cc, 1))
    return N, Cc, HW


def batchnorm_fwd(f_cfg, x, gamma, beta, eps_code: int, training: bool, o_cfg, run_mean, run_var,
                  mom_code: int):
    """-> (y, xhat, inv); run_mean / run_var (optimizer format) updated in place when training."""
    fc, oc = _cfg(f_cfg), _cfg(o_cfg)
    x = x.contiguous()
    N, Cc, HW = _bn_shape(x)
    n = C.c_size_t()
    _native.check(_native.lib().pnn_batchnorm_workspace(Cc, C.byref(n)))
    ws = _ws.get(x.device, n.value)
    y, xh = torch.empty_like(x), torch.empty_like(x)
    inv = torch.empty((Cc,), dtype=x.dtype, device=x.device)
    _native.check(_native.lib().pnn_batchnorm_fwd(fc.nbits, fc.es, x.data_ptr(), N, Cc, HW,
                                                  gamma.contiguous().data_ptr(), beta.contiguous().data_ptr(),
                                                  int(eps_code), int(bool(training)), oc.nbits, oc.es,
                                                  run_mean.data_ptr(), run_var.data_ptr(), int(mom_code),
                                                  y.data_ptr(), xh.data_ptr(), inv.data_ptr(), ws.data_ptr(),
                                                  ws.numel(), _stream_ptr(x.device)))
    return y, xh, inv


def batchnorm_bwd(f_cfg, xhat, inv, b_cfg, dy, gamma_b, g_cfg, raw: bool = False):
    """-> (dx, dgamma, dbeta) or, raw, (dx, (dgamma words, nar), (dbeta words, nar))."""
    fc, bc, gc = _cfg(f_cfg), _cfg(b_cfg), _cfg(g_cfg)
    dy = dy.contiguous()
    N, Cc, HW = _bn_shape(dy)
    n = C.c_size_t()
    _native.check(_native.lib().pnn_batchnorm_workspace(Cc, C.byref(n)))
    ws = _ws.get(dy.device, n.value)
    dx = torch.empty_like(dy)
    dev = dy.device
    if raw:
        gw = torch.empty((Cc, 2), dtype=torch.int64, device=dev)
        gn = torch.empty((Cc,), dtype=torch.uint8, device=dev)
        bw = torch.empty((Cc, 2), dtype=torch.int64, device=dev)
        bn_ = torch.empty((Cc,), dtype=torch.uint8, device=dev)
        ptrs = (None, None, gw.data_ptr(), gn.data_ptr(), bw.data_ptr(), bn_.data_ptr())
    else:
        dg = torch.empty((Cc,), dtype=gc.code_dtype, device=dev)
        db = torch.empty((Cc,), dtype=gc.code_dtype, device=dev)
        ptrs = (dg.data_ptr(), db.data_ptr(), None, None, None, None)
    _native.check(_native.lib().pnn_batchnorm_bwd(fc.nbits, fc.es, xhat.contiguous().data_ptr(),
                                                  inv.contiguous().data_ptr(), bc.nbits, bc.es, dy.data_ptr(),
                                                  N, Cc, HW, gamma_b.contiguous().data_ptr(), gc.nbits, gc.es,
                                                  dx.data_ptr(), *ptrs, ws.data_ptr(), ws.numel(),
                                                  _stream_ptr(dev)))
    if raw:
        return dx, (gw, gn), (bw, bn_)
    return dx, dg, db


def sgd_step_momentum(opt_cfg, master, velocity, g_cfg, grad, lr_code: int, mu_code: int, copies=(),
                      grad_scale_log2: int = 0):
    """v = mu*v + ldexp(convert(grad), -s); master -= lr*v (in place, optimizer format)."""
    oc, gc = _cfg(opt_cfg), _cfg(g_cfg)
    cps = [(_cfg(c), t) for c, t in copies] + [(oc, None)] * (2 - len(copies))
    (c1, t1), (c2, t2) = cps[0], cps[1]
    _native.check(_native.lib().pnn_sgd_step_momentum(
        oc.nbits, oc.es, master.data_ptr(), velocity.data_ptr(), gc.nbits, gc.es, grad.contiguous().data_ptr(),
        master.numel(), int(lr_code), int(mu_code), c1.nbits, c1.es, t1.data_ptr() if t1 is not None else None,
        c2.nbits, c2.es, t2.data_ptr() if t2 is not None else None, int(grad_scale_log2),
        _stream_ptr(master.device)))
    return master
