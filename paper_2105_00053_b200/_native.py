"""ctypes binding of libpnn_b200.so (the C-ABI declared in include/pnn_b200.h).

The product path.  There is deliberately no CPU fallback: if the shared
library is missing or a call returns a nonzero status, we raise.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import threading

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
# PNN_B200_LIB: an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("PNN_B200_LIB") or os.path.join(PKG_DIR, "libpnn_b200.so")
HEADER_PATH = os.path.join(REPO_DIR, "include", "pnn_b200.h")

_lock = threading.Lock()
_lib: C.CDLL | None = None

_i64 = C.c_int64
_vp = C.c_void_p
_SIGS = {
    "pnn_last_error": (C.c_char_p, []),
    "pnn_abi_version": (C.c_int, []),
    "pnn_format_supported": (C.c_int, [C.c_int, C.c_int]),
    "pnn_code_bytes": (C.c_int, [C.c_int]),
    "pnn_quire_gemm_workspace": (C.c_int, [C.c_int, C.c_int, _i64, _i64, _i64, C.POINTER(C.c_size_t)]),
    "pnn_quire_gemm": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _vp, _i64, _i64, _i64, _vp, C.c_size_t, _vp]),
    "pnn_quire_gemm_splitk": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp,
                                        C.c_size_t, _vp]),
    "pnn_quire_gemm_profiled": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _vp, _i64, _i64, _i64, _vp,
                                          C.c_size_t, _vp, C.POINTER(C.c_float)]),
    "pnn_matmul_host": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _vp, _i64, _i64, _i64]),
    "pnn_decode_x": (C.c_int, [C.c_int, C.c_int, _vp, _i64, _vp, _vp, _vp]),
    "pnn_quire_round": (C.c_int, [C.c_int, C.c_int, _vp, _i64, _vp, _vp]),
    "pnn_pack_round": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "pnn_conv_algo": (C.c_int, [C.c_int]),
    "pnn_conv2d_workspace": (C.c_int, [C.c_int, C.c_int, C.c_int] + [_i64] * 7 + [C.c_int, C.c_int, C.c_int,
                                                                           C.POINTER(C.c_size_t)]),
    "pnn_conv2d_fwd": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [_vp] + [_i64] * 3 +
                       [_vp, C.c_int, C.c_int, _vp, _vp, C.c_size_t, _vp]),
    "pnn_conv2d_saved_bytes": (C.c_int, [C.c_int, C.c_int] + [_i64] * 7 + [C.c_int, C.c_int,
                                                                           C.POINTER(C.c_size_t)]),
    "pnn_conv2d_fwd_save": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [_vp] + [_i64] * 3 +
                            [_vp, C.c_int, C.c_int, _vp, _vp, C.c_size_t, _vp, C.c_size_t, _vp]),
    "pnn_conv2d_fwd_layer": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [_vp] + [_i64] * 3 +
                             [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, C.c_size_t, _vp, C.c_size_t,
                              _vp]),
    "pnn_conv2d_backward_workspace": (C.c_int, [C.c_int] * 6 + [_i64] * 7 + [C.c_int] * 5 +
                                      [C.POINTER(C.c_size_t)]),
    "pnn_conv2d_backward": (C.c_int, [C.c_int] * 6 + [_vp, _vp, _vp, C.c_size_t, _vp] + [_i64] * 7 +
                            [C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, C.c_size_t, _vp]),
    "pnn_conv2d_dgrad": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [_vp] + [_i64] * 5 +
                         [C.c_int, C.c_int, _vp, _vp, C.c_size_t, _vp]),
    "pnn_conv2d_wgrad": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [_vp] + [_i64] * 5 +
                         [C.c_int, C.c_int, _vp, _vp, _vp, _vp, C.c_size_t, _vp]),
    "pnn_bias_grad_workspace": (C.c_int, [_i64, C.POINTER(C.c_size_t)]),
    "pnn_bias_grad": (C.c_int, [C.c_int, C.c_int, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, C.c_size_t,
                                _vp]),
    "pnn_convert": (C.c_int, [C.c_int] * 4 + [_vp, _vp, _i64, _vp]),
    "pnn_relu_fwd": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _i64, _vp]),
    "pnn_relu_bwd": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int, C.c_int, _vp, _vp, _i64, _vp]),
    "pnn_maxpool2d_fwd": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [C.c_int, C.c_int, _vp, _vp, _vp]),
    "pnn_maxpool2d_bwd": (C.c_int, [C.c_int, C.c_int, _vp, _vp] + [_i64] * 4 + [C.c_int, C.c_int, _vp, _vp]),
    "pnn_maxpool2d_bwd_scatter_workspace": (C.c_int, [_i64, _i64, C.POINTER(C.c_size_t)]),
    "pnn_maxpool2d_bwd_scatter": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _i64, _vp, _i64, _vp, C.c_size_t,
                                            _vp]),
    "pnn_softmax_xent_grad": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _i64, _i64, C.c_int, C.c_int, _vp, _vp,
                                        _vp]),
    "pnn_softmax_xent_loss": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _vp, _i64, _i64, C.c_int, _vp, _vp, _vp,
                                        _vp, _vp]),
    "pnn_conv2d_backward_gated": (C.c_int, [C.c_int] * 6 + [_vp, _vp, _vp, _vp, _vp, C.c_size_t, _vp] +
                                  [_i64] * 7 + [C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, C.c_size_t, _vp]),
    "pnn_bias_grad_gated": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int, _vp, _i64, _i64, _i64, _vp, _vp, _vp,
                                      _vp, C.c_size_t, _vp]),
    "pnn_variant_min_work": (C.c_int64, [C.c_int64]),
    "pnn_sgd_step_multi": (C.c_int, [C.c_int] * 4 + [C.c_uint32] + [C.c_int] * 6 +
                           [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pnn_maxpool2d_relu_bwd_x": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int, C.c_int, _vp] + [_i64] * 4 +
                                 [C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "pnn_maxpool2d_bwd_x": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int, C.c_int, _vp] + [_i64] * 4 +
                            [C.c_int, C.c_int, _vp, _vp]),
    "pnn_softmax_xent": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _i64, _i64, C.c_int, _vp, _vp, _vp, _vp, _vp,
                                   _vp]),
    "pnn_sgd_step": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int, C.c_int, _vp, _i64, C.c_uint32, C.c_int,
                               C.c_int, _vp, C.c_int, C.c_int, _vp, _vp]),
    "pnn_softmax_xent_scaled": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _i64, _i64, C.c_int, C.c_int, _vp,
                                          _vp, _vp, _vp, _vp, _vp]),
    "pnn_sgd_step_scaled": (C.c_int, [C.c_int, C.c_int, _vp, C.c_int, C.c_int, _vp, _i64, C.c_uint32,
                                      C.c_int, C.c_int, _vp, C.c_int, C.c_int, _vp, C.c_int, _vp]),
    "pnn_loss_reduce": (C.c_int, [C.c_int, C.c_int, _vp, _i64, C.c_int, _vp, _vp]),
    "pnn_act_fwd": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, _vp, _i64, _vp]),
    "pnn_act_bwd": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, C.c_int, C.c_int, _vp, _vp, _i64, _vp]),
    "pnn_dropout": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _i64, C.c_uint64, _vp, C.c_uint32, C.c_uint32,
                              _vp]),
    "pnn_mse": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _i64, _i64, C.c_int, _vp, _vp, _vp]),
    "pnn_batchnorm_workspace": (C.c_int, [_i64, C.POINTER(C.c_size_t)]),
    "pnn_batchnorm_fwd": (C.c_int, [C.c_int, C.c_int, _vp, _i64, _i64, _i64, _vp, _vp, C.c_uint32, C.c_int,
                                    C.c_int, C.c_int, _vp, _vp, C.c_uint32, _vp, _vp, _vp, _vp, C.c_size_t,
                                    _vp]),
    "pnn_batchnorm_bwd": (C.c_int, [C.c_int, C.c_int, _vp, _vp, C.c_int, C.c_int, _vp, _i64, _i64, _i64, _vp,
                                    C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_size_t,
                                    _vp]),
    "pnn_sgd_step_momentum": (C.c_int, [C.c_int, C.c_int, _vp, _vp, C.c_int, C.c_int, _vp, _i64, C.c_uint32,
                                        C.c_uint32, C.c_int, C.c_int, _vp, C.c_int, C.c_int, _vp, C.c_int,
                                        _vp]),
    "pnn_avgpool2d_fwd": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [C.c_int, C.c_int, C.c_int,
                                                                         C.c_uint32, _vp, _vp]),
    "pnn_avgpool2d_bwd": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [C.c_int, C.c_int, C.c_uint32,
                                                                         _vp, _vp]),
    "pnn_from_float64": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _i64, _vp]),
    "pnn_scalar_eval": (C.c_int, [C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _i64, _vp]),
    "pnn_quire_lanes": (C.c_int, [C.c_int, C.c_int]),
    "pnn_quire_to_lanes": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _i64, _vp, _vp]),
    "pnn_lanes_to_posit": (C.c_int, [C.c_int, C.c_int, _vp, _i64, _vp, _vp, _vp]),
    "pnn_matmul_seq": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "pnn_conv2d_fwd_seq": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [_vp] + [_i64] * 3 +
                           [_vp, C.c_int, C.c_int, _vp, _vp]),
    "pnn_conv2d_dgrad_seq": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [_vp] + [_i64] * 5 +
                             [C.c_int, C.c_int, _vp, _vp]),
    "pnn_conv2d_wgrad_seq": (C.c_int, [C.c_int, C.c_int, _vp] + [_i64] * 4 + [_vp] + [_i64] * 5 +
                             [C.c_int, C.c_int, _vp, _vp]),
    "pnn_bias_grad_seq": (C.c_int, [C.c_int, C.c_int, _vp, _i64, _i64, _i64, _vp, _vp]),
    "pnn_probe_int8_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
}


class PnnError(RuntimeError):
    """A nonzero status from the C-ABI (message from pnn_last_error())."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[pnn status {code}] {msg}")
        self.code = code


class PnnInvalidArgument(PnnError, ValueError):
    """PNN_EINVAL -- the reference raises std::invalid_argument here."""


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                    "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def header_symbols() -> list[str]:
    """Every function the public C header declares."""
    txt = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(pnn_[a-z0-9_]+)\s*\(", txt)))


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().pnn_last_error().decode(errors="replace")
        if rc == 1:
            raise PnnInvalidArgument(rc, msg)
        raise PnnError(rc, msg)
