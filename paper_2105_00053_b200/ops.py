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
    if not use_quire:
        raise NotImplementedError("non-quire sequential-rounding matmul is outside this path "
                                  "(SURVEY.md §8f item 1)")
    if cfg is None:
        raise _native.PnnInvalidArgument(1, "matmul: posit config required")
    cfg = _cfg(cfg)
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
