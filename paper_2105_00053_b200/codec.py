"""Host <-> device code movement and float ingestion (from_float64 on device)."""
from __future__ import annotations

import numpy as np
import torch

from . import _native, ops


def from_float64_array(x, cfg, device="cuda") -> np.ndarray:
    """from_float64 (posit.cpp:502-508) of every element -> uint64 codes (host)."""
    return from_float64_device(x, cfg, device).cpu().numpy().astype(np.uint64)


def from_float64_device(x, cfg, device="cuda") -> torch.Tensor:
    """from_float64 of every element -> packed codes (device tensor)."""
    cfg = ops._cfg(cfg)
    xd = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(device)
    out = torch.empty(xd.shape, dtype=cfg.code_dtype, device=device)
    _native.check(_native.lib().pnn_from_float64(cfg.nbits, cfg.es, xd.data_ptr(), out.data_ptr(), xd.numel(),
                                                 ops._stream_ptr(xd.device)))
    return out


def to_device(codes: np.ndarray, cfg, device="cuda") -> torch.Tensor:
    cfg = ops._cfg(cfg)
    return torch.from_numpy(np.ascontiguousarray(codes).astype(cfg.np_code_dtype)).to(device)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().astype(np.int64).astype(np.uint64)
