"""Model checkpoints in the "PNN1" format (the format is
specified only in the reference's SPEC, "External Interfaces": magic "PNN1",
then per-tensor records {name length + bytes, nbits, es, rank, extents, raw bit
patterns packed little-endian in ceil(nbits/8) bytes each}).

Field widths (the SPEC leaves them open; fixed here): name length uint32 LE,
name UTF-8, nbits uint8, es uint8, rank uint8, extents int64 LE, then the codes.
Records follow each other to the end of the file.  save -> load -> save is
byte-identical; a truncated file, a bad magic or a record that does not match
the model (name, shape, posit format) raises ValueError.

Host-side plumbing only: the codes are copied to / from the device tensors."""
from __future__ import annotations

import struct
from typing import Iterable

import numpy as np

MAGIC = b"PNN1"


def _code_bytes(nbits: int) -> int:
    return (nbits + 7) // 8


def dumps(records: Iterable[tuple[str, tuple[int, int], np.ndarray]]) -> bytes:
    """records: (name, (nbits, es), integer code array) -> file bytes."""
    out = [MAGIC]
    for name, (nbits, es), codes in records:
        if not (2 <= nbits <= 32) or es < 0:
            raise ValueError(f"{name}: bad posit format ({nbits},{es})")
        a = np.asarray(codes)
        nb = name.encode("utf-8")
        out.append(struct.pack("<I", len(nb)) + nb)
        out.append(struct.pack("<BBB", nbits, es, a.ndim))
        out.append(struct.pack(f"<{a.ndim}q", *a.shape))
        dt = {1: "<u1", 2: "<u2", 3: "<u4", 4: "<u4"}[_code_bytes(nbits)]
        mask = (1 << nbits) - 1
        vals = (a.astype(np.uint64) & np.uint64(mask)).astype(dt)
        raw = vals.tobytes()
        if _code_bytes(nbits) == 3:  # 3-byte codes: drop the high byte of each word
            raw = bytes(b for i, b in enumerate(raw) if i % 4 != 3)
        out.append(raw)
    return b"".join(out)


def loads(data: bytes) -> list[tuple[str, tuple[int, int], np.ndarray]]:
    if data[:4] != MAGIC:
        raise ValueError("not a PNN1 checkpoint (bad magic)")
    pos, recs = 4, []

    def take(n):
        nonlocal pos
        if pos + n > len(data):
            raise ValueError("truncated PNN1 checkpoint")
        b = data[pos:pos + n]
        pos += n
        return b

    while pos < len(data):
        (ln,) = struct.unpack("<I", take(4))
        name = take(ln).decode("utf-8")
        nbits, es, rank = struct.unpack("<BBB", take(3))
        shape = struct.unpack(f"<{rank}q", take(8 * rank)) if rank else ()
        if any(d < 0 for d in shape) or not (2 <= nbits <= 32):
            raise ValueError(f"{name}: corrupt record header")
        n = int(np.prod(shape, dtype=np.int64)) if rank else 1
        cb = _code_bytes(nbits)
        raw = take(n * cb)
        if cb == 3:
            raw = b"".join(raw[i:i + 3] + b"\x00" for i in range(0, len(raw), 3))
            cb = 4
        vals = np.frombuffer(raw, dtype={1: "<u1", 2: "<u2", 4: "<u4"}[cb]).astype(np.uint64)
        recs.append((name, (nbits, es), vals.reshape(shape)))
    return recs


def save_tensors(path: str, records) -> None:
    with open(path, "wb") as f:
        f.write(dumps(records))


def load_tensors(path: str):
    with open(path, "rb") as f:
        return loads(f.read())


def _param_records(model):
    from .codec import to_host

    recs = []
    for i, p in enumerate(model.params()):
        cfg = p.st.optimizer
        recs.append((f"param{i}", (cfg.nbits, cfg.es), to_host(p.master)))
    return recs


def save_model(model, path: str) -> None:
    """Master weights (p_optimizer codes) of every parameter, in order."""
    save_tensors(path, _param_records(model))


def load_model(model, path: str) -> None:
    """Restore the master weights in place (device tensors keep their storage,
    so a captured CUDA graph stays valid) and refresh every stage copy."""
    import torch

    from . import ops

    recs = load_tensors(path)
    params = model.params()
    if len(recs) != len(params):
        raise ValueError(f"checkpoint has {len(recs)} tensors, model {len(params)}")
    for i, ((name, fmt, codes), p) in enumerate(zip(recs, params)):
        cfg = p.st.optimizer
        if name != f"param{i}" or fmt != (cfg.nbits, cfg.es) or tuple(codes.shape) != p.shape:
            raise ValueError(f"checkpoint record {name} {fmt} {tuple(codes.shape)} does not match "
                             f"param{i} posit({cfg.nbits},{cfg.es}) {p.shape}")
    for (_, _, codes), p in zip(recs, params):
        cfg = p.st.optimizer
        p.master.copy_(torch.from_numpy(codes.astype(cfg.np_code_dtype)).to(p.master.device))
        for c in p.stage_formats():
            p.copies[c].copy_(ops.convert_tensor(p.master, cfg, c))
