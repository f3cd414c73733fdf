"""Model checkpoints in the "PNN1" format (the format is
specified only in the reference's SPEC, "External Interfaces": magic "PNN1",
then per-tensor records {name length + bytes, nbits, es, rank, extents, raw bit
patterns packed little-endian in ceil(nbits/8) bytes each}).

Field widths (the SPEC leaves them open; fixed here): name length uint32 LE,
name UTF-8, nbits uint8, es uint8, rank uint8, extents int64 LE, then the codes.
Records follow each other to the end of the file.  save_model() adds a config
record (meta.stage_precisions: (nbits, es) of the five stages) checked on
load, and the momentum velocities of an SGD optimizer (meta.sgd + velocityI).  save -> load -> save is
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


STAGES = ("forward", "backward", "gradient", "optimizer", "loss")
META_STAGES = "meta.stage_precisions"   # uint8 [5, 2]: (nbits, es) per stage, STAGES order
META_SGD = "meta.sgd"                   # uint8 [1]: 1 = momentum velocity records follow


def _model_stages(model):
    params = model.params()
    sts = {tuple((getattr(p.st, k).nbits, getattr(p.st, k).es) for k in STAGES) for p in params}
    if len(sts) != 1:
        raise ValueError("model parameters disagree on their stage precisions")
    return np.array(sorted(sts)[0], np.uint64).ravel()


def _records(model, optimizer=None):
    from .codec import to_host

    recs = [(META_STAGES, (8, 0), _model_stages(model))]
    params = model.params()
    for i, p in enumerate(params):
        cfg = p.st.optimizer
        recs.append((f"param{i}", (cfg.nbits, cfg.es), to_host(p.master)))
    vel = getattr(optimizer, "velocity", None) if optimizer is not None and optimizer.momentum else None
    recs.append((META_SGD, (8, 0), np.array([1 if vel is not None else 0], np.uint64)))
    if vel is not None:
        for i, (p, v) in enumerate(zip(params, vel)):
            cfg = p.st.optimizer
            recs.append((f"velocity{i}", (cfg.nbits, cfg.es), to_host(v)))
    return recs


def save_model(model, path: str, optimizer=None) -> None:
    """Stage precisions of the model (a config record checked on load), the
    master weights (p_optimizer codes) of every parameter in order, and -- for
    an SGD with momentum -- its velocity tensors, so training resumes bit-exactly."""
    save_tensors(path, _records(model, optimizer))


def load_model(model, path: str, optimizer=None) -> None:
    """Restore the master weights in place (device tensors keep their storage,
    so a captured CUDA graph stays valid) and refresh every stage copy.  A
    checkpoint written for other stage precisions, another architecture, or
    without the velocity a momentum optimizer needs is rejected (ValueError)."""
    import torch

    from . import ops

    recs = load_tensors(path)
    params = model.params()
    byname = {}
    for name, fmt, codes in recs:
        if name in byname:
            raise ValueError(f"checkpoint record {name} appears twice")
        byname[name] = (fmt, codes)
    if META_STAGES in byname:  # files written before the config record carry none
        got = byname[META_STAGES][1].ravel()
        want = _model_stages(model)
        if got.shape != want.shape or (got != want).any():
            raise ValueError(f"checkpoint stage precisions {got.reshape(-1, 2).tolist()} differ from the "
                             f"model's {want.reshape(-1, 2).tolist()} ({', '.join(STAGES)})")
    weights = [r for r in recs if r[0].startswith("param")]
    if len(weights) != len(params):
        raise ValueError(f"checkpoint has {len(weights)} tensors, model {len(params)}")
    for i, ((name, fmt, codes), p) in enumerate(zip(weights, params)):
        cfg = p.st.optimizer
        if name != f"param{i}" or fmt != (cfg.nbits, cfg.es) or tuple(codes.shape) != p.shape:
            raise ValueError(f"checkpoint record {name} {fmt} {tuple(codes.shape)} does not match "
                             f"param{i} posit({cfg.nbits},{cfg.es}) {p.shape}")
    has_vel = META_SGD in byname and int(byname[META_SGD][1].ravel()[0]) == 1
    want_vel = optimizer is not None and bool(optimizer.momentum)
    if want_vel and not has_vel:
        raise ValueError("checkpoint has no momentum velocity for this optimizer")
    if want_vel:
        for i, p in enumerate(params):
            rec = byname.get(f"velocity{i}")
            cfg = p.st.optimizer
            if rec is None or rec[0] != (cfg.nbits, cfg.es) or tuple(rec[1].shape) != p.shape:
                raise ValueError(f"checkpoint velocity{i} missing or does not match param{i}")
    for (_, _, codes), p in zip(weights, params):
        cfg = p.st.optimizer
        p.master.copy_(torch.from_numpy(codes.astype(cfg.np_code_dtype)).to(p.master.device))
        for c in p.stage_formats():
            p.copies[c].copy_(ops.convert_tensor(p.master, cfg, c))
    if want_vel:
        for i, (p, v) in enumerate(zip(params, optimizer.velocity)):
            codes = byname[f"velocity{i}"][1]
            v.copy_(torch.from_numpy(codes.astype(p.st.optimizer.np_code_dtype)).to(v.device))
