"""Dataset ingestion (semantics from the reference SPEC's
"data" module -- the reference has no loader code): MNIST / Fashion-MNIST IDX
files, CIFAR-10 binary batches, normalisation and seeded mini-batches quantised
to the forward posit format on the device.

Host-side plumbing.  The datasets are not in this container; the tests write
small synthetic files in the canonical formats."""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass

import numpy as np


@dataclass
class Dataset:
    images: np.ndarray  # float64 [N, C, H, W] staging, pixels / 255 in [0, 1]
    labels: np.ndarray  # int32 [N], 0..9
    split: str = "train"


def _read(path: str) -> bytes:
    with open(path, "rb") as f:
        return f.read()


def load_idx(images_path: str, labels_path: str, split: str = "train") -> Dataset:
    """Big-endian IDX: images magic 0x00000803 [N, 28, 28] ubyte, labels
    0x00000801 [N] ubyte.  Bad magic, truncation or a count mismatch raise."""
    im, lb = _read(images_path), _read(labels_path)
    if len(im) < 16 or struct.unpack(">I", im[:4])[0] != 0x803:
        raise ValueError("IDX images: bad magic")
    if len(lb) < 8 or struct.unpack(">I", lb[:4])[0] != 0x801:
        raise ValueError("IDX labels: bad magic")
    n, h, w = struct.unpack(">III", im[4:16])
    (nl,) = struct.unpack(">I", lb[4:8])
    if (h, w) != (28, 28):
        raise ValueError(f"IDX images: expected 28x28, got {h}x{w}")
    if n != nl:
        raise ValueError(f"IDX count mismatch: {n} images, {nl} labels")
    if len(im) < 16 + n * h * w or len(lb) < 8 + n:
        raise ValueError("IDX: truncated file")
    x = np.frombuffer(im, dtype=np.uint8, count=n * h * w, offset=16).reshape(n, 1, h, w)
    y = np.frombuffer(lb, dtype=np.uint8, count=n, offset=8).astype(np.int32)
    if (y > 9).any():
        raise ValueError("IDX labels outside 0..9")
    return Dataset(x.astype(np.float64) / 255.0, y, split)


CIFAR_RECORD = 1 + 3 * 32 * 32


def load_cifar10(paths, split: str = "train") -> Dataset:
    """CIFAR-10 binary batches: records of 1 label byte + 3072 pixel bytes
    (R, G, B planes of 32x32).  `paths`: a directory (data_batch_1..5.bin or
    test_batch.bin by split) or a list of files."""
    if isinstance(paths, str) and os.path.isdir(paths):
        names = ([f"data_batch_{i}.bin" for i in range(1, 6)] if split == "train"
                 else ["test_batch.bin"])
        paths = [os.path.join(paths, n) for n in names]
    xs, ys = [], []
    for p in paths:
        raw = _read(p)
        if len(raw) % CIFAR_RECORD:
            raise ValueError(f"{p}: size is not a multiple of the 3073-byte record")
        rec = np.frombuffer(raw, dtype=np.uint8).reshape(-1, CIFAR_RECORD)
        y = rec[:, 0].astype(np.int32)
        if (y > 9).any():
            raise ValueError(f"{p}: label outside 0..9")
        xs.append(rec[:, 1:].reshape(-1, 3, 32, 32))
        ys.append(y)
    return Dataset(np.concatenate(xs).astype(np.float64) / 255.0, np.concatenate(ys), split)


def normalize(ds: Dataset, mean, std) -> Dataset:
    """(x - mean) / std in float64 staging (per channel when mean/std are sequences)."""
    m = np.asarray(mean, dtype=np.float64).reshape(1, -1, 1, 1)
    s = np.asarray(std, dtype=np.float64).reshape(1, -1, 1, 1)
    return Dataset((ds.images - m) / s, ds.labels, ds.split)


def channel_stats(ds: Dataset):
    """Per-channel mean / std of a training split (the CIFAR-10 normalisation)."""
    return ds.images.mean(axis=(0, 2, 3)), ds.images.std(axis=(0, 2, 3))


def permutation(n: int, seed: int) -> np.ndarray:
    """Seeded Fisher-Yates shuffle (PCG64 draws), reproducible across runs."""
    rng = np.random.Generator(np.random.PCG64(seed))
    p = np.arange(n)
    for i in range(n - 1, 0, -1):
        j = int(rng.integers(0, i + 1))
        p[i], p[j] = p[j], p[i]
    return p


def batches(ds: Dataset, batch_size: int, seed: int, cfg, device="cuda"):
    """Mini-batches (posit codes in `cfg` on the device, int32 labels); the
    last partial batch is emitted with a smaller B.  Quantisation to posit is
    the only float -> posit boundary (from_float64 on the device)."""
    import torch

    from .codec import from_float64_device

    order = permutation(len(ds.labels), seed)
    for i in range(0, len(order), batch_size):
        idx = order[i:i + batch_size]
        x = from_float64_device(ds.images[idx], cfg)
        yield x, torch.from_numpy(ds.labels[idx].copy()).to(device)
