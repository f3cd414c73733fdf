"""Generate the committed golden fixtures from the UNMODIFIED reference.

Runs here (where /root/reference exists): builds oracle/_ref/libpnn_ref.so
from the reference's own sources (oracle/Makefile) and records its outputs on
seeded inputs into tests/golden/*.npz.  The GPU box has no /root/reference;
tests there read only these fixtures and the prebuilt libraries.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import bind  # noqa: E402

FORMATS = [(8, 0), (8, 1), (8, 2), (12, 1), (16, 1)]


def rand_codes(rng, n, shape, nar_ok=False):
    c = rng.integers(0, 1 << n, shape).astype(np.uint64)
    if not nar_ok:
        c[c == (1 << (n - 1))] = 0
    return c


def main():
    bind.build(reference=True)
    ref = bind.Reference()
    rng = np.random.default_rng(20210430)
    out = {}
    # quire GEMM (matmul_quire, tensor_ops.cpp:166-185), ragged shapes
    for (n, es) in FORMATS:
        for (m, k, nn) in [(1, 1, 1), (5, 7, 6), (33, 57, 29), (130, 300, 140)]:
            A = rand_codes(rng, n, (m, k))
            B = rand_codes(rng, n, (k, nn))
            key = f"gemm_{n}_{es}_{m}x{k}x{nn}"
            out[key + "_A"], out[key + "_B"] = A, B
            out[key + "_C"] = ref.matmul(n, es, A, B)
        # NaR-carrying case
        A = rand_codes(rng, n, (17, 40), nar_ok=True)
        B = rand_codes(rng, n, (40, 19), nar_ok=True)
        A[3, 5] = 1 << (n - 1)
        B[7, 11] = 1 << (n - 1)
        A[4, :] = 0
        A[4, 9] = 1 << (n - 1)
        key = f"gemmnar_{n}_{es}"
        out[key + "_A"], out[key + "_B"] = A, B
        out[key + "_C"] = ref.matmul(n, es, A, B)
    # conv2d family (tensor_ops.cpp:494-618), LeNet/CIFAR-like small shapes
    for (n, es) in FORMATS:
        for (N, Cc, H, W, F, K, s, p) in [(2, 1, 12, 12, 3, 5, 1, 0), (2, 3, 8, 8, 4, 3, 1, 1),
                                          (1, 2, 9, 7, 3, 3, 2, 1)]:
            x = rand_codes(rng, n, (N, Cc, H, W))
            w = rand_codes(rng, n, (F, Cc, K, K))
            b = rand_codes(rng, n, (F,))
            y = ref.conv2d(n, es, x, w, b, s, p)
            dy = rand_codes(rng, n, y.shape)
            key = f"conv_{n}_{es}_{N}x{Cc}x{H}x{W}_{F}x{K}_s{s}p{p}"
            out[key + "_x"], out[key + "_w"], out[key + "_b"], out[key + "_y"] = x, w, b, y
            out[key + "_dy"] = dy
            out[key + "_dx"] = ref.conv2d_input_grad(n, es, dy, w, x.shape, s, p)
            out[key + "_dw"] = ref.conv2d_weight_grad(n, es, dy, x, w.shape, s, p)
            out[key + "_db"] = ref.conv2d_bias_grad(n, es, dy)
    # convert_tensor over every code (posit.cpp:487-495)
    for (sn, se, dn, de) in [(16, 1, 12, 1), (12, 1, 8, 1), (12, 1, 8, 0), (8, 0, 12, 1),
                             (16, 1, 8, 0), (8, 1, 16, 1)]:
        x = np.arange(1 << sn, dtype=np.uint64)
        out[f"convert_{sn}_{se}_{dn}_{de}"] = ref.convert_tensor(sn, se, dn, de, x)
    path = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
