"""Per-pass device timings of the conv layers of the CIFAR CNN (BASELINE config
3/4 shapes) for the implicit (TMA gather) and explicit (im2col pack) paths.

  python tools/profile_conv.py [--batch 512] [--fmt 12,1] [--iters 20]

Prints one JSON line per (layer, pass, algo): device us per call (CUDA events,
warm, inputs resident), int8 tensor ops per call (MACs x D^2 x 2), and the
fraction of the measured int8 tensor peak (MEASURED_PEAKS / probe)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_00053_b200 import ops  # noqa: E402

# (name, C, H, F, K, pad) at input size H x H
LAYERS = [("conv1", 3, 32, 32, 3, 1), ("conv2", 32, 32, 32, 3, 1), ("conv3", 32, 16, 64, 3, 1),
          ("conv4", 64, 16, 64, 3, 1), ("fc1", 4096, 1, 512, 1, 0), ("fc2", 512, 1, 10, 1, 0)]
DIGITS = {(8, 0): 2, (8, 1): 4, (12, 1): 6, (16, 1): 8}


def rand_codes(rng, n, shape, dtype):
    c = rng.integers(0, 1 << n, size=shape)
    c[c == (1 << (n - 1))] = 0
    return torch.from_numpy(c.astype(dtype)).cuda()


def timed(fn, iters):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000.0 / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=512)
    ap.add_argument("--fmt", default="12,1")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--algos", default="0,1")
    ap.add_argument("--layers", default="")
    args = ap.parse_args()
    cfg = tuple(int(v) for v in args.fmt.split(","))
    n = cfg[0]
    dt = ops._cfg(cfg).np_code_dtype
    D = DIGITS.get(cfg, 0)
    import ctypes as C

    from paper_2105_00053_b200 import _native
    tops_c, ms_c = C.c_double(), C.c_double()
    peak = None
    if _native.lib().pnn_probe_int8_peak(20000, C.byref(tops_c), C.byref(ms_c)) == 0:
        peak = tops_c.value  # measured kind::i8 tcgen05 peak, TOP/s
    rng = np.random.default_rng(0)
    B = args.batch
    for name, C, H, F, K, p in LAYERS:
        if args.layers and name not in args.layers.split(","):
            continue
        x = rand_codes(rng, n, (B, C, H, H), dt)
        w = rand_codes(rng, n, (F, C, K, K), dt)
        b = rand_codes(rng, n, (F,), dt)
        OH = H + 2 * p - K + 1
        dy = rand_codes(rng, n, (B, F, OH, OH), dt)
        macs = B * F * OH * OH * C * K * K
        passes = [("fwd", lambda: ops.conv2d(cfg, x, w, b, 1, p)),
                  ("wgrad", lambda: ops.conv2d_weight_grad(cfg, dy, x, w.shape, 1, p))]
        if name != "conv1":
            passes.insert(1, ("dgrad", lambda: ops.conv2d_input_grad(cfg, dy, w, x.shape, 1, p)))
        for pname, fn in passes:
            for algo in (int(a) for a in args.algos.split(",")):
                prev = ops.conv_algo(algo)
                try:
                    us = timed(fn, args.iters)
                except Exception as e:  # ineligible when forced
                    us = None
                    err = str(e)[:60]
                finally:
                    ops.conv_algo(prev)
                tops = 2.0 * macs * D * D / (us * 1e-6) / 1e12 if us else None
                rec = {"layer": name, "pass": pname, "algo": ["auto", "explicit", "implicit"][algo],
                       "fmt": list(cfg), "batch": B, "us": us, "posit_macs": macs,
                       "int8_tops": tops, "frac_of_int8_peak": (tops / peak if (tops and peak) else None)}
                if us is None:
                    rec["error"] = err
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
