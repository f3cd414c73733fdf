"""Training-step throughput on one B200 (BASELINE configs 0, 2, 3, 4) next to
the reference CPU implementation of the same step.

GPU: nn.train_step on device-resident packed codes (inputs generated once, as
in bench.py); CUDA events around K steps after W warm-up steps.
CPU reference: oracle/step.py composed from the UNMODIFIED reference
library's tensor kernels (oracle/_ref/libpnn_ref.so: conv2d, conv2d_input_grad,
conv2d_weight_grad, conv2d_bias_grad, maxpool2d(+backward), convert_tensor with
a ThreadPool of all host cores) plus the Appendix-A elementwise pieces from the
restatement -- one step, timed with time.perf_counter.

    python tools/bench_train.py [--configs 0,2,3,4] [--steps K] [--cpu]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle import bind  # noqa: E402
from oracle.step import CIFAR_CNN, LENET5, blob_images, oracle_step  # noqa: E402
from paper_2105_00053_b200 import codec, nn, ops  # noqa: E402

P80, P81, P121, P161 = ops.P80, ops.P81, ops.P121, ops.P161
# MACs per image of one training step (forward + input grads except layer 1 + weight grads)


def step_macs(layers, hw=32, cin=1):
    fwd = dgrad = wgrad = 0
    H = hw
    C = cin
    for L in layers:
        if L[0] == "conv":
            _, ci, co, k, s, p, first = L
            OH = (H + 2 * p - k) // s + 1
            m = OH * OH * co * ci * k * k
            fwd += m
            wgrad += m
            if not first:
                dgrad += m
            H, C = OH, co
        elif L[0] == "pool":
            H //= L[2]
        elif L[0] == "linear":
            _, fi, fo, first = L
            fwd += fi * fo
            wgrad += fi * fo
            if not first:
                dgrad += fi * fo
    return fwd + dgrad + wgrad


class HybridRef:
    """Tensor kernels from the reference library, Appendix-A pieces from the restatement."""

    def __init__(self, threads):
        self.ref = bind.Reference()
        self.po = bind.Restatement()
        self.t = threads

    def conv2d(self, n, es, x, w, b, s, p):
        return self.ref.conv2d(n, es, x, w, b, s, p, threads=self.t)

    def conv2d_input_grad(self, n, es, dy, w, xs, s, p):
        return self.ref.conv2d_input_grad(n, es, dy, w, xs, s, p, threads=self.t)

    def conv2d_weight_grad(self, n, es, dy, x, ws, s, p):
        return self.ref.conv2d_weight_grad(n, es, dy, x, ws, s, p, threads=self.t)

    def conv2d_bias_grad(self, n, es, dy):
        return self.ref.conv2d_bias_grad(n, es, dy)

    def maxpool2d(self, n, es, x, k, s):
        return self.ref.maxpool2d(n, es, x, k, s)

    def maxpool2d_backward(self, n, es, dy, am, xs):
        return self.ref.maxpool2d_backward(n, es, dy, am, xs)

    def convert_tensor(self, *a):
        return self.ref.convert_tensor(*a)

    def __getattr__(self, name):  # relu_fwd/bwd, softmax_xent, sgd, from_float64
        return getattr(self.po, name)


CONFIGS = {
    "0": dict(name="config0 LeNet-5 B=64 all posit(16,1)", layers="lenet",
              st=(P161, P161, P161, P161, P161), batch=64),
    "2": dict(name="config2 LeNet-5 B=256 fwd(8,0) bwd/grad(12,1) loss/opt(16,1)", layers="lenet",
              st=(P80, P121, P121, P161, P161), batch=256),
    "3": dict(name="config3 CIFAR CNN B=512 (1 GPU) fwd(8,1) grad(12,1) opt/loss(16,1)", layers="cifar",
              st=(P81, P121, P121, P161, P161), batch=512),
    "3b": dict(name="config3 formats, B=1024 (the bench.py training leg, 1 GPU)", layers="cifar",
               st=(P81, P121, P121, P161, P161), batch=1024),
    "4a": dict(name="config4 CIFAR CNN B=1024 (1 GPU) uniform posit(8,0)", layers="cifar",
               st=(P80,) * 5, batch=1024),
    "4b": dict(name="config4 CIFAR CNN B=1024 (1 GPU) uniform posit(8,1)", layers="cifar",
               st=(P81,) * 5, batch=1024),
    "4c": dict(name="config4 CIFAR CNN B=1024 (1 GPU) uniform posit(12,1)", layers="cifar",
               st=(P121,) * 5, batch=1024),
    "4d": dict(name="config4 CIFAR CNN B=1024 (1 GPU) uniform posit(16,1)", layers="cifar",
               st=(P161,) * 5, batch=1024),
}


def run(cfg_key, steps, warmup, cpu, graph=False):
    c = CONFIGS[cfg_key]
    st = nn.StagePrecisions(*c["st"])
    B = c["batch"]
    rng = np.random.default_rng(1)
    if c["layers"] == "lenet":
        model = nn.lenet5(st, seed=7)
        x = blob_images(3, B)[0] if cfg_key == "2" else rng.random((B, 1, 32, 32))
        layers, cin = LENET5, 1
    else:
        model = nn.cifar_cnn(st, seed=7)
        x = rng.uniform(-1.0, 1.0, (B, 3, 32, 32))
        layers, cin = CIFAR_CNN, 3
    labels = rng.integers(0, 10, B).astype(np.int32)
    xd = codec.from_float64_device(x, st.forward)
    lab = torch.from_numpy(labels).cuda()
    loss_fn = nn.CrossEntropyLoss(st)
    opt = nn.SGD(model.params(), 1.0 / 16, st)
    params0 = [(codec.to_host(l.w.master), codec.to_host(l.b.master))
               for l in model.layers if isinstance(l, nn.Conv2d)]
    g = nn.GraphedTrainStep(model, loss_fn, opt, xd, lab, B, warmup=1) if graph else None

    def one():
        return g.step() if g else nn.train_step(model, loss_fn, opt, xd, lab, B)

    for _ in range(max(warmup, 2 if graph else 0)):
        one()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    for _ in range(steps):
        one()
    e.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps
    dev_ms = s.elapsed_time(e) / steps
    macs = step_macs(layers, 32, cin) * B
    out = {"config": c["name"], "batch": B, "steps": steps, "cuda_graph": graph, "gpu_ms_per_step": dev_ms,
           "gpu_wall_ms_per_step": wall * 1e3, "images_per_s": B / (dev_ms / 1e3),
           "posit_mac_per_s": macs / (dev_ms / 1e3), "macs_per_step": macs}
    if cpu:
        threads = os.cpu_count() or 1
        h = HybridRef(threads)
        f = (st.forward.nbits, st.forward.es)
        xq = codec.to_host(codec.from_float64_device(x, st.forward))
        std = {k: (getattr(st, k).nbits, getattr(st, k).es)
               for k in ("forward", "backward", "gradient", "optimizer", "loss")}
        t0 = time.perf_counter()
        oracle_step(h, layers, std, params0, xq, labels, 1.0 / 16, B)
        tcpu = time.perf_counter() - t0
        out["cpu_reference"] = {"s_per_step": tcpu, "images_per_s": B / tcpu, "threads": threads,
                                "kind": "reference tensor kernels (oracle/_ref) + restated Appendix-A "
                                        "elementwise (oracle/posit_oracle.c)"}
        out["speedup_vs_cpu"] = tcpu / (dev_ms / 1e3)
        del f
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,2,3,4a,4b,4c,4d")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--graph", action="store_true", help="replay a CUDA-graph-captured step")
    a = ap.parse_args()
    for k in a.configs.split(","):
        print(json.dumps(run(k, a.steps, a.warmup, a.cpu and k in ("0", "2"), a.graph)), flush=True)


if __name__ == "__main__":
    main()
