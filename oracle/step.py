"""CPU oracle of one training step (TEST INFRASTRUCTURE ONLY).

The reference has no layer / loss / optimizer code (layers.cpp, losses.cpp,
optimizer.cpp, model.cpp are placeholders), so a training
step's semantics are pinned once, here, from SURVEY.md Appendix A and
composed purely from the oracle's restatement of the reference's tensor
kernels (oracle/posit_oracle.c -- conv2d / conv2d_input_grad /
conv2d_weight_grad / conv2d_bias_grad / maxpool2d(+backward) /
convert_tensor, tensor_ops.cpp) plus the Appendix-A scalar pieces (ReLU,
softmax cross-entropy, SGD) restated in the same C file.

A layer description is a list of tuples:
    ("conv", cin, cout, k, stride, pad, first_layer)   ("linear", fin, fout, first_layer)
    ("relu",)   ("pool", k, stride)   ("flatten",)
    ("tanh",)  ("sigmoid",)  ("avgpool", k, stride)  ("dropout", p, seed)  ("bn", training)
Params are host uint64 code arrays in the optimizer format, one (w, b) pair
per conv / linear (and one (gamma, beta) pair per bn), in order.
"""
from __future__ import annotations

import math

import numpy as np

LENET5 = [("conv", 1, 6, 5, 1, 0, True), ("relu",), ("pool", 2, 2),
          ("conv", 6, 16, 5, 1, 0, False), ("relu",), ("pool", 2, 2), ("flatten",),
          ("linear", 400, 120, False), ("relu",), ("linear", 120, 84, False), ("relu",),
          ("linear", 84, 10, False)]

CIFAR_CNN = [("conv", 3, 32, 3, 1, 1, True), ("relu",), ("conv", 32, 32, 3, 1, 1, False), ("relu",),
             ("pool", 2, 2), ("conv", 32, 64, 3, 1, 1, False), ("relu",),
             ("conv", 64, 64, 3, 1, 1, False), ("relu",), ("pool", 2, 2), ("flatten",),
             ("linear", 4096, 512, False), ("relu",), ("linear", 512, 10, False)]


def _cv(po, src, dst, x):
    """convert_tensor (same format returns the input, tensor_ops.cpp:808)."""
    if tuple(src) == tuple(dst):
        return x
    return po.convert_tensor(*src, *dst, x)


def _onehot(po, lf, labels, classes):
    one = po.from_float64(*lf, 1.0)
    t = np.zeros((len(labels), classes), np.uint64)
    t[np.arange(len(labels)), labels] = one
    return t


def oracle_step(po, layers, st, params, x, labels, lr, global_batch, record=None, grad_scale_log2=0,
                state=None, loss="xent", momentum=0.0, velocity=None):
    """One SGD step.  st = dict(forward, backward, gradient, optimizer, loss) of
    (nbits, es); x = input codes in the forward format; returns (loss_code,
    new_params, grads) and fills ``record`` (if given) with every activation
    and gradient, keyed like the GPU model's recording.  grad_scale_log2 = s:
    loss scaling by 2^s (dlogits carry 2^s, SGD unscales).

    §8f.2 layers (rounding sequences in oracle/layers_oracle.c):
    ("tanh",) ("sigmoid",) ("avgpool", k, stride) ("dropout", p, seed or None
    in eval) ("bn", training) -- a bn layer owns a (gamma, beta) params pair
    and ``state[layer index] = [running_mean, running_var]`` (updated in
    place).  loss: "xent" (softmax cross-entropy) or "mse" (one-hot targets).
    momentum != 0: ``velocity`` = one [vw, vb] list per params pair, updated
    in place (SGD with momentum)."""
    f, b, g, o, lf = (tuple(st[k]) for k in ("forward", "backward", "gradient", "optimizer", "loss"))
    lb = int(round(math.log2(global_batch)))
    rec = record if record is not None else {}
    caches = []
    h = x
    pi = 0
    for li, L in enumerate(layers):
        kind = L[0]
        if kind in ("conv", "linear"):
            w, bias = params[pi]
            pi += 1
            if kind == "conv":
                _, cin, cout, k, s, p, first = L
                xin = h
            else:
                _, fin, fout, first = L
                k, s, p = 1, 1, 0
                xin = h.reshape(h.shape[0], -1, 1, 1)
            y = po.conv2d(*f, xin, _cv(po, o, f, w), _cv(po, o, f, bias), s, p)
            caches.append((kind, xin, w, (k, s, p), first, h.shape))
            h = y if kind == "conv" else y.reshape(y.shape[0], -1)
        elif kind == "relu":
            caches.append(("relu", h))
            h = po.relu_fwd(*f, h)
        elif kind == "pool":
            _, k, s = L
            y, am = po.maxpool2d(*f, h, k, s)
            caches.append(("pool", h.shape, am))
            h = y
        elif kind == "flatten":
            caches.append(("flatten", h.shape))
            h = h.reshape(h.shape[0], -1)
        elif kind in ("tanh", "sigmoid"):
            h = po.act_fwd(1 if kind == "tanh" else 2, *f, h)
            caches.append((kind, h))
        elif kind == "avgpool":
            _, k, s = L
            caches.append(("avgpool", h.shape, k, s))
            h = po.avgpool2d(*f, h, k, s, True, po.from_float64(*f, 1.0 / (k * k)))
        elif kind == "dropout":
            _, p, seed = L
            if seed is None:
                caches.append(("dropout", None, None))
            else:
                thresh = int(p * 4294967296.0)
                caches.append(("dropout", seed, thresh, p))
                h = po.dropout(*f, h, seed, thresh, po.from_float64(*f, 1.0 / (1.0 - p)))
        elif kind == "bn":
            gamma, beta = params[pi]
            rs = state[li]
            y, xh, inv, rm, rv = po.batchnorm_fwd(
                f, h, _cv(po, o, f, gamma), _cv(po, o, f, beta), po.from_float64(*f, 1e-5), L[1], o,
                rs[0], rs[1], po.from_float64(*o, 0.1))
            rs[0], rs[1] = rm, rv
            caches.append(("bn", pi, gamma, xh, inv))
            pi += 1
            h = y
        rec[f"act{li}"] = h
    z = _cv(po, f, lf, h)
    if loss == "mse":
        Bn, classes = z.shape
        lw, d = po.mse(*lf, z, _onehot(po, lf, labels, classes), global_batch * classes, grad_scale_log2)
    else:
        lw, d, rows = po.softmax_xent(*lf, z, labels, lb, grad_scale_log2)
        rec["loss_rows"] = rows
    dy = _cv(po, lf, b, d)
    rec["dlogits"] = dy
    grads = [None] * len(params)
    for li in range(len(layers) - 1, -1, -1):
        c = caches[li]
        kind = c[0]
        if kind in ("conv", "linear"):
            pi -= 1
            _, xin, w, (k, s, p), first, in_shape = c
            dy4 = dy if kind == "conv" else dy.reshape(dy.shape[0], -1, 1, 1)
            dyg = _cv(po, b, g, dy4)
            xg = _cv(po, f, g, xin)
            dw = po.conv2d_weight_grad(*g, dyg, xg, w.shape, s, p)
            db = po.conv2d_bias_grad(*g, dyg)
            grads[pi] = (dw, db)
            rec[f"grad_w{pi}"], rec[f"grad_b{pi}"] = dw, db
            if first:
                break
            dx = po.conv2d_input_grad(*b, dy4, _cv(po, o, b, w), xin.shape, s, p)
            dy = dx if kind == "conv" else dx.reshape(in_shape)
        elif kind == "relu":
            dy = po.relu_bwd(*f, c[1], dy)
        elif kind == "pool":
            dy = po.maxpool2d_backward(*b, dy, c[2], c[1])
        elif kind == "flatten":
            dy = dy.reshape(c[1])
        elif kind in ("tanh", "sigmoid"):
            dy = po.act_bwd(1 if kind == "tanh" else 2, f, c[1], b, dy)
        elif kind == "avgpool":
            _, shape, k, s = c
            dy = po.avgpool2d_backward(*b, dy, k, s, shape, po.from_float64(*b, 1.0 / (k * k)))
        elif kind == "dropout":
            if c[1] is not None:
                dy = po.dropout(*b, dy, c[1], c[2], po.from_float64(*b, 1.0 / (1.0 - c[3])))
        elif kind == "bn":
            _, bpi, gamma, xh, inv = c
            pi = bpi
            dy, dgm, dbt = po.batchnorm_bwd(f, xh, inv, b, dy, _cv(po, o, b, gamma), g)
            grads[bpi] = (dgm, dbt)
            rec[f"grad_w{bpi}"], rec[f"grad_b{bpi}"] = dgm, dbt
        rec[f"dact{li}"] = dy
    lr_code = po.from_float64(*o, lr)
    new_params = []
    if momentum:
        mu = po.from_float64(*o, momentum)
        for i, ((w, bias), (dw, db)) in enumerate(zip(params, grads)):
            w2, velocity[i][0] = po.sgd_momentum(o, w, velocity[i][0], g, dw, lr_code, mu, grad_scale_log2)
            b2, velocity[i][1] = po.sgd_momentum(o, bias, velocity[i][1], g, db, lr_code, mu, grad_scale_log2)
            new_params.append((w2, b2))
    else:
        for (w, bias), (dw, db) in zip(params, grads):
            new_params.append((po.sgd(*o, w, *g, dw, lr_code, grad_scale_log2),
                               po.sgd(*o, bias, *g, db, lr_code, grad_scale_log2)))
    return lw, new_params, grads


def blob_images(seed: int, n: int, classes: int = 10, shape=(1, 32, 32), sigma: float = 0.3):
    """Config-2 synthetic data: per-class Gaussian blobs (sigma 0.3) clipped to
    [0, 1): class centres uniform in [0,1)^shape from the seed."""
    rng = np.random.default_rng(seed)
    centres = rng.random((classes,) + tuple(shape))
    labels = rng.integers(0, classes, n)
    x = centres[labels] + sigma * rng.standard_normal((n,) + tuple(shape))
    x = np.clip(x, 0.0, np.nextafter(1.0, 0.0))
    return x, labels.astype(np.int32)
