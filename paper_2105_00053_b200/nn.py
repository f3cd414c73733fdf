"""PyTorch-like layer / loss / optimizer API over the B200 quire kernels.

The reference ships this layer only as specification (the
files proj/src/layers.cpp, losses.cpp, optimizer.cpp, model.cpp are one-line
placeholders), so the semantics are the ones pinned in
SURVEY.md Appendix A and restated identically by the CPU oracle step
(oracle/step.py):

* StagePrecisions: p_forward, p_backward, p_gradient,
  p_optimizer, p_loss -- quires everywhere.
* MixedParam: master copy in p_optimizer, stage copies
  refreshed with convert after every update (Appendix A.6/A.7).
* Conv2d / Linear: bias inside the forward quire (tensor_ops.cpp:292,
  Appendix A.1); input grad in p_backward; weight / bias grads accumulated in
  p_gradient quires (operands converted to p_gradient).
* ReLU (A.2), MaxPool2d (A.3, reference kernel), Flatten (A.4),
  CrossEntropyLoss (A.5), SGD lr, momentum 0 (A.7), no input grad for the
  first layer (A.8).

Every tensor is a CUDA tensor of packed posit codes; every operation is a
libpnn_b200.so kernel.  Data-parallel training (dp.py) reuses the same layers
with the gradient reductions deferred to raw quire words.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .ops import PositConfig


@dataclass(frozen=True)
class StagePrecisions:
    forward: PositConfig
    backward: PositConfig
    gradient: PositConfig
    optimizer: PositConfig
    loss: PositConfig

    @staticmethod
    def uniform(cfg) -> "StagePrecisions":
        c = ops._cfg(cfg)
        return StagePrecisions(c, c, c, c, c)

    @staticmethod
    def posit82_star() -> "StagePrecisions":
        """posit(8,2)* = O12L10 (Table 4): optimizer
        posit(12,2), loss posit(10,2), everything else posit(8,2)."""
        return StagePrecisions(ops.P82, ops.P82, ops.P82, ops.P122, ops.P102)


class MixedParam:
    """Master copy in p_optimizer plus converted copies per stage format."""

    def __init__(self, master_codes: torch.Tensor, st: StagePrecisions):
        self.st = st
        self.master = master_codes
        self.copies: dict[PositConfig, torch.Tensor] = {}
        self.grad: torch.Tensor | None = None      # codes in p_gradient
        self.grad_words = None                      # raw quire words (data-parallel)
        self.grad_nar = None
        self.refresh()

    def stage_formats(self):
        st = self.st
        return sorted({st.forward, st.backward, st.gradient} - {st.optimizer},
                      key=lambda c: (c.nbits, c.es))

    def refresh(self):
        for cfg in self.stage_formats():
            self.copies[cfg] = ops.convert_tensor(self.master, self.st.optimizer, cfg)

    def as_(self, cfg: PositConfig) -> torch.Tensor:
        if cfg == self.st.optimizer:
            return self.master
        return self.copies[cfg]

    @property
    def shape(self):
        return tuple(self.master.shape)


def kaiming_uniform_codes(shape, fan_in, cfg: PositConfig, rng: np.random.Generator):
    """fp32 Kaiming-uniform U(-sqrt(6/fan_in), +sqrt(6/fan_in)) rounded to posit
    codes (Appendix A.9); generated on the host once, identical for the oracle."""
    from .codec import from_float64_array

    bound = np.float32(math.sqrt(6.0 / fan_in))
    w = rng.uniform(-1.0, 1.0, size=shape).astype(np.float32) * bound
    return from_float64_array(w.astype(np.float64), cfg)


class Module:
    training = True

    def params(self):
        return []


class Conv2d(Module):
    def __init__(self, cin, cout, k, st: StagePrecisions, stride=1, pad=0, rng=None,
                 first_layer=False, device="cuda"):
        self.cin, self.cout, self.k, self.stride, self.pad = cin, cout, k, stride, pad
        self.st = st
        self.first_layer = first_layer
        rng = rng or np.random.default_rng(0)
        fan_in = cin * k * k
        w = kaiming_uniform_codes((cout, cin, k, k), fan_in, st.optimizer, rng)
        b = np.zeros((cout,), np.uint64)
        dt = st.optimizer.np_code_dtype
        self.w = MixedParam(torch.from_numpy(w.astype(dt)).to(device), st)
        self.b = MixedParam(torch.from_numpy(b.astype(dt)).to(device), st)
        self.x = None
        self.saved = None

    def params(self):
        return [self.w, self.b]

    def forward_relu(self, x, want_pre=False):
        """This layer followed by a ReLU in one pass (relu fused into the GEMM
        epilogue): (relu(y), y if want_pre else None), or None when the
        geometry has no implicit forward (caller runs the two layers)."""
        f = self.st.forward
        n = ops.conv2d_saved_bytes(f, x.shape, self.w.shape, self.stride, self.pad) if self.training else 0
        saved = torch.empty(n, dtype=torch.uint8, device=x.device) if n else None
        res = ops.conv2d_fwd_layer(f, x, self.w.as_(f), self.b.as_(f), self.stride, self.pad, saved,
                                   relu=True, want_pre=want_pre)
        if res is None:
            return None
        self.x = x
        self.saved = saved
        return res

    def forward(self, x):
        f = self.st.forward
        self.x = x
        self.saved = None
        if self.training:
            # keep x's digit planes for the weight gradient (ops.conv2d_backward)
            n = ops.conv2d_saved_bytes(f, x.shape, self.w.shape, self.stride, self.pad)
            if n:
                self.saved = torch.empty(n, dtype=torch.uint8, device=x.device)
                return ops.conv2d_fwd_save(f, x, self.w.as_(f), self.b.as_(f), self.stride, self.pad,
                                           self.saved)
        return ops.conv2d(f, x, self.w.as_(f), self.b.as_(f), self.stride, self.pad)

    def backward_gated(self, dy, gate, raw=False, want_gated=False):
        """Backward of this layer and the ReLU after it in one pass (the ReLU's
        gate applied in the digitisers and in the bias-gradient sum): dy = the
        ReLU's output gradient, gate = the ReLU's forward output.  Returns (dx,
        the ReLU's input gradient if want_gated else None) or None when the
        fused path is not eligible."""
        st = self.st
        g = st.gradient
        bias_direct = st.backward == g  # bias grad straight from (dy, gate), nothing materialised
        res = ops.conv2d_backward_gated(st.forward, st.backward, g, dy, gate, self.x, self.saved,
                                        None if self.first_layer else self.w.as_(st.backward),
                                        self.x.shape, self.w.shape, self.stride, self.pad,
                                        need_dx=not self.first_layer, raw=raw,
                                        want_gated=want_gated or not bias_direct)
        if res is None:
            return None
        self.saved = None
        dx, dw, dyb = res
        bg = ops.conv2d_bias_grad_gated(g, dy, st.forward, gate, raw=raw) if bias_direct else None
        if bg is None:
            if dyb is None:
                dyb = ops.relu_bwd(st.forward, gate, st.backward, dy)
            bg = ops.conv2d_bias_grad(g, ops.convert_tensor(dyb, st.backward, g), raw=raw)
        if raw:
            _, self.w.grad_words, self.w.grad_nar = dw
            _, self.b.grad_words, self.b.grad_nar = bg
        else:
            self.w.grad = dw
            self.b.grad = bg
        return dx, dyb

    def backward(self, dy, raw=False):
        """dy in p_backward -> dx in p_backward (None for the first layer)."""
        st = self.st
        g = st.gradient
        dyg = ops.convert_tensor(dy, st.backward, g)
        fused = ops.conv2d_backward(st.forward, st.backward, g, dy, self.x, self.saved,
                                    None if self.first_layer else self.w.as_(st.backward),
                                    self.x.shape, self.w.shape, self.stride, self.pad,
                                    need_dx=not self.first_layer, raw=raw)
        self.saved = None
        if fused is not None:
            dx, dw = fused
            if raw:
                _, self.w.grad_words, self.w.grad_nar = dw
                _, self.b.grad_words, self.b.grad_nar = ops.conv2d_bias_grad(g, dyg, raw=True)
            else:
                self.w.grad = dw
                self.b.grad = ops.conv2d_bias_grad(g, dyg)
            return dx
        xg = ops.convert_tensor(self.x, st.forward, g)
        if raw:
            _, self.w.grad_words, self.w.grad_nar = ops.conv2d_weight_grad(
                g, dyg, xg, self.w.shape, self.stride, self.pad, raw=True)
            _, self.b.grad_words, self.b.grad_nar = ops.conv2d_bias_grad(g, dyg, raw=True)
        else:
            self.w.grad = ops.conv2d_weight_grad(g, dyg, xg, self.w.shape, self.stride, self.pad)
            self.b.grad = ops.conv2d_bias_grad(g, dyg)
        if self.first_layer:
            return None
        return ops.conv2d_input_grad(st.backward, dy, self.w.as_(st.backward), self.x.shape,
                                     self.stride, self.pad)


class Linear(Conv2d):
    """y = round(x W^T + b): the 1x1 convolution of [B, in, 1, 1] (Appendix A.1)."""

    def __init__(self, fin, fout, st, rng=None, first_layer=False, device="cuda"):
        super().__init__(fin, fout, 1, st, rng=rng, first_layer=first_layer, device=device)

    def forward(self, x):
        B = x.shape[0]
        return super().forward(x.reshape(B, -1, 1, 1)).reshape(B, -1)

    def backward(self, dy, raw=False):
        B = dy.shape[0]
        dx = super().backward(dy.reshape(B, -1, 1, 1), raw=raw)
        return None if dx is None else dx.reshape(B, -1)


class ReLU(Module):
    def __init__(self, st: StagePrecisions):
        self.st = st
        self.x = None

    def forward(self, x):
        self.x = x
        return ops.relu_fwd(self.st.forward, x)

    def backward(self, dy, raw=False):
        return ops.relu_bwd(self.st.forward, self.x, self.st.backward, dy)


class MaxPool2d(Module):
    def __init__(self, k, st: StagePrecisions, stride=None):
        self.k, self.stride, self.st = k, stride or k, st
        self.argmax = None
        self.x = None
        self.x_shape = None

    def forward(self, x):
        self.x_shape = x.shape
        self.x = self.argmax = None
        y = ops.maxpool2d_noidx(self.st.forward, x, self.k, self.stride)
        if y is not None:  # 2x2 tiled: keep x, recompute the argmax in backward
            self.x = x
            return y
        y, self.argmax = ops.maxpool2d(self.st.forward, x, self.k, self.stride)
        return y

    def backward_relu(self, dy, relu):
        """Backward of this pool and the ReLU before it in one pass (the pool's
        input is that ReLU's output); None when the pool keeps an argmax."""
        if self.x is None or relu.x is None or (relu.x is not self.x and relu.x.data_ptr() != self.x.data_ptr()):
            return None
        return ops.maxpool2d_backward_x(self.st.forward, self.x, self.st.backward, dy, self.k, self.stride,
                                        relu_gate=True)

    def backward(self, dy, raw=False):
        if self.x is not None:
            return ops.maxpool2d_backward_x(self.st.forward, self.x, self.st.backward, dy, self.k,
                                            self.stride)
        return ops.maxpool2d_backward(self.st.backward, dy, self.argmax, self.x_shape, self.k,
                                      self.stride)


class _Act(Module):
    kind = 0

    def __init__(self, st: StagePrecisions):
        self.st = st
        self.y = None

    def forward(self, x):
        self.y = ops.act_fwd(self.kind, self.st.forward, x)
        return self.y

    def backward(self, dy, raw=False):
        return ops.act_bwd(self.kind, self.st.forward, self.y, self.st.backward, dy)


class Tanh(_Act):
    """tanh_posit layer (posit_math.cpp:109-118); backward dy*(1 - y*y) in p_backward."""
    kind = ops.ACT_TANH


class Sigmoid(_Act):
    """sigmoid_posit layer (posit_math.cpp:120-130); backward dy*(y*(1 - y))."""
    kind = ops.ACT_SIGMOID


class AvgPool2d(Module):
    """avgpool2d / avgpool2d_backward (tensor_ops.cpp:672-720), quire window
    sum times 1/k^2 quantised in the forward / backward format."""

    def __init__(self, k, st: StagePrecisions, stride=None):
        from .codec import from_float64_array

        self.k, self.stride, self.st = k, stride or k, st
        r = np.array([1.0 / (k * k)])
        self.recip_f = int(from_float64_array(r, st.forward)[0])
        self.recip_b = int(from_float64_array(r, st.backward)[0])
        self.x_shape = None

    def forward(self, x):
        self.x_shape = x.shape
        return ops.avgpool2d(self.st.forward, x, self.k, self.stride, True, self.recip_f)

    def backward(self, dy, raw=False):
        return ops.avgpool2d_backward(self.st.backward, dy, self.k, self.stride, self.x_shape,
                                      self.recip_b)


class Dropout(Module):
    """Seeded dropout: the mask of step t uses seed + t, t a
    device counter advanced after every training forward (so a captured CUDA
    graph draws a fresh mask per replay); identity in eval mode."""

    def __init__(self, p, st: StagePrecisions, seed=0, device="cuda"):
        from .codec import from_float64_array

        self.p, self.st, self.seed = p, st, int(seed)
        self.thresh = ops.dropout_threshold(p)
        s = np.array([1.0 / (1.0 - p)])
        self.scale_f = int(from_float64_array(s, st.forward)[0])
        self.scale_b = int(from_float64_array(s, st.backward)[0])
        self.counter = torch.zeros((1,), dtype=torch.int64, device=device)
        self.cur = None
        self.used = False

    def forward(self, x):
        if not self.training:
            self.used = False
            return x
        self.cur = self.counter.clone()
        self.counter.add_(1)
        self.used = True
        return ops.dropout(self.st.forward, x, self.seed, self.thresh, self.scale_f, self.cur)

    def backward(self, dy, raw=False):
        if not self.used:
            return dy
        return ops.dropout(self.st.backward, dy, self.seed, self.thresh, self.scale_b, self.cur)


class BatchNorm2d(Module):
    """Per-channel batch normalisation (rounding sequence in
    oracle/layers_oracle.c): gamma / beta are MixedParams (master in
    p_optimizer), running mean / variance live in p_optimizer.  Works on
    [N, C, H, W] and on [N, C] (BatchNorm1d after a Linear)."""

    def __init__(self, C, st: StagePrecisions, eps=1e-5, momentum=0.1, device="cuda"):
        from .codec import from_float64_array

        self.C, self.st = C, st
        dt = st.optimizer.np_code_dtype
        one = from_float64_array(np.ones(C), st.optimizer).astype(dt)
        self.gamma = MixedParam(torch.from_numpy(one).to(device), st)
        self.beta = MixedParam(torch.zeros((C,), dtype=st.optimizer.code_dtype, device=device), st)
        self.running_mean = torch.zeros((C,), dtype=st.optimizer.code_dtype, device=device)
        self.running_var = torch.from_numpy(one.copy()).to(device)
        self.eps_code = int(from_float64_array(np.array([eps]), st.forward)[0])
        self.mom_code = int(from_float64_array(np.array([momentum]), st.optimizer)[0])
        self.xhat = self.inv = None

    def params(self):
        return [self.gamma, self.beta]

    def forward(self, x):
        f = self.st.forward
        y, self.xhat, self.inv = ops.batchnorm_fwd(f, x, self.gamma.as_(f), self.beta.as_(f), self.eps_code,
                                                   self.training, self.st.optimizer, self.running_mean,
                                                   self.running_var, self.mom_code)
        return y

    def backward(self, dy, raw=False):
        st = self.st
        out = ops.batchnorm_bwd(st.forward, self.xhat, self.inv, st.backward, dy,
                                self.gamma.as_(st.backward), st.gradient, raw=raw)
        if raw:
            dx, (self.gamma.grad_words, self.gamma.grad_nar), (self.beta.grad_words, self.beta.grad_nar) = out
        else:
            dx, self.gamma.grad, self.beta.grad = out
        return dx


class Flatten(Module):
    def __init__(self):
        self.shape = None

    def forward(self, x):
        self.shape = x.shape
        return x.reshape(x.shape[0], -1)

    def backward(self, dy, raw=False):
        return dy.reshape(self.shape)


class CrossEntropyLoss(Module):
    """Softmax cross-entropy in p_loss (Appendix A.5); the gradient is already
    divided by the GLOBAL batch (2^-log2_batch).  grad_scale_log2 = s scales
    the logit gradient by 2^s (loss scaling, SPEC scale_gradients); pair it
    with SGD(..., grad_scale_log2=s), which unscales in p_optimizer."""

    def __init__(self, st: StagePrecisions, grad_scale_log2: int = 0):
        self.st = st
        self.grad_scale_log2 = int(grad_scale_log2)
        self._side = None
        self._pending = False

    def join(self):
        """Make the current stream wait for a deferred loss (see defer=True)."""
        if self._pending:
            torch.cuda.current_stream().wait_stream(self._side)
            self._pending = False

    def __call__(self, logits_fwd, labels, global_batch: int, raw=False, defer=False):
        """defer=True: the logit gradient is computed on the current stream and
        the loss (per-row log, quire sum) on a side stream, off the backward
        pass's critical path; call join() before reading the loss."""
        lb = int(round(math.log2(global_batch)))
        if 1 << lb != global_batch:
            raise ValueError("global batch must be a power of two (Appendix A.5)")
        z = ops.convert_tensor(logits_fwd, self.st.forward, self.st.loss)
        if defer:
            raw_words = raw and ops.quire_bits(self.st.loss) <= 128
            d, srows = ops.softmax_xent_grad(self.st.loss, z, labels, lb, self.grad_scale_log2)
            cur = torch.cuda.current_stream(z.device)
            if self._side is None:
                self._side = torch.cuda.Stream(device=z.device)
            self._side.wait_stream(cur)
            with torch.cuda.stream(self._side):
                out = ops.softmax_xent_loss(self.st.loss, z, labels, srows, lb, raw=raw_words)
            for t in (z, srows, labels):
                t.record_stream(self._side)
            self._pending = True
            self.rows = out[1]
            dz = ops.convert_tensor(d, self.st.loss, self.st.backward)
            if raw_words:
                return out[0], dz, out[2], out[3]
            if raw:
                return out[0], dz, None, None
            return out[0], dz
        # raw quire words need W <= 128; wider loss quires (posit(10,2)) hand
        # the data-parallel path the loss rows instead (word = nar = None)
        raw_words = raw and ops.quire_bits(self.st.loss) <= 128
        out = ops.softmax_xent(self.st.loss, z, labels, lb, raw=raw_words,
                               grad_scale_log2=self.grad_scale_log2)
        self.rows = out[2]
        dz = ops.convert_tensor(out[1], self.st.loss, self.st.backward)
        if raw_words:
            loss, _, rows, word, nar = out
            return loss, dz, word, nar
        if raw:
            return out[0], dz, None, None
        return out[0], dz


class MSELoss(Module):
    """Mean squared error against one-hot targets in p_loss (
    rounding sequence in oracle/layers_oracle.c): loss = sum (z - t)^2 / G,
    dlogits = (z - t) * (2 / G) with G = global batch x classes."""

    def __init__(self, st: StagePrecisions, grad_scale_log2: int = 0):
        self.st = st
        self.grad_scale_log2 = int(grad_scale_log2)
        self._onehot = {}

    def targets(self, labels, classes: int):
        from .codec import from_float64_array

        key = (classes, labels.device)
        if key not in self._onehot:
            one = int(from_float64_array(np.array([1.0]), self.st.loss)[0])
            self._onehot[key] = torch.tensor([0, one], dtype=torch.int64, device=labels.device)
        return self._onehot[key][torch.nn.functional.one_hot(labels.long(), classes)].to(
            self.st.loss.code_dtype)

    def join(self):  # the MSE loss is computed in line (no deferred work)
        pass

    def __call__(self, logits_fwd, labels, global_batch: int, raw=False, defer=False):
        if raw:
            raise NotImplementedError("MSELoss has no data-parallel (raw) mode")
        B, classes = logits_fwd.shape
        z = ops.convert_tensor(logits_fwd, self.st.forward, self.st.loss)
        loss, g = ops.mse(self.st.loss, z, self.targets(labels, classes), global_batch * classes,
                          self.grad_scale_log2)
        return loss, ops.convert_tensor(g, self.st.loss, self.st.backward)


class Sequential(Module):
    def __init__(self, *layers):
        self.layers = list(layers)

    def train(self, mode: bool = True):
        for l in self.layers:
            l.training = mode
        return self

    def eval(self):
        return self.train(False)

    def params(self):
        return [p for l in self.layers for p in l.params()]

    def forward(self, x, record=None):
        i, n = 0, len(self.layers)
        self._relu_fused = set()  # indices of ReLU layers fused into the preceding Conv2d
        while i < n:
            l = self.layers[i]
            nxt = self.layers[i + 1] if i + 1 < n else None
            if type(l) is Conv2d and type(nxt) is ReLU:
                # Conv2d + ReLU in one GEMM epilogue; the ReLU layer's backward gate
                # reads relu(y) (positive(relu(v)) == positive(v), relu(NaR) = 0)
                res = l.forward_relu(x, want_pre=record is not None)
                if res is not None:
                    y, pre = res
                    nxt.x = y
                    self._relu_fused.add(i + 1)
                    if record is not None:
                        record[f"act{i}"] = pre
                        record[f"act{i + 1}"] = y
                    x = y
                    i += 2
                    continue
            x = l.forward(x)
            if record is not None:
                record[f"act{i}"] = x
            i += 1
        return x

    # Backward of a fused Conv2d + ReLU pair through Conv2d.backward_gated (the
    # ReLU gate applied inside the dy digitiser and the bias-gradient sum) is
    # bit-identical but measured slower on B200 than the vectorised relu_bwd
    # kernel followed by the conv backward (config-3 step 2.94 -> 3.04 ms: the
    # gate tests cost more ALU in those two kernels than the 5 B/element
    # relu_bwd pass), so it is off by default.
    fuse_relu_backward = False

    def backward(self, dy, raw=False, record=None, on_layer=None):
        """on_layer(layer): called once each parameter-holding layer's gradients
        exist (the data-parallel exchange starts there, dp.QuireAllReduce)."""
        fused = getattr(self, "_relu_fused", set()) if self.fuse_relu_backward else set()
        notify = (lambda l: on_layer(l) if l.params() else None) if on_layer is not None else (lambda l: None)
        i = len(self.layers) - 1
        while i >= 0:
            if i in fused:  # ReLU i fused with Conv2d i-1: one backward, gate in the digitisers
                res = self.layers[i - 1].backward_gated(dy, self.layers[i].x, raw=raw,
                                                        want_gated=record is not None)
                if res is not None:
                    notify(self.layers[i - 1])
                    dx, dy_relu = res
                    if record is not None:
                        record[f"dact{i}"] = dy_relu
                    dy = dx
                    if dy is None:
                        break
                    if record is not None:
                        record[f"dact{i - 1}"] = dy
                    i -= 2
                    continue
            if (record is None and isinstance(self.layers[i], MaxPool2d) and i >= 1
                    and type(self.layers[i - 1]) is ReLU):
                # ReLU -> MaxPool: one backward pass (the pool's input is the ReLU's output)
                d2 = self.layers[i].backward_relu(dy, self.layers[i - 1])
                if d2 is not None:
                    dy = d2
                    i -= 2
                    continue
            dy = self.layers[i].backward(dy, raw=raw)
            notify(self.layers[i])
            if dy is None:
                break
            if record is not None:
                record[f"dact{i}"] = dy
            i -= 1
        return dy


class SGD:
    """master = sub(master, mul(lr, convert(grad -> p_opt))), copies refreshed
    (Appendix A.7; momentum 0)."""

    def __init__(self, params, lr: float, st: StagePrecisions, grad_scale_log2: int = 0,
                 momentum: float = 0.0):
        from .codec import from_float64_array

        self.params = params
        self.st = st
        self.grad_scale_log2 = int(grad_scale_log2)
        self.momentum = float(momentum)
        if self.momentum:
            self.mu_code = int(from_float64_array(np.array([momentum]), st.optimizer)[0])
            self.velocity = [torch.zeros_like(p.master) for p in params]
        self.lr_code = int(from_float64_array(np.array([lr]), st.optimizer)[0])

    def step(self):
        st = self.st
        if not self.momentum and self.params:
            # one launch for the whole model (all parameters share the stage formats)
            fmts = self.params[0].stage_formats()
            if all(p.stage_formats() == fmts for p in self.params):
                fused = fmts[:2]
                ops.sgd_step_multi(st.optimizer, st.gradient, self.lr_code, [p.master for p in self.params],
                                   [p.grad for p in self.params], fused,
                                   [tuple(p.copies[c] for c in fused) for p in self.params],
                                   self.grad_scale_log2)
                for p in self.params:
                    for c in fmts[2:]:
                        p.copies[c] = ops.convert_tensor(p.master, st.optimizer, c)
                return
        for i, p in enumerate(self.params):
            fmts = p.stage_formats()
            fused = [(c, p.copies[c]) for c in fmts[:2]]  # refreshed inside the SGD kernel
            if self.momentum:
                ops.sgd_step_momentum(st.optimizer, p.master, self.velocity[i], st.gradient, p.grad,
                                      self.lr_code, self.mu_code, fused, self.grad_scale_log2)
            else:
                ops.sgd_step(st.optimizer, p.master, st.gradient, p.grad, self.lr_code, fused,
                             grad_scale_log2=self.grad_scale_log2)
            for c in fmts[2:]:
                p.copies[c] = ops.convert_tensor(p.master, st.optimizer, c)


def lenet5(st: StagePrecisions, seed: int = 0, device="cuda") -> Sequential:
    """LeNet-5 of BASELINE configs 0/2: conv 1->6 5x5, ReLU, maxpool 2, conv
    6->16 5x5, ReLU, maxpool 2, Linear 400->120->84->10 with ReLU."""
    rng = np.random.default_rng(seed)
    return Sequential(
        Conv2d(1, 6, 5, st, rng=rng, first_layer=True, device=device), ReLU(st), MaxPool2d(2, st),
        Conv2d(6, 16, 5, st, rng=rng, device=device), ReLU(st), MaxPool2d(2, st), Flatten(),
        Linear(400, 120, st, rng=rng, device=device), ReLU(st),
        Linear(120, 84, st, rng=rng, device=device), ReLU(st),
        Linear(84, 10, st, rng=rng, device=device))


def cifar_cnn(st: StagePrecisions, seed: int = 0, device="cuda") -> Sequential:
    """CIFAR-shape CNN of BASELINE configs 3/4 (Appendix A.10): conv 3->32 3x3
    pad 1, ReLU, conv 32->32, ReLU, maxpool; conv 32->64, ReLU, conv 64->64,
    ReLU, maxpool; Linear 4096->512, ReLU, 512->10."""
    rng = np.random.default_rng(seed)
    return Sequential(
        Conv2d(3, 32, 3, st, pad=1, rng=rng, first_layer=True, device=device), ReLU(st),
        Conv2d(32, 32, 3, st, pad=1, rng=rng, device=device), ReLU(st), MaxPool2d(2, st),
        Conv2d(32, 64, 3, st, pad=1, rng=rng, device=device), ReLU(st),
        Conv2d(64, 64, 3, st, pad=1, rng=rng, device=device), ReLU(st), MaxPool2d(2, st),
        Flatten(), Linear(4096, 512, st, rng=rng, device=device), ReLU(st),
        Linear(512, 10, st, rng=rng, device=device))


def lenet5_classic(st: StagePrecisions, seed: int = 0, device="cuda") -> Sequential:
    """The original LeNet-5 activations (SPEC Fig. 2 layer set): tanh and
    average pooling, sigmoid before the classifier."""
    rng = np.random.default_rng(seed)
    return Sequential(
        Conv2d(1, 6, 5, st, rng=rng, first_layer=True, device=device), Tanh(st), AvgPool2d(2, st),
        Conv2d(6, 16, 5, st, rng=rng, device=device), Tanh(st), AvgPool2d(2, st), Flatten(),
        Linear(400, 120, st, rng=rng, device=device), Tanh(st),
        Linear(120, 84, st, rng=rng, device=device), Sigmoid(st),
        Linear(84, 10, st, rng=rng, device=device))


def cnn_bn_dropout(st: StagePrecisions, seed: int = 0, device="cuda", hw: int = 32) -> Sequential:
    """A CIFAR-shape CNN (hw x hw inputs) with batch normalisation (2-D and
    1-D) and dropout."""
    rng = np.random.default_rng(seed)
    return Sequential(
        Conv2d(3, 32, 3, st, pad=1, rng=rng, first_layer=True, device=device), BatchNorm2d(32, st, device=device),
        ReLU(st), MaxPool2d(2, st),
        Conv2d(32, 32, 3, st, pad=1, rng=rng, device=device), BatchNorm2d(32, st, device=device), ReLU(st),
        MaxPool2d(2, st), Flatten(),
        Linear(32 * (hw // 4) ** 2, 64, st, rng=rng, device=device), BatchNorm2d(64, st, device=device),
        ReLU(st),
        Dropout(0.25, st, seed=seed + 1, device=device),
        Linear(64, 10, st, rng=rng, device=device))


def train_step(model: Sequential, loss_fn: CrossEntropyLoss, opt: SGD, x_fwd, labels,
               global_batch: int, record=None):
    """One SGD step on one device; returns the loss code tensor [1] (p_loss)."""
    logits = model.forward(x_fwd, record)
    loss, dz = loss_fn(logits, labels, global_batch, defer=True)  # loss beside the backward
    if record is not None:
        record["dlogits"] = dz
    model.backward(dz, record=record)
    if record is not None:
        for i, p in enumerate([q for q in model.params()]):
            record[f"grad_{'wb'[i % 2]}{i // 2}"] = p.grad
    opt.step()
    loss_fn.join()
    return loss


class GraphedTrainStep:
    """One training step captured as a CUDA graph (every kernel of forward,
    loss, backward and SGD on one stream; no host round trips), replayed per
    step.  Feed new data by copying into ``x`` / ``labels`` before ``step()``.
    The first call runs ``warmup`` eager steps (sizing workspaces), then
    captures; each capture/replay is a real, bit-identical training step."""

    def __init__(self, model: Sequential, loss_fn: CrossEntropyLoss, opt: SGD, x_static, labels_static,
                 global_batch: int, warmup: int = 1, step_fn=None):
        self.model, self.loss_fn, self.opt = model, loss_fn, opt
        self.x, self.labels, self.B = x_static, labels_static, global_batch
        self.warmup = warmup
        self.graph = None
        self.loss = None
        # step_fn: the step to capture (default: train_step on this device; the
        # data-parallel step passes dp.dp_train_step -- its NCCL all-reduce is
        # captured into the same graph)
        self.step_fn = step_fn or (lambda: train_step(self.model, self.loss_fn, self.opt, self.x,
                                                      self.labels, self.B))

    def step(self):
        if self.graph is None:
            if self.warmup > 0:
                self.warmup -= 1
                return self.step_fn()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s), torch.cuda.graph(self.graph, stream=s):
                self.loss = self.step_fn()
            torch.cuda.current_stream().wait_stream(s)
        self.graph.replay()
        return self.loss


def layer_description(model: Sequential):
    """The oracle-step layer list (oracle/step.py) of a model."""
    out = []
    for l in model.layers:
        if isinstance(l, Linear):
            out.append(("linear", l.cin, l.cout, l.first_layer))
        elif isinstance(l, Conv2d):
            out.append(("conv", l.cin, l.cout, l.k, l.stride, l.pad, l.first_layer))
        elif isinstance(l, ReLU):
            out.append(("relu",))
        elif isinstance(l, MaxPool2d):
            out.append(("pool", l.k, l.stride))
        elif isinstance(l, Flatten):
            out.append(("flatten",))
        elif isinstance(l, Tanh):
            out.append(("tanh",))
        elif isinstance(l, Sigmoid):
            out.append(("sigmoid",))
        elif isinstance(l, AvgPool2d):
            out.append(("avgpool", l.k, l.stride))
        elif isinstance(l, Dropout):
            # the seed the NEXT training forward will use
            step = int(l.counter.item()) if l.training else None
            out.append(("dropout", l.p, None if step is None else l.seed + step))
        elif isinstance(l, BatchNorm2d):
            out.append(("bn", l.training))
        else:
            raise TypeError(f"no oracle description for {type(l).__name__}")
    return out
