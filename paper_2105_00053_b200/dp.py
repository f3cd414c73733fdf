"""Data-parallel training over 1/2/4/8 GPUs of one node.

One process per GPU (torchrun; torch.distributed over NCCL for the plumbing).
The global batch is split contiguously across ranks.  Forward, input-grad and
the elementwise kernels are per-sample; the only exchange is the batch sum
of the weight / bias gradients and of the loss, which every rank emits as
UNROUNDED quire words (raw mode of conv2d_weight_grad / bias_grad /
softmax_xent).  Those are packed into 60-bit int64 lanes
(pnn_quire_to_lanes), summed with one NCCL all-reduce per bucket, carry-
normalised and rounded once (pnn_lanes_to_posit): bit-identical to the
single-process reference for any rank count, because the quire is exact and
addition mod 2^W is associative.  The SGD update is then replicated.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _native, nn, ops


def shard_bounds(global_batch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous batch shard [lo, hi) of this rank (equal shards)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if global_batch % world:
        raise ValueError("global batch must divide evenly across ranks")
    per = global_batch // world
    return rank * per, (rank + 1) * per


def lanes_for(cfg) -> int:
    cfg = ops._cfg(cfg)
    L = _native.lib().pnn_quire_lanes(cfg.nbits, cfg.es)
    if L <= 0:
        raise _native.PnnError(2, f"no quire lanes for posit({cfg.nbits},{cfg.es})")
    return L


@dataclass
class BucketPlan:
    """Where each parameter's lanes live inside the flat all-reduce buffer."""
    lanes: int                 # L + 1 int64 per element
    offsets: list[int]         # element offset per parameter
    numels: list[int]
    total: int                 # elements

    @staticmethod
    def build(numels: list[int], L: int) -> "BucketPlan":
        offs, acc = [], 0
        for n in numels:
            offs.append(acc)
            acc += n
        return BucketPlan(L + 1, offs, list(numels), acc)


class QuireAllReduce:
    """Sum the ranks' raw gradient quires of every parameter, round once.

    Overlapped use (dp_train_step): the backward pass hands over each layer as
    soon as its raw gradient words exist (``layer_ready``); that layer's lanes
    are packed on the compute stream and all-reduced + rounded on a side
    stream while the backward of the earlier layers runs (the Linear layers,
    ~97% of the CIFAR CNN's parameters, finish first).  ``reduce`` then joins
    and handles whatever was not handed over.  Same bits either way: each
    parameter's sum is exact and rounded once."""

    def __init__(self, params, grad_cfg, group=None, device="cuda"):
        self.params = params
        self.cfg = ops._cfg(grad_cfg)
        self.L = lanes_for(self.cfg)
        self.plan = BucketPlan.build([p.master.numel() for p in params], self.L)
        self.buf = torch.empty((self.plan.total, self.plan.lanes), dtype=torch.int64, device=device)
        self.group = group
        self._index = {id(p): i for i, p in enumerate(params)}
        self._done = set()
        self._comm = None

    def _distributed(self):
        return (self.group is not False and torch.distributed.is_available()
                and torch.distributed.is_initialized())

    def _pack(self, i, sp):
        p, off, n = self.params[i], self.plan.offsets[i], self.plan.numels[i]
        _native.check(_native.lib().pnn_quire_to_lanes(self.cfg.nbits, self.cfg.es, p.grad_words.data_ptr(),
                                                       p.grad_nar.data_ptr(), n, self.buf[off:off + n].data_ptr(),
                                                       sp))

    def _unpack(self, i, sp):
        p, off, n = self.params[i], self.plan.offsets[i], self.plan.numels[i]
        g = torch.empty(p.master.shape, dtype=self.cfg.code_dtype, device=self.buf.device)
        _native.check(_native.lib().pnn_lanes_to_posit(self.cfg.nbits, self.cfg.es,
                                                       self.buf[off:off + n].data_ptr(), n, g.data_ptr(), None,
                                                       sp))
        p.grad = g

    def layer_ready(self, layer):
        """Start the exchange of one layer's parameters (called by the backward)."""
        idx = sorted(self._index[id(q)] for q in layer.params() if id(q) in self._index)
        if not idx or any(i in self._done for i in idx):
            return
        cur = torch.cuda.current_stream(self.buf.device)
        for i in idx:
            self._pack(i, cur.cuda_stream)
        if self._comm is None:
            self._comm = torch.cuda.Stream(device=self.buf.device)
        self._comm.wait_stream(cur)
        lo = self.plan.offsets[idx[0]]
        hi = self.plan.offsets[idx[-1]] + self.plan.numels[idx[-1]]
        contiguous = all(self.plan.offsets[b] == self.plan.offsets[a] + self.plan.numels[a]
                         for a, b in zip(idx, idx[1:]))
        with torch.cuda.stream(self._comm):
            if self._distributed():
                if contiguous:
                    torch.distributed.all_reduce(self.buf[lo:hi], op=torch.distributed.ReduceOp.SUM,
                                                 group=self.group)
                else:
                    for i in idx:
                        o, n = self.plan.offsets[i], self.plan.numels[i]
                        torch.distributed.all_reduce(self.buf[o:o + n], op=torch.distributed.ReduceOp.SUM,
                                                     group=self.group)
            for i in idx:
                self._unpack(i, self._comm.cuda_stream)
        self._done.update(idx)

    def reduce(self):
        sp = ops._stream_ptr(self.buf.device)
        rest = [i for i in range(len(self.params)) if i not in self._done]
        for i in rest:
            self._pack(i, sp)
        if rest and self._distributed():
            if len(rest) == len(self.params):  # nothing handed over: one all-reduce of the buffer
                torch.distributed.all_reduce(self.buf, op=torch.distributed.ReduceOp.SUM, group=self.group)
            else:
                for i in rest:
                    o, n = self.plan.offsets[i], self.plan.numels[i]
                    torch.distributed.all_reduce(self.buf[o:o + n], op=torch.distributed.ReduceOp.SUM,
                                                 group=self.group)
        for i in rest:
            self._unpack(i, sp)
        if self._comm is not None and self._done:
            torch.cuda.current_stream(self.buf.device).wait_stream(self._comm)
        self._done = set()


def reduce_loss(loss_cfg, word, nar, global_batch: int, group=None):
    """All-reduce the raw loss quire word, round once, ldexp by -log2(B)."""
    cfg = ops._cfg(loss_cfg)
    L = lanes_for(cfg)
    lib = _native.lib()
    lanes = torch.empty((1, L + 1), dtype=torch.int64, device=word.device)
    sp = ops._stream_ptr(word.device)
    _native.check(lib.pnn_quire_to_lanes(cfg.nbits, cfg.es, word.data_ptr(), nar.data_ptr(), 1,
                                         lanes.data_ptr(), sp))
    if group is not False and torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.all_reduce(lanes, op=torch.distributed.ReduceOp.SUM, group=group)
    code = torch.empty((1,), dtype=cfg.code_dtype, device=word.device)
    _native.check(lib.pnn_lanes_to_posit(cfg.nbits, cfg.es, lanes.data_ptr(), 1, code.data_ptr(), None, sp))
    lb = int(round(math.log2(global_batch)))
    return ops.scalar_eval(cfg, 7, code.to(torch.int32),
                           torch.full((1,), -lb, dtype=torch.int32, device=word.device)).to(cfg.code_dtype)


def gather_loss(loss_cfg, rows, global_batch: int, group=None):
    """All-gather every rank's per-sample loss rows (rank order = batch
    order) and reduce them once: the exact quire sum is order-independent, so
    this equals the single-process loss for any rank count."""
    full = rows
    if group is not False and torch.distributed.is_available() and torch.distributed.is_initialized():
        world = torch.distributed.get_world_size(group)
        full = torch.empty((rows.numel() * world,), dtype=rows.dtype, device=rows.device)
        torch.distributed.all_gather_into_tensor(full, rows.contiguous(), group=group)
    return ops.loss_reduce(loss_cfg, full, int(round(math.log2(global_batch))))


def dp_train_step(model: nn.Sequential, loss_fn: nn.CrossEntropyLoss, opt: nn.SGD, reducer: QuireAllReduce,
                  x_shard, labels_shard, global_batch: int, group=None):
    """One data-parallel SGD step on this rank's shard; returns the global loss."""
    logits = model.forward(x_shard)
    _, dz, word, nar = loss_fn(logits, labels_shard, global_batch, raw=True, defer=True)
    model.backward(dz, raw=True, on_layer=reducer.layer_ready)  # exchange overlaps the backward
    reducer.reduce()
    loss_fn.join()  # the loss words / rows were computed beside the backward pass
    if word is None:  # loss quire wider than the 128-bit raw word
        loss = gather_loss(loss_fn.st.loss, loss_fn.rows, global_batch, group)
    else:
        loss = reduce_loss(loss_fn.st.loss, word, nar, global_batch, group)
    opt.step()
    return loss
