"""Rank body of the multi-process data-parallel tests (tests/test_dp_multiproc_gpu.py).

Each rank runs dp.dp_train_step -- raw quire words packed into int64 lanes as
each layer's backward finishes, all-reduced on a side stream through a REAL
process group, rounded once -- on its contiguous shard of a seeded global
batch, for `steps` steps, eager and (NCCL only: gloo collectives are host-side
and cannot be captured) replayed from a CUDA graph.  Rank 0 writes the final
master weights and losses to `<out>/rank0_<mode>.npz`; the test compares them
with a single-process nn.train_step over the whole batch.

Two launchers:
  * torch.multiprocessing.spawn(run, ...) with backend "gloo" -- both ranks on
    cuda:0 (the one GPU of the test box).  gloo moves the lanes through host
    memory; no kernel of one rank waits on another's (B200_PROFILING.md).
  * python -m torch.distributed.run --nproc-per-node N tests/dp_worker.py <out>
    with backend "nccl", one GPU per rank (needs >= 2 GPUs).
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GLOBAL_B = 64
STEPS = 2


def problem(model_name: str):
    """(stage precisions, model factory, inputs per step as float64, labels per step)."""
    from paper_2105_00053_b200 import nn, ops

    rng = np.random.default_rng(77)
    if model_name == "cifar":
        st = nn.StagePrecisions(ops.P81, ops.P121, ops.P121, ops.P161, ops.P161)
        xs = [rng.uniform(-1, 1, (GLOBAL_B, 3, 32, 32)) for _ in range(STEPS)]
        make = lambda dev: nn.cifar_cnn(st, seed=11, device=dev)  # noqa: E731
    else:
        st = nn.StagePrecisions.uniform(ops.P161)
        xs = [rng.random((GLOBAL_B, 1, 32, 32)) for _ in range(STEPS)]
        make = lambda dev: nn.lenet5(st, seed=11, device=dev)  # noqa: E731
    labels = [rng.integers(0, 10, GLOBAL_B).astype(np.int32) for _ in range(STEPS)]
    return st, make, xs, labels


def single_process(model_name: str, device="cuda"):
    """Reference run: nn.train_step over the whole batch on one device."""
    from paper_2105_00053_b200 import codec, nn

    st, make, xs, labels = problem(model_name)
    model = make(device)
    lf, opt = nn.CrossEntropyLoss(st), nn.SGD(model.params(), 1.0 / 16, st)
    losses = []
    for x, lab in zip(xs, labels):
        xd = codec.from_float64_device(x, st.forward)
        loss = nn.train_step(model, lf, opt, xd, torch.from_numpy(lab).to(device), GLOBAL_B)
        losses.append(int(codec.to_host(loss)[0]))
    return losses, [codec.to_host(p.master) for p in model.params()]


def run_rank(rank: int, world: int, model_name: str, graphed: bool, device: torch.device):
    from paper_2105_00053_b200 import codec, dp, nn

    st, make, xs, labels = problem(model_name)
    lo, hi = dp.shard_bounds(GLOBAL_B, rank, world)
    model = make(device)
    lf, opt = nn.CrossEntropyLoss(st), nn.SGD(model.params(), 1.0 / 16, st)
    red = dp.QuireAllReduce(model.params(), st.gradient, device=device)
    x_static = codec.from_float64_device(xs[0][lo:hi], st.forward).to(device)
    lab_static = torch.from_numpy(labels[0][lo:hi]).to(device)
    fn = lambda: dp.dp_train_step(model, lf, opt, red, x_static, lab_static, GLOBAL_B)  # noqa: E731
    step = nn.GraphedTrainStep(model, lf, opt, x_static, lab_static, GLOBAL_B, warmup=1,
                               step_fn=fn).step if graphed else fn
    losses = []
    for i in range(STEPS):
        x_static.copy_(codec.from_float64_device(xs[i][lo:hi], st.forward).to(device))
        lab_static.copy_(torch.from_numpy(labels[i][lo:hi]).to(device))
        loss = step()
        losses.append(int(codec.to_host(loss)[0]))
    torch.cuda.synchronize(device)
    return losses, [codec.to_host(p.master) for p in model.params()]


def save(out_dir: str, tag: str, losses, masters):
    np.savez(os.path.join(out_dir, f"{tag}.npz"), losses=np.array(losses, np.uint64),
             **{f"m{i}": m for i, m in enumerate(masters)})


def spawn_main(rank: int, world: int, port: int, out_dir: str, model_name: str):
    """torch.multiprocessing.spawn entry: gloo, every rank on cuda:0."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        losses, masters = run_rank(rank, world, model_name, False, dev)
        save(out_dir, f"rank{rank}_{model_name}_gloo", losses, masters)
    finally:
        dist.destroy_process_group()


def torchrun_main(out_dir: str, model_name: str):
    """torchrun entry: NCCL, one GPU per rank, eager then graph-captured."""
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    try:
        for graphed in (False, True):
            losses, masters = run_rank(rank, world, model_name, graphed, dev)
            save(out_dir, f"rank{rank}_{model_name}_nccl_{'graph' if graphed else 'eager'}", losses, masters)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    torchrun_main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "cifar")
