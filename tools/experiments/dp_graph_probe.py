"""Probe (torchrun, any N): the data-parallel training step eager vs captured
in a CUDA graph (NCCL all-reduce inside), device ms/step, and bit-identity of
the two paths' weights after the same number of steps."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2105_00053_b200 import codec, dp, nn, ops  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
st = nn.StagePrecisions(ops.P81, ops.P121, ops.P121, ops.P161, ops.P161)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
rng = np.random.default_rng(3 + rank)
x = codec.from_float64_device(rng.uniform(-1.0, 1.0, (B, 3, 32, 32)), st.forward)
lab = torch.from_numpy(rng.integers(0, 10, B).astype(np.int32)).to(dev)


def make():
    model = nn.cifar_cnn(st, seed=7)
    loss_fn = nn.CrossEntropyLoss(st)
    opt = nn.SGD(model.params(), 1.0 / 16, st)
    red = dp.QuireAllReduce(model.params(), st.gradient)
    return model, loss_fn, opt, red


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


m1, l1, o1, r1 = make()
eager = timed(lambda: dp.dp_train_step(m1, l1, o1, r1, x, lab, B * world))
m2, l2, o2, r2 = make()
g = nn.GraphedTrainStep(m2, l2, o2, x, lab, B * world, warmup=1,
                        step_fn=lambda: dp.dp_train_step(m2, l2, o2, r2, x, lab, B * world))
graph = timed(g.step)
same = all((codec.to_host(p.master) == codec.to_host(q.master)).all()
           for p, q in zip(m1.params(), m2.params()))
if rank == 0:
    print(f"world={world} B/gpu={B}: eager {eager:.3f} ms/step, graph {graph:.3f} ms/step, "
          f"weights identical after 23 steps: {same}", flush=True)
dist.destroy_process_group()
