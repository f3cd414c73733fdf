"""Data-parallel training through a real process group (the
overlapped exchange -- lanes packed on the compute stream as each layer's
backward finishes, all-reduced and rounded on a side stream -- was only ever
run with group=False or at world size 1).

* world 2 over gloo, two processes on the test box's one GPU: each rank runs
  dp.dp_train_step on its half of the batch with the real all-reduce; the
  final weights and the losses of every rank must equal the single-process
  step over the whole batch, bit for bit.
* world 2..N over NCCL with torchrun, eager and graph-captured (needs >= 2
  GPUs; skipped on a 1-GPU box).
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import dp_worker  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _check(out_dir, tag, want_losses, want_masters):
    got = np.load(os.path.join(out_dir, f"{tag}.npz"))
    assert got["losses"].tolist() == want_losses, tag
    for i, w in enumerate(want_masters):
        assert (got[f"m{i}"] == w).all(), (tag, i)


@pytest.mark.parametrize("model_name", ["lenet", "cifar"])
def test_dp_world2_gloo_equals_single_process(cuda, tmp_path, model_name):
    import torch.multiprocessing as mp

    world = 2
    mp.spawn(dp_worker.spawn_main, args=(world, _free_port(), str(tmp_path), model_name), nprocs=world,
             join=True)
    want_losses, want_masters = dp_worker.single_process(model_name)
    for r in range(world):
        _check(str(tmp_path), f"rank{r}_{model_name}_gloo", want_losses, want_masters)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="NCCL data parallelism needs >= 2 GPUs")
def test_dp_nccl_torchrun_eager_and_graph_equal_single_process(cuda, tmp_path):
    world = min(torch.cuda.device_count(), 8)
    while dp_worker.GLOBAL_B % world:
        world -= 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(HERE, "dp_worker.py"), str(tmp_path), "cifar"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    want_losses, want_masters = dp_worker.single_process("cifar")
    for rank in range(world):
        for mode in ("eager", "graph"):
            _check(str(tmp_path), f"rank{rank}_cifar_nccl_{mode}", want_losses, want_masters)
