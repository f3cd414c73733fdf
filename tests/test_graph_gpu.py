"""A CUDA-graph-captured training step is the same computation: after 4 steps
(1 eager warm-up + capture + replays) weights and loss equal 4 eager steps."""
import numpy as np
import pytest
import torch

from paper_2105_00053_b200 import codec, nn, ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mixed", [False, True])
def test_graphed_step_bit_identical(cuda, mixed):
    st = (nn.StagePrecisions(ops.P80, ops.P121, ops.P121, ops.P161, ops.P161) if mixed
          else nn.StagePrecisions.uniform(ops.P161))
    B = 64
    rng = np.random.default_rng(12)
    x = codec.from_float64_device(rng.random((B, 1, 32, 32)), st.forward)
    lab = torch.from_numpy(rng.integers(0, 10, B).astype(np.int32)).cuda()
    a, b = nn.lenet5(st, seed=4), nn.lenet5(st, seed=4)
    la_fn, lb_fn = nn.CrossEntropyLoss(st), nn.CrossEntropyLoss(st)
    oa, ob = nn.SGD(a.params(), 1 / 16, st), nn.SGD(b.params(), 1 / 16, st)
    g = nn.GraphedTrainStep(b, lb_fn, ob, x, lab, B, warmup=1)
    for _ in range(4):
        la = nn.train_step(a, la_fn, oa, x, lab, B)
        lb = g.step()
    torch.cuda.synchronize()
    assert int(codec.to_host(la)[0]) == int(codec.to_host(lb)[0])
    for p, q in zip(a.params(), b.params()):
        assert (codec.to_host(p.master) == codec.to_host(q.master)).all()


def test_graphed_dp_step_bit_identical(cuda):
    """The data-parallel step (raw quire words -> lanes -> NCCL all-reduce ->
    round once) captured in a CUDA graph equals the eager step, bit for bit
    (world size 1 on the test box; the same capture runs per rank under torchrun)."""
    import os

    import torch.distributed as dist

    from paper_2105_00053_b200 import dp

    own = not dist.is_initialized()
    if own:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        st = nn.StagePrecisions(ops.P81, ops.P121, ops.P121, ops.P161, ops.P161)
        B = 64
        rng = np.random.default_rng(21)
        x = codec.from_float64_device(rng.uniform(-1, 1, (B, 3, 32, 32)), st.forward)
        lab = torch.from_numpy(rng.integers(0, 10, B).astype(np.int32)).cuda()
        runs = []
        for graphed in (False, True):
            model = nn.cifar_cnn(st, seed=5)
            lf, opt = nn.CrossEntropyLoss(st), None
            opt = nn.SGD(model.params(), 1 / 16, st)
            red = dp.QuireAllReduce(model.params(), st.gradient)
            fn = lambda: dp.dp_train_step(model, lf, opt, red, x, lab, B)  # noqa: E731
            step = nn.GraphedTrainStep(model, lf, opt, x, lab, B, warmup=1, step_fn=fn).step if graphed else fn
            for _ in range(4):
                loss = step()
            torch.cuda.synchronize()
            runs.append((int(codec.to_host(loss)[0]), [codec.to_host(p.master) for p in model.params()]))
        assert runs[0][0] == runs[1][0]
        for a, b in zip(runs[0][1], runs[1][1]):
            assert (a == b).all()
    finally:
        if own:
            dist.destroy_process_group()
