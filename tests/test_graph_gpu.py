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
