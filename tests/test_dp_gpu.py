"""Data-parallel exactness on one B200: the global batch is split into
`world` shards, each shard's backward runs in raw-quire mode on its own model
replica, the shards' lanes are summed (what NCCL all-reduce does across GPUs)
and rounded once -- gradients and loss must equal the single-process step
bit for bit, for 2, 4 and 8 simulated ranks.  (Multi-process NCCL needs more
than the one GPU this environment grants; the rank logic is covered by
tests/test_dp_cpu.py with gloo.)"""
import numpy as np
import pytest
import torch

from paper_2105_00053_b200 import codec, dp, nn, ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_raw_quire_sum_equals_full_batch(cuda, world):
    st = nn.StagePrecisions(ops.P80, ops.P121, ops.P121, ops.P161, ops.P161)
    B = 64
    rng = np.random.default_rng(world)
    x = codec.from_float64_device(rng.random((B, 1, 32, 32)), st.forward)
    labels = torch.from_numpy(rng.integers(0, 10, B).astype(np.int32)).cuda()
    ref = nn.lenet5(st, seed=3)
    loss_fn = nn.CrossEntropyLoss(st)
    ref_loss, dz = loss_fn(ref.forward(x), labels, B)
    ref.backward(dz)
    ref_grads = [codec.to_host(p.grad) for p in ref.params()]

    lanes_sum = None
    loss_lanes = None
    for r in range(world):
        lo, hi = dp.shard_bounds(B, r, world)
        rep = nn.lenet5(st, seed=3)
        _, dzr, word, nar = loss_fn(rep.forward(x[lo:hi]), labels[lo:hi], B, raw=True)
        rep.backward(dzr, raw=True)
        lanes = [ops.quire_to_lanes(st.gradient, p.grad_words, p.grad_nar) for p in rep.params()]
        ll = ops.quire_to_lanes(st.loss, word, nar)
        lanes_sum = lanes if lanes_sum is None else [a + b for a, b in zip(lanes_sum, lanes)]
        loss_lanes = ll if loss_lanes is None else loss_lanes + ll
    for i, (ls, want) in enumerate(zip(lanes_sum, ref_grads)):
        got = codec.to_host(ops.lanes_to_posit(st.gradient, ls)).reshape(want.shape)
        assert (got == want).all(), i
    lc = ops.lanes_to_posit(st.loss, loss_lanes)
    lb = int(np.log2(B))
    loss = ops.scalar_eval(st.loss, 7, lc.to(torch.int32), torch.full((1,), -lb, dtype=torch.int32, device="cuda"))
    assert int(codec.to_host(loss)[0]) & 0xFFFF == int(codec.to_host(ref_loss)[0])


def test_dp_train_step_world1_equals_train_step(cuda):
    st = nn.StagePrecisions.uniform(ops.P161)
    B = 32
    rng = np.random.default_rng(1)
    x = codec.from_float64_device(rng.random((B, 1, 32, 32)), st.forward)
    labels = torch.from_numpy(rng.integers(0, 10, B).astype(np.int32)).cuda()
    a, b = nn.lenet5(st, seed=9), nn.lenet5(st, seed=9)
    la = nn.train_step(a, nn.CrossEntropyLoss(st), nn.SGD(a.params(), 1 / 16, st), x, labels, B)
    red = dp.QuireAllReduce(b.params(), st.gradient, group=False)
    lb = dp.dp_train_step(b, nn.CrossEntropyLoss(st), nn.SGD(b.params(), 1 / 16, st), red, x, labels, B,
                          group=False)
    assert int(codec.to_host(la)[0]) == int(codec.to_host(lb)[0])
    for p, q in zip(a.params(), b.params()):
        assert (codec.to_host(p.master) == codec.to_host(q.master)).all()


@pytest.mark.parametrize("world", [1, 4])
def test_posit82_star_sharded_with_loss_scaling(cuda, world):
    """The posit(8,2)* preset: gradients go through (8,2) quire lanes; the
    posit(10,2) loss quire (W = 138) is wider than a raw word, so the loss
    rows are gathered and reduced once -- both equal the full-batch step."""
    st = nn.StagePrecisions.posit82_star()
    B, s = 64, 5
    rng = np.random.default_rng(world + 40)
    x = codec.from_float64_device(rng.random((B, 1, 32, 32)), st.forward)
    labels = torch.from_numpy(rng.integers(0, 10, B).astype(np.int32)).cuda()
    ref = nn.lenet5(st, seed=4)
    ref_loss = nn.train_step(ref, nn.CrossEntropyLoss(st, s), nn.SGD(ref.params(), 1 / 16, st, s), x, labels, B)

    reps, rows = [], []
    lanes_sum = None
    for r in range(world):
        lo, hi = dp.shard_bounds(B, r, world)
        rep = nn.lenet5(st, seed=4)
        lf = nn.CrossEntropyLoss(st, s)
        _, dzr, word, nar = lf(rep.forward(x[lo:hi]), labels[lo:hi], B, raw=True)
        assert word is None and nar is None
        rows.append(lf.rows)
        rep.backward(dzr, raw=True)
        lanes = [ops.quire_to_lanes(st.gradient, p.grad_words, p.grad_nar) for p in rep.params()]
        lanes_sum = lanes if lanes_sum is None else [a + b for a, b in zip(lanes_sum, lanes)]
        reps.append(rep)
    rep = reps[0]
    for p, ls in zip(rep.params(), lanes_sum):
        p.grad = ops.lanes_to_posit(st.gradient, ls).reshape(p.master.shape)
    nn.SGD(rep.params(), 1 / 16, st, s).step()
    loss = dp.gather_loss(st.loss, torch.cat(rows), B, group=False)
    assert int(codec.to_host(loss)[0]) == int(codec.to_host(ref_loss)[0])
    for p, q in zip(ref.params(), rep.params()):
        assert (codec.to_host(p.master) == codec.to_host(q.master)).all()
