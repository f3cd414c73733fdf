"""Data-parallel reduction on CPU: world_size-2 gloo processes.

Each rank accumulates the exact quire of its contiguous shard of a batch
reduction (the weight-gradient shape: per output, a dot product over the
batch), encodes it in 61-bit int64 lanes + a NaR lane (oracle/dp_ref.py,
the restatement of csrc/dp.cu), all-reduces with gloo SUM, carry-normalises
and rounds once.  The result must be bit-identical to the single-process
quire over the whole batch (the reference's conv2d_weight_grad semantics),
for every format of the configs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_00053_b200 import dp

FORMATS = [(8, 0), (8, 1), (12, 1), (16, 1)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(n, seed=0, outs=24, batch=96):
    rng = np.random.default_rng(seed + n)
    nar = 1 << (n - 1)
    a = rng.integers(0, 1 << n, (outs, batch)).astype(np.uint64)
    b = rng.integers(0, 1 << n, (outs, batch)).astype(np.uint64)
    a[a == nar] = 0
    b[b == nar] = 0
    a[5, 70] = nar  # one output carries a NaR term (in rank 1's shard)
    return a, b


def _rank_main(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import dp_ref
    from oracle.bind import Restatement

    po = Restatement()
    out = {}
    for (n, es) in FORMATS:
        W = 4 * ((n - 2) << es) + n
        a, b = _problem(n)
        lo, hi = dp.shard_bounds(a.shape[1], rank, world)
        vals, nars = [], []
        for o in range(a.shape[0]):
            q = po.quire(n, es)
            for k in range(lo, hi):
                q.add_product(int(a[o, k]), int(b[o, k]))
            v, nr = po.quire_words(q)
            vals.append(v)
            nars.append(nr)
        lanes = torch.tensor(dp_ref.words_to_lanes(vals, nars, W), dtype=torch.int64)
        dist.all_reduce(lanes, op=dist.ReduceOp.SUM)
        tv, tn = dp_ref.lanes_to_words(lanes.tolist(), W)
        out[(n, es)] = [(1 << (n - 1)) if nr else po.round_words(n, es, v) for v, nr in zip(tv, tn)]
    results[rank] = out
    dist.destroy_process_group()


def test_gloo_world2_quire_allreduce_bit_identical(po):
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_rank_main, args=(world, _free_port(), results), nprocs=world, join=True)
    for (n, es) in FORMATS:
        a, b = _problem(n)
        want = []
        for o in range(a.shape[0]):
            q = po.quire(n, es)
            for k in range(a.shape[1]):
                q.add_product(int(a[o, k]), int(b[o, k]))
            want.append(q.to_posit())
        for r in range(world):
            assert results[r][(n, es)] == want, (r, n, es)
        assert want[5] == 1 << (n - 1)


def test_shard_bounds_and_bucket_plan():
    assert dp.shard_bounds(512, 0, 8) == (0, 64)
    assert dp.shard_bounds(512, 7, 8) == (448, 512)
    with pytest.raises(ValueError):
        dp.shard_bounds(100, 0, 8)
    plan = dp.BucketPlan.build([150, 6, 2400, 16], 2)
    assert plan.offsets == [0, 150, 156, 2556] and plan.total == 2572 and plan.lanes == 3


def test_lane_counts_match_design():
    from oracle import dp_ref

    # (8,0) 1, (8,1) 1, (12,1) 2, (16,1) 3 lanes
    assert [dp_ref.lane_count(4 * ((n - 2) << es) + n) for n, es in FORMATS] == [1, 1, 2, 3]
    assert [dp.lanes_for(f) for f in FORMATS] == [1, 1, 2, 3]
    # 8 ranks of maximal 60-bit digits never overflow a signed int64 lane
    assert 8 * ((1 << 60) - 1) < (1 << 63)
