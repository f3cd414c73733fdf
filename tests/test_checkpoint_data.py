"""the "PNN1" checkpoint format and the IDX / CIFAR-10
loaders (semantics from the reference SPEC; the datasets themselves are not in
the container, so the tests write small files in the canonical formats)."""
import struct

import numpy as np
import pytest

from paper_2105_00053_b200 import checkpoint, data


def _recs(rng):
    out = []
    for i, (nb, es, shape) in enumerate([(8, 0, (4, 3)), (8, 2, (7,)), (12, 1, (2, 3, 4)),
                                         (16, 1, (5, 1, 3, 3)), (24, 2, (6,)), (16, 1, ())]):
        codes = rng.integers(0, 1 << nb, size=shape).astype(np.uint64)
        out.append((f"t{i}", (nb, es), codes))
    return out


def test_pnn1_round_trip_byte_identical():
    rng = np.random.default_rng(0)
    recs = _recs(rng)
    blob = checkpoint.dumps(recs)
    assert blob[:4] == b"PNN1"
    back = checkpoint.loads(blob)
    assert [(n, f, a.shape) for n, f, a in back] == [(n, f, np.asarray(a).shape) for n, f, a in recs]
    for (_, _, a), (_, _, b) in zip(recs, back):
        assert (np.asarray(a) == b).all()
    assert checkpoint.dumps(back) == blob  # load -> save is byte-identical
    # record layout: name length, name, nbits, es, rank, extents, little-endian codes
    n0 = struct.unpack("<I", blob[4:8])[0]
    assert blob[8:8 + n0] == b"t0" and blob[8 + n0:11 + n0] == bytes([8, 0, 2])


def test_pnn1_errors():
    rng = np.random.default_rng(1)
    blob = checkpoint.dumps(_recs(rng))
    with pytest.raises(ValueError):
        checkpoint.loads(b"PNN2" + blob[4:])
    with pytest.raises(ValueError):
        checkpoint.loads(blob[:-3])  # truncated codes
    with pytest.raises(ValueError):
        checkpoint.loads(blob[:9])  # truncated header


def _idx(tmp_path, n=5, magic_i=0x803, magic_l=0x801, nl=None, hw=(28, 28), cut=0):
    rng = np.random.default_rng(2)
    px = rng.integers(0, 256, size=(n, *hw)).astype(np.uint8)
    lab = rng.integers(0, 10, size=n).astype(np.uint8)
    ip, lp = tmp_path / "img.idx", tmp_path / "lab.idx"
    ib = struct.pack(">IIII", magic_i, n, *hw) + px.tobytes()
    ip.write_bytes(ib[:len(ib) - cut])
    lp.write_bytes(struct.pack(">II", magic_l, n if nl is None else nl) + lab.tobytes())
    return str(ip), str(lp), px, lab


def test_idx_loader(tmp_path):
    ip, lp, px, lab = _idx(tmp_path)
    ds = data.load_idx(ip, lp)
    assert ds.images.shape == (5, 1, 28, 28) and ds.images.dtype == np.float64
    assert (ds.images[:, 0] == px / 255.0).all() and (ds.labels == lab).all()
    assert (data.load_idx(ip, lp).images == ds.images).all()  # byte-exact re-read
    for kw in ({"magic_i": 0x804}, {"magic_l": 0x802}, {"nl": 4}, {"hw": (27, 28)}, {"cut": 10}):
        ip, lp, _, _ = _idx(tmp_path, **kw)
        with pytest.raises(ValueError):
            data.load_idx(ip, lp)


def test_cifar10_loader_and_normalisation(tmp_path):
    rng = np.random.default_rng(3)
    rec = np.zeros((4, data.CIFAR_RECORD), np.uint8)
    rec[:, 0] = [3, 0, 9, 1]
    rec[:, 1:] = rng.integers(0, 256, size=(4, 3072))
    p = tmp_path / "data_batch_1.bin"
    p.write_bytes(rec.tobytes())
    ds = data.load_cifar10([str(p)])
    assert ds.images.shape == (4, 3, 32, 32) and list(ds.labels) == [3, 0, 9, 1]
    assert (ds.images[1, 2].ravel() == rec[1, 1 + 2048:] / 255.0).all()  # B plane of record 1
    assert (data.normalize(ds, 0.0, 1.0).images == ds.images).all()
    m, s = data.channel_stats(ds)
    z = data.normalize(ds, m, s).images
    assert np.allclose(z.mean(axis=(0, 2, 3)), 0) and np.allclose(z.std(axis=(0, 2, 3)), 1)
    p.write_bytes(rec.tobytes()[:-1])
    with pytest.raises(ValueError):
        data.load_cifar10([str(p)])
    rec[0, 0] = 10
    p.write_bytes(rec.tobytes())
    with pytest.raises(ValueError):
        data.load_cifar10([str(p)])


def test_seeded_permutation():
    a, b = data.permutation(1000, 7), data.permutation(1000, 7)
    assert (a == b).all() and sorted(a) == list(range(1000))
    assert (a != data.permutation(1000, 8)).any()


@pytest.mark.gpu
def test_batches_quantise_like_from_float64(cuda, po, tmp_path):
    from paper_2105_00053_b200 import codec, ops

    rng = np.random.default_rng(4)
    ds = data.Dataset(rng.random((10, 1, 28, 28)), rng.integers(0, 10, 10).astype(np.int32))
    got = list(data.batches(ds, 4, seed=5, cfg=ops.P80))
    assert [x.shape[0] for x, _ in got] == [4, 4, 2]  # last partial batch
    order = data.permutation(10, 5)
    x0 = codec.to_host(got[0][0]).ravel()
    want = np.array([po.from_float64(8, 0, v) for v in ds.images[order[:4]].ravel()], np.uint64)
    assert (x0 == want).all()
    assert (got[0][1].cpu().numpy() == ds.labels[order[:4]]).all()


@pytest.mark.gpu
def test_model_checkpoint_round_trip(cuda, tmp_path):
    import torch

    from paper_2105_00053_b200 import codec, nn, ops

    st = nn.StagePrecisions(ops.P80, ops.P121, ops.P121, ops.P161, ops.P161)
    a = nn.lenet5(st, seed=1)
    path = str(tmp_path / "lenet.pnn1")
    checkpoint.save_model(a, path)
    b = nn.lenet5(st, seed=2)
    checkpoint.load_model(b, path)
    for p, q in zip(a.params(), b.params()):
        assert (codec.to_host(p.master) == codec.to_host(q.master)).all()
        for c in q.stage_formats():
            assert (codec.to_host(q.copies[c]) ==
                    codec.to_host(ops.convert_tensor(q.master, st.optimizer, c))).all()
    checkpoint.save_model(b, str(tmp_path / "again.pnn1"))
    assert open(path, "rb").read() == open(str(tmp_path / "again.pnn1"), "rb").read()
    with pytest.raises(ValueError):  # a different architecture / format is rejected
        checkpoint.load_model(nn.cifar_cnn(st, seed=0), path)
    with pytest.raises(ValueError):
        checkpoint.load_model(nn.lenet5(nn.StagePrecisions.uniform(ops.P121)), path)
    # same optimizer format and shapes, other stage precisions: the config record rejects it
    with pytest.raises(ValueError, match="stage precisions"):
        checkpoint.load_model(nn.lenet5(nn.StagePrecisions(ops.P81, ops.P121, ops.P121, ops.P161, ops.P161)),
                              path)
    del torch


@pytest.mark.gpu
def test_checkpoint_resumes_momentum_bit_exactly(cuda, tmp_path):
    """SGD with momentum: save after step 1 (weights + velocity), load into a
    fresh model and optimizer, run step 2 on both: identical weights, velocity
    and loss (bit-exact persistence)."""
    import torch

    from paper_2105_00053_b200 import codec, nn, ops

    st = nn.StagePrecisions(ops.P80, ops.P121, ops.P121, ops.P161, ops.P161)
    rng = np.random.default_rng(9)
    B = 16
    xs = [codec.from_float64_device(rng.random((B, 1, 32, 32)), st.forward) for _ in range(2)]
    ys = [torch.from_numpy(rng.integers(0, 10, B).astype(np.int32)).cuda() for _ in range(2)]
    a = nn.lenet5(st, seed=3)
    opt_a = nn.SGD(a.params(), 1.0 / 16, st, momentum=0.5)
    nn.train_step(a, nn.CrossEntropyLoss(st), opt_a, xs[0], ys[0], B)
    path = str(tmp_path / "mom.pnn1")
    checkpoint.save_model(a, path, opt_a)
    b = nn.lenet5(st, seed=4)
    opt_b = nn.SGD(b.params(), 1.0 / 16, st, momentum=0.5)
    with pytest.raises(ValueError, match="velocity"):
        checkpoint.load_model(b, _save_plain(a, tmp_path), opt_b)
    checkpoint.load_model(b, path, opt_b)
    la = nn.train_step(a, nn.CrossEntropyLoss(st), opt_a, xs[1], ys[1], B)
    lb = nn.train_step(b, nn.CrossEntropyLoss(st), opt_b, xs[1], ys[1], B)
    assert (codec.to_host(la) == codec.to_host(lb)).all()
    for p, q, u, v in zip(a.params(), b.params(), opt_a.velocity, opt_b.velocity):
        assert (codec.to_host(p.master) == codec.to_host(q.master)).all()
        assert (codec.to_host(u) == codec.to_host(v)).all()
    assert any(codec.to_host(v).any() for v in opt_b.velocity)


def _save_plain(model, tmp_path):
    path = str(tmp_path / "plain.pnn1")
    checkpoint.save_model(model, path)  # no optimizer: no velocity records
    return path
