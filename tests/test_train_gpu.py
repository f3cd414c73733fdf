"""Whole training steps on the GPU vs the CPU oracle step (oracle/step.py):
every activation, every gradient, the loss and the updated weights must be
bit-identical (BASELINE configs 0, 2 and the config-3 CNN at a small batch)."""
import numpy as np
import pytest
import torch

from oracle.step import blob_images, oracle_step
from paper_2105_00053_b200 import codec, nn, ops

pytestmark = pytest.mark.gpu

P80, P81, P121, P161 = ops.P80, ops.P81, ops.P121, ops.P161


def st_dict(st):
    return {k: (getattr(st, k).nbits, getattr(st, k).es)
            for k in ("forward", "backward", "gradient", "optimizer", "loss")}


def run_and_compare(po, model, st, x64, labels, lr, steps=1, grad_scale_log2=0):
    B = x64.shape[0]
    f = (st.forward.nbits, st.forward.es)
    xq = np.array([po.from_float64(*f, v) for v in x64.ravel()], np.uint64).reshape(x64.shape)
    xd = codec.from_float64_device(x64, st.forward)
    assert (codec.to_host(xd) == xq).all(), "device from_float64 ingestion differs"
    layers = nn.layer_description(model)
    params = [(codec.to_host(l.w.master), codec.to_host(l.b.master))
              for l in model.layers if isinstance(l, nn.Conv2d)]
    loss_fn = nn.CrossEntropyLoss(st, grad_scale_log2=grad_scale_log2)
    opt = nn.SGD(model.params(), lr, st, grad_scale_log2=grad_scale_log2)
    lab = torch.from_numpy(labels.astype(np.int32)).cuda()
    for step in range(steps):
        rec_gpu, rec_cpu = {}, {}
        loss = nn.train_step(model, loss_fn, opt, xd, lab, B, record=rec_gpu)
        torch.cuda.synchronize()
        lw, params, _ = oracle_step(po, layers, st_dict(st), params, xq, labels, lr, B, rec_cpu,
                                    grad_scale_log2=grad_scale_log2)
        for k, v in rec_cpu.items():
            if k == "loss_rows":
                continue
            assert k in rec_gpu, k
            got = codec.to_host(rec_gpu[k]).reshape(v.shape)
            bad = np.argwhere(got != v)
            assert bad.size == 0, (step, k, len(bad), bad[:3].tolist())
        assert int(codec.to_host(loss)[0]) == lw, (step, "loss")
        got_params = [(codec.to_host(l.w.master), codec.to_host(l.b.master))
                      for l in model.layers if isinstance(l, nn.Conv2d)]
        for i, ((gw, gb), (ww, wb)) in enumerate(zip(got_params, params)):
            assert (gw.reshape(ww.shape) == ww).all(), (step, "w", i)
            assert (gb == wb).all(), (step, "b", i)
        # stage copies equal convert(master) after the update
        for l in model.layers:
            if isinstance(l, nn.Conv2d):
                for c, t in l.w.copies.items():
                    want = po.convert_tensor(st.optimizer.nbits, st.optimizer.es, c.nbits, c.es,
                                             codec.to_host(l.w.master))
                    assert (codec.to_host(t) == want).all()
    return lw


def test_config0_lenet5_p161_b64(cuda, po):
    """BASELINE config 0: LeNet-5, one SGD step (lr 1/16), all stages posit(16,1), B=64."""
    st = nn.StagePrecisions.uniform(P161)
    rng = np.random.default_rng(2105)
    x = rng.random((64, 1, 32, 32))
    labels = rng.integers(0, 10, 64)
    model = nn.lenet5(st, seed=7)
    run_and_compare(po, model, st, x, labels, 1.0 / 16, steps=1)


def test_init_is_fp32_kaiming_rounded(cuda, po):
    st = nn.StagePrecisions.uniform(P161)
    model = nn.lenet5(st, seed=7)
    rng = np.random.default_rng(7)
    w = (rng.uniform(-1.0, 1.0, size=(6, 1, 5, 5)).astype(np.float32) * np.float32(np.sqrt(6.0 / 25)))
    want = np.array([po.from_float64(16, 1, float(v)) for v in w.astype(np.float64).ravel()], np.uint64)
    assert (codec.to_host(model.layers[0].w.master).ravel() == want).all()


def test_config2_lenet5_mixed_b256_steps(cuda, po):
    """BASELINE config 2 (3 of its 100 steps): forward (8,0); backward and
    gradient (12,1); loss and optimizer (16,1); batch 256; blob data."""
    st = nn.StagePrecisions(P80, P121, P121, P161, P161)
    x, labels = blob_images(seed=31, n=256)
    model = nn.lenet5(st, seed=11)
    run_and_compare(po, model, st, x, labels, 1.0 / 16, steps=3)


def test_config3_cifar_cnn_formats_small_batch(cuda, po):
    """The config-3 CNN and formats (forward (8,1), gradient (12,1), optimizer
    and loss (16,1)) at batch 4."""
    st = nn.StagePrecisions(P81, P121, P121, P161, P161)
    rng = np.random.default_rng(3)
    x = rng.uniform(-1.0, 1.0, (4, 3, 32, 32))
    labels = rng.integers(0, 10, 4)
    model = nn.cifar_cnn(st, seed=5)
    run_and_compare(po, model, st, x, labels, 1.0 / 16, steps=1)


@pytest.mark.parametrize("scale", [0, 6])
def test_posit82_star_lenet5_loss_scaled(cuda, po, scale):
    """The posit(8,2)* preset (O12L10: optimizer (12,2), loss (10,2), the rest
    (8,2)) with and without loss scaling by 2^6, two steps."""
    st = nn.StagePrecisions.posit82_star()
    x, labels = blob_images(seed=41, n=64)
    model = nn.lenet5(st, seed=13)
    run_and_compare(po, model, st, x, labels, 1.0 / 16, steps=2, grad_scale_log2=scale)


def test_loss_scaling_changes_small_gradients(cuda, po):
    """With posit(8,2) gradients, scaling by 2^6 changes the update (small
    gradients escape the low-precision tail) -- the point of the feature."""
    st = nn.StagePrecisions.posit82_star()
    x, labels = blob_images(seed=41, n=64)
    a, b = nn.lenet5(st, seed=13), nn.lenet5(st, seed=13)
    xd = codec.from_float64_device(x, st.forward)
    lab = torch.from_numpy(labels.astype(np.int32)).cuda()
    for m, s in ((a, 0), (b, 6)):
        nn.train_step(m, nn.CrossEntropyLoss(st, s), nn.SGD(m.params(), 1 / 16, st, s), xd, lab, 64)
    diff = sum(int((codec.to_host(p.master) != codec.to_host(q.master)).sum())
               for p, q in zip(a.params(), b.params()))
    assert diff > 0
