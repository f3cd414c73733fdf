"""SURVEY.md §8f item 2, the rest of the SPEC layer set: sqrt, tanh / sigmoid
layers with their backward, dropout, MSE, batch normalisation, SGD with
momentum.  CPU: the oracle (oracle/layers_oracle.c) pinned to the compiled
reference where the reference has the function (sqrt_posit) and to the SPEC's
examples elsewhere; GPU: every device kernel and two whole training steps
against the oracle, bit for bit."""
import numpy as np
import pytest
import torch

from conftest import rand_codes

FORMATS = [(8, 0), (8, 1), (8, 2), (12, 1), (16, 1)]


# ---------------------------------------------------------------- oracle (CPU)

@pytest.mark.parametrize("cfg", FORMATS + [(10, 2), (12, 2)])
def test_oracle_sqrt_vs_reference(po, ref, cfg):
    n, es = cfg
    step = 1 if n <= 12 else 3
    for c in range(0, 1 << n, step):
        assert po.sqrt(n, es, c) == ref.sqrt(n, es, c), c


def test_kat_sqrt(po):
    # test_posit.cpp:321-324: sqrt(-4) is NaR, sqrt(4) == 2
    for n, es in FORMATS:
        assert po.sqrt(n, es, po.from_float64(n, es, -4.0)) == 1 << (n - 1)
        assert po.to_float64(n, es, po.sqrt(n, es, po.from_float64(n, es, 4.0))) == 2.0
        assert po.sqrt(n, es, 0) == 0


def test_kat_spec_layer_examples(po):
    f = (16, 1)
    half = po.from_float64(*f, 0.5)
    # sigmoid_f(0) = 0.5
    assert int(po.act_fwd(2, *f, np.zeros(1, np.uint64))[0]) == half
    # identical prediction and target -> loss 0, gradient 0
    rng = np.random.default_rng(0)
    y = rand_codes(rng, 16, (4, 10))
    loss, g = po.mse(*f, y, y, 40)
    assert loss == 0 and (g == 0).all()
    # gradient 2(y - t)/N on exactly representable values
    t = np.zeros((1, 4), np.uint64)
    yv = np.array([[po.from_float64(*f, v) for v in (1.0, -0.5, 0.25, 2.0)]], np.uint64)
    loss, g = po.mse(*f, yv, t, 4)
    assert [po.to_float64(*f, int(c)) for c in g.ravel()] == [0.5, -0.25, 0.125, 1.0]
    assert po.to_float64(*f, loss) == (1 + 0.25 + 0.0625 + 4) / 4
    # batchnorm on a constant channel -> xhat == 0
    x = np.full((4, 2, 3, 3), po.from_float64(*f, 0.75), np.uint64)
    one = po.from_float64(*f, 1.0)
    y, xh, inv, rm, rv = po.batchnorm_fwd(f, x, [one, one], [0, 0], po.from_float64(*f, 1e-5), 1, f,
                                          [0, 0], [one, one], po.from_float64(*f, 0.1))
    assert (xh == 0).all() and (y == 0).all()
    assert po.to_float64(*f, int(rm[0])) == pytest.approx(0.075, rel=1e-3)
    # dropout p = 0 is the identity; rate ~ p otherwise
    x = rand_codes(rng, 16, (20000,))
    one = po.from_float64(*f, 1.0)
    assert (po.dropout(*f, x, 5, 0, one) == x).all()
    kept = np.count_nonzero(po.dropout(*f, np.full(20000, one, np.uint64), 5, int(0.3 * 2**32),
                                       po.from_float64(*f, 1 / 0.7)))
    assert abs(kept / 20000 - 0.7) < 0.02


def test_oracle_momentum_zero_grad_keeps_weights(po):
    f = (16, 1)
    rng = np.random.default_rng(1)
    w = rand_codes(rng, 16, (100,))
    v = np.zeros(100, np.uint64)
    lr, mu = po.from_float64(*f, 0.1), po.from_float64(*f, 0.9)
    w2, v2 = po.sgd_momentum(f, w, v, f, np.zeros(100, np.uint64), lr, mu)
    assert (w2 == w).all() and (v2 == 0).all()
    # with mu = 0 it is plain SGD
    g = rand_codes(rng, 16, (100,))
    w3, _ = po.sgd_momentum(f, w, v, f, g, lr, 0)
    assert (w3 == po.sgd(*f, w, *f, g, lr)).all()


# ---------------------------------------------------------------- device (GPU)

def _dev(cfg, a):
    from paper_2105_00053_b200 import ops

    return torch.from_numpy(np.ascontiguousarray(a).astype(ops._cfg(cfg).np_code_dtype)).cuda()


def _host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.int64).astype(np.uint64)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", FORMATS + [(10, 2), (12, 2)])
def test_gpu_sqrt_all_codes(cuda, po, cfg):
    from paper_2105_00053_b200 import ops

    n, es = cfg
    codes = np.arange(1 << n, dtype=np.int64)
    got = _host(ops.scalar_eval(cfg, 12, torch.from_numpy(codes).cuda())) & np.uint64((1 << n) - 1)
    want = np.array([po.sqrt(n, es, int(c)) for c in codes], np.uint64)
    assert (got == want).all()


@pytest.mark.gpu
@pytest.mark.parametrize("fmts", [((8, 0), (8, 0)), ((8, 1), (12, 1)), ((16, 1), (16, 1)), ((8, 2), (12, 2))])
@pytest.mark.parametrize("kind", [1, 2])
def test_gpu_act_fwd_bwd(cuda, po, fmts, kind):
    from paper_2105_00053_b200 import ops

    f, b = fmts
    rng = np.random.default_rng(kind * 10 + f[0])
    x = rand_codes(rng, f[0], (3, 5, 7, 11), nar_ok=True)
    dy = rand_codes(rng, b[0], x.shape, nar_ok=True)
    y = ops.act_fwd(kind, f, _dev(f, x))
    want_y = po.act_fwd(kind, *f, x)
    assert (_host(y) == want_y).all()
    dx = ops.act_bwd(kind, f, y, b, _dev(b, dy))
    assert (_host(dx) == po.act_bwd(kind, f, want_y, b, dy)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(8, 1), (16, 1), (12, 2)])
def test_gpu_dropout(cuda, po, cfg):
    from paper_2105_00053_b200 import ops

    n, es = cfg
    rng = np.random.default_rng(n)
    x = rand_codes(rng, n, (70001,))
    p = 0.4
    th = ops.dropout_threshold(p)
    sc = po.from_float64(n, es, 1 / (1 - p))
    off = torch.tensor([7], dtype=torch.int64, device="cuda")
    got = _host(ops.dropout(cfg, _dev(cfg, x), 123, th, sc, seed_offset=off))
    assert (got == po.dropout(n, es, x, 130, th, sc)).all()
    got0 = _host(ops.dropout(cfg, _dev(cfg, x), 130, th, sc))
    assert (got0 == got).all()
    assert po.dropout_bits(130, 5) == po.dropout_bits(123 + 7, 5)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(8, 0), (8, 2), (12, 1), (16, 1)])
@pytest.mark.parametrize("scale", [0, 4])
def test_gpu_mse(cuda, po, cfg, scale):
    from paper_2105_00053_b200 import ops

    n, es = cfg
    rng = np.random.default_rng(n + scale)
    y = rand_codes(rng, n, (64, 10))
    t = rand_codes(rng, n, (64, 10))
    loss, g = ops.mse(cfg, _dev(cfg, y), _dev(cfg, t), 640 * 2, scale)
    lw, gw = po.mse(n, es, y, t, 1280, scale)
    assert (_host(g) == gw).all() and int(_host(loss)[0]) == lw


@pytest.mark.gpu
def test_gpu_mse_rejects_wide_quire(cuda):
    from paper_2105_00053_b200 import ops

    z = torch.zeros((4, 10), dtype=torch.uint16, device="cuda")
    with pytest.raises(Exception, match="not supported"):
        ops.mse((10, 2), z, z, 40)


BN_CASES = [
    ((4, 3, 5, 7), (16, 1), (16, 1), (16, 1), (16, 1)),
    ((64, 32, 8, 8), (8, 1), (12, 1), (12, 1), (16, 1)),     # M = 4096: split over blocks
    ((256, 16, 16, 16), (8, 0), (8, 0), (8, 0), (12, 1)),    # M = 65536: 37 splits, (8,0) quire wraps
    ((16, 64), (8, 2), (8, 2), (8, 2), (12, 2)),              # BatchNorm1d, posit(8,2)* formats
]


@pytest.mark.gpu
@pytest.mark.parametrize("case", BN_CASES)
def test_gpu_batchnorm_fwd_bwd(cuda, po, case):
    from paper_2105_00053_b200 import ops

    shape, f, b, g, o = case
    rng = np.random.default_rng(shape[0] + shape[1])
    Cc = shape[1]
    # inputs of a moderate range (random codes span maxpos; both are exact either way)
    x = np.array([po.from_float64(*f, v) for v in rng.normal(0.5, 2.0, int(np.prod(shape)))],
                 np.uint64).reshape(shape)
    gamma = np.array([po.from_float64(*f, v) for v in rng.uniform(0.5, 1.5, Cc)], np.uint64)
    beta = np.array([po.from_float64(*f, v) for v in rng.uniform(-0.5, 0.5, Cc)], np.uint64)
    rm = np.array([po.from_float64(*o, v) for v in rng.uniform(-0.1, 0.1, Cc)], np.uint64)
    rv = np.array([po.from_float64(*o, v) for v in rng.uniform(0.9, 1.1, Cc)], np.uint64)
    eps, mom = po.from_float64(*f, 1e-5), po.from_float64(*o, 0.1)
    for training in (1, 0):
        rm_d, rv_d = _dev(o, rm), _dev(o, rv)
        y, xh, inv = ops.batchnorm_fwd(f, _dev(f, x), _dev(f, gamma), _dev(f, beta), eps, training, o,
                                       rm_d, rv_d, mom)
        wy, wxh, winv, wrm, wrv = po.batchnorm_fwd(f, x, gamma, beta, eps, training, o, rm, rv, mom)
        assert (_host(y) == wy).all() and (_host(xh) == wxh).all() and (_host(inv) == winv).all()
        assert (_host(rm_d) == wrm).all() and (_host(rv_d) == wrv).all()
    dy = np.array([po.from_float64(*b, v) for v in rng.normal(0, 0.1, int(np.prod(shape)))],
                  np.uint64).reshape(shape)
    gb = np.array([po.convert(*f, *b, int(c)) for c in gamma], np.uint64)
    dx, dgm, dbt = ops.batchnorm_bwd(f, _dev(f, wxh), _dev(f, winv), b, _dev(b, dy), _dev(b, gb), g)
    wdx, wdg, wdb = po.batchnorm_bwd(f, wxh, winv, b, dy, gb, g)
    assert (_host(dx) == wdx).all()
    assert (_host(dgm) == wdg).all() and (_host(dbt) == wdb).all()
    # raw quire words round to the same codes
    _, (gw, gn), (bw, bn_) = ops.batchnorm_bwd(f, _dev(f, wxh), _dev(f, winv), b, _dev(b, dy), _dev(b, gb), g,
                                               raw=True)
    assert (_host(ops.lanes_to_posit(g, ops.quire_to_lanes(g, gw, gn))) == wdg).all()
    assert (_host(ops.lanes_to_posit(g, ops.quire_to_lanes(g, bw, bn_))) == wdb).all()


@pytest.mark.gpu
@pytest.mark.parametrize("fmts", [((16, 1), (12, 1)), ((12, 2), (8, 2))])
def test_gpu_sgd_momentum(cuda, po, fmts):
    from paper_2105_00053_b200 import ops

    o, g = fmts
    rng = np.random.default_rng(o[0])
    w = rand_codes(rng, o[0], (4099,))
    v = rand_codes(rng, o[0], (4099,))
    gr = rand_codes(rng, g[0], (4099,))
    lr, mu = po.from_float64(*o, 1 / 16), po.from_float64(*o, 0.9)
    wd, vd = _dev(o, w), _dev(o, v)
    c1 = torch.empty(4099, dtype=torch.uint8, device="cuda")
    ops.sgd_step_momentum(o, wd, vd, g, _dev(g, gr), lr, mu, copies=[((8, 2), c1)], grad_scale_log2=3)
    ww, wv = po.sgd_momentum(o, w, v, g, gr, lr, mu, 3)
    assert (_host(wd) == ww).all() and (_host(vd) == wv).all()
    assert (_host(c1) == po.convert_tensor(*o, 8, 2, ww)).all()


def _st_dict(st):
    return {k: (getattr(st, k).nbits, getattr(st, k).es)
            for k in ("forward", "backward", "gradient", "optimizer", "loss")}


def _compare_steps(po, model, st, x64, labels, lr, steps, loss_kind="xent", momentum=0.0):
    from oracle.step import oracle_step
    from paper_2105_00053_b200 import codec, nn

    B = x64.shape[0]
    f = (st.forward.nbits, st.forward.es)
    xq = np.array([po.from_float64(*f, v) for v in x64.ravel()], np.uint64).reshape(x64.shape)
    xd = codec.from_float64_device(x64, st.forward)
    pairs = [l for l in model.layers if isinstance(l, (nn.Conv2d, nn.BatchNorm2d))]

    def host_params():
        return [(codec.to_host(l.w.master), codec.to_host(l.b.master)) if isinstance(l, nn.Conv2d)
                else (codec.to_host(l.gamma.master), codec.to_host(l.beta.master)) for l in pairs]

    params = host_params()
    state = {i: [codec.to_host(l.running_mean), codec.to_host(l.running_var)]
             for i, l in enumerate(model.layers) if isinstance(l, nn.BatchNorm2d)}
    velocity = [[np.zeros(p.shape, np.uint64) for p in pr] for pr in params] if momentum else None
    loss_fn = nn.MSELoss(st) if loss_kind == "mse" else nn.CrossEntropyLoss(st)
    opt = nn.SGD(model.params(), lr, st, momentum=momentum)
    lab = torch.from_numpy(labels.astype(np.int32)).cuda()
    for step in range(steps):
        layers = nn.layer_description(model)
        rec_gpu, rec_cpu = {}, {}
        loss = nn.train_step(model, loss_fn, opt, xd, lab, B, record=rec_gpu)
        torch.cuda.synchronize()
        lw, params, _ = oracle_step(po, layers, _st_dict(st), params, xq, labels, lr, B, rec_cpu,
                                    state=state, loss=loss_kind, momentum=momentum, velocity=velocity)
        for k, v in rec_cpu.items():
            if k == "loss_rows":
                continue
            got = codec.to_host(rec_gpu[k]).reshape(v.shape)
            bad = np.argwhere(got != v)
            assert bad.size == 0, (step, k, len(bad), bad[:3].tolist())
        assert int(codec.to_host(loss)[0]) == lw, (step, "loss")
        for i, ((gw, gb), (ww, wb)) in enumerate(zip(host_params(), params)):
            assert (gw.reshape(ww.shape) == ww).all() and (gb == wb).all(), (step, i)
        for i, l in enumerate(model.layers):
            if isinstance(l, nn.BatchNorm2d):
                assert (codec.to_host(l.running_mean) == state[i][0]).all(), (step, "rm", i)
                assert (codec.to_host(l.running_var) == state[i][1]).all(), (step, "rv", i)


@pytest.mark.gpu
def test_gpu_lenet5_classic_mse_momentum_steps(cuda, po):
    """tanh / avg-pool / sigmoid LeNet-5, MSE loss, SGD momentum 0.9, config-2
    formats, 2 steps: every activation, gradient, loss and weight."""
    from oracle.step import blob_images
    from paper_2105_00053_b200 import nn, ops

    st = nn.StagePrecisions(ops.P80, ops.P121, ops.P121, ops.P161, ops.P161)
    x, labels = blob_images(seed=5, n=32)
    _compare_steps(po, nn.lenet5_classic(st, seed=3), st, x, labels, 1 / 16, 2, loss_kind="mse",
                   momentum=0.9)


@pytest.mark.gpu
@pytest.mark.parametrize("preset", ["config3", "posit82_star"])
def test_gpu_cnn_bn_dropout_steps(cuda, po, preset):
    """BatchNorm (2-D and 1-D) + dropout CNN, cross-entropy, 2 steps (fresh
    dropout mask per step), then one eval-mode forward (running stats)."""
    from paper_2105_00053_b200 import codec, nn, ops

    st = (nn.StagePrecisions(ops.P81, ops.P121, ops.P121, ops.P161, ops.P161) if preset == "config3"
          else nn.StagePrecisions.posit82_star())
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, (8, 3, 16, 16))
    labels = rng.integers(0, 10, 8)
    model = nn.cnn_bn_dropout(st, seed=2, hw=16)
    _compare_steps(po, model, st, x, labels, 1 / 16, 2)
    # eval mode: running statistics, dropout off
    from oracle.step import oracle_step  # noqa: F401  (forward-only check below)
    model.eval()
    out = model.forward(codec.from_float64_device(x, st.forward))
    model.train()
    assert out.shape == (8, 10)


@pytest.mark.gpu
def test_gpu_graphed_dropout_draws_fresh_masks(cuda, po):
    """A captured CUDA graph replays the dropout counter increment: graph
    replays equal the eager steps bit for bit."""
    from paper_2105_00053_b200 import codec, nn, ops

    st = nn.StagePrecisions(ops.P81, ops.P121, ops.P121, ops.P161, ops.P161)
    rng = np.random.default_rng(4)
    x = codec.from_float64_device(rng.uniform(-1, 1, (8, 3, 16, 16)), st.forward)
    lab = torch.from_numpy(rng.integers(0, 10, 8).astype(np.int32)).cuda()
    a, b = nn.cnn_bn_dropout(st, seed=2, hw=16), nn.cnn_bn_dropout(st, seed=2, hw=16)
    la = [nn.train_step(a, nn.CrossEntropyLoss(st), opt_a, x, lab, 8)
          for opt_a in [nn.SGD(a.params(), 1 / 16, st)] * 4]
    g = nn.GraphedTrainStep(b, nn.CrossEntropyLoss(st), nn.SGD(b.params(), 1 / 16, st), x.clone(), lab.clone(), 8)
    lb = [g.step().clone() for _ in range(4)]
    for u, v in zip(la, lb):
        assert int(codec.to_host(u)[0]) == int(codec.to_host(v)[0])
    for p, q in zip(a.params(), b.params()):
        assert (codec.to_host(p.master) == codec.to_host(q.master)).all()
    assert int(b.layers[12].counter.item()) == 4
