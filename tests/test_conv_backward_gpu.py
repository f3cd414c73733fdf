"""Layer-level Conv2d pair (pnn_conv2d_fwd_save / pnn_conv2d_backward): the
forward keeps x's digit planes, the fused backward reads them for the weight
gradient (same format, or an exact widening by whole digits: posit(8,1)
forward digits under a posit(12,1) gradient, BASELINE config 3), folds the
stage conversions into its digitisers and digitises dy once for both passes.
Every output must equal the per-pass calls of the same step -- the weight
gradient of the converted operands (conv2d_weight_grad(p_g, convert(dy),
convert(x))) and the input gradient (conv2d_input_grad(p_b, dy, w)) --, which
the implicit-conv tests pin to the oracle; one case is checked against the
oracle directly."""
import numpy as np
import pytest
import torch

from conftest import rand_codes
from paper_2105_00053_b200 import ops

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def all_variants():
    """Launch the reduced-digit variants even for these small test problems."""
    from paper_2105_00053_b200 import _native
    prev = _native.lib().pnn_variant_min_work(0)
    yield
    _native.lib().pnn_variant_min_work(prev)

P80, P81, P121, P161 = (8, 0), (8, 1), (12, 1), (16, 1)

# (forward, backward, gradient) stage formats
STAGES = [
    (P81, P121, P121),  # config 3: saved (8,1) digits one digit up, dy shared
    (P80, P80, P80),    # uniform (config 4)
    (P81, P81, P81),
    (P121, P121, P121),
    (P161, P161, P161),
    (P80, P121, P121),  # es differs: x digitised through the conversion LUT
    (P121, P161, P161),  # widening without a kernel variant: LUT path
    (P121, P81, P121),  # p_b != p_g: dy converted in the weight-gradient digitiser
]

# (N, C, H, W, F, K, pad)
SHAPES = [
    (2, 32, 8, 8, 32, 3, 1),
    (3, 32, 16, 16, 64, 3, 1),
    (2, 64, 16, 16, 64, 3, 1),
    (2, 3, 32, 32, 32, 3, 1),    # folded first layer
    (2, 32, 10, 10, 32, 3, 0),   # valid conv (fwd box inside the image; no implicit dgrad)
    (2, 32, 8, 8, 40, 3, 1),     # F not a multiple of the N tile: dy digits not shared
]


def dev(cfg, a):
    return torch.from_numpy(np.ascontiguousarray(a).astype(ops._cfg(cfg).np_code_dtype)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.int64).astype(np.uint64)


def run_pair(ff, fb, fg, x, w, b, dy, wb, K, pad, need_dx, raw):
    n = ops.conv2d_saved_bytes(ff, x.shape, w.shape, 1, pad)
    saved = torch.empty(n, dtype=torch.uint8, device="cuda") if n else None
    y = (ops.conv2d_fwd_save(ff, x, w, b, 1, pad, saved) if saved is not None
         else ops.conv2d(ff, x, w, b, 1, pad))
    res = ops.conv2d_backward(ff, fb, fg, dy, x, saved, wb, x.shape, w.shape, 1, pad, need_dx, raw=raw)
    return y, res


@pytest.mark.parametrize("stages", STAGES)
@pytest.mark.parametrize("shape", SHAPES)
def test_fused_backward_equals_per_pass(cuda, stages, shape):
    ff, fb, fg = stages
    N, C, H, W, F, K, pad = shape
    rng = np.random.default_rng(hash((stages, shape)) & 0xFFFF)
    x = dev(ff, rand_codes(rng, ff[0], (N, C, H, W)))
    w = dev(ff, rand_codes(rng, ff[0], (F, C, K, K)))
    b = dev(ff, rand_codes(rng, ff[0], (F,)))
    OH, OW = H + 2 * pad - K + 1, W + 2 * pad - K + 1
    dy = dev(fb, rand_codes(rng, fb[0], (N, F, OH, OW)))
    wb = dev(fb, rand_codes(rng, fb[0], (F, C, K, K)))
    need_dx = C % 32 == 0 and F % 32 == 0 and pad > 0  # implicit input grad: C, F % 32, pad = K // 2
    y, res = run_pair(ff, fb, fg, x, w, b, dy, wb, K, pad, need_dx, raw=False)
    assert res is not None, "fused backward should be eligible for this shape"
    dx, dw = res
    assert (host(y) == host(ops.conv2d(ff, x, w, b, 1, pad))).all()
    dyg = ops.convert_tensor(dy, fb, fg)
    xg = ops.convert_tensor(x, ff, fg)
    want_dw = host(ops.conv2d_weight_grad(fg, dyg, xg, w.shape, 1, pad))
    assert (host(dw) == want_dw).all(), int((host(dw) != want_dw).sum())
    if need_dx:
        want_dx = host(ops.conv2d_input_grad(fb, dy, wb, x.shape, 1, pad))
        assert (host(dx) == want_dx).all(), int((host(dx) != want_dx).sum())
    else:
        assert dx is None
    # raw quire words (data-parallel input) equal the per-pass raw words
    _, res = run_pair(ff, fb, fg, x, w, b, dy, wb, K, pad, False, raw=True)
    _, words, nar = res[1]
    _, ww, wn = ops.conv2d_weight_grad(fg, dyg, xg, w.shape, 1, pad, raw=True)
    assert (host(words) == host(ww)).all() and (host(nar) == host(wn)).all()


@pytest.mark.parametrize("stages", [(P81, P121, P121), (P80, P80, P80), (P161, P161, P161)])
def test_fused_backward_nar(cuda, stages):
    """NaR in x (saved NaR map), in dy (shared pixel map / channel map), in w."""
    ff, fb, fg = stages
    N, C, H, W, F, K, pad = 2, 32, 8, 8, 32, 3, 1
    rng = np.random.default_rng(7)
    xa = rand_codes(rng, ff[0], (N, C, H, W))
    xa[1, 5, 0, 7] = 1 << (ff[0] - 1)
    dya = rand_codes(rng, fb[0], (N, F, H, W))
    dya[0, 9, 3, 3] = 1 << (fb[0] - 1)
    wba = rand_codes(rng, fb[0], (F, C, K, K))
    wba[4, 2, 1, 1] = 1 << (fb[0] - 1)
    x, dy, wb = dev(ff, xa), dev(fb, dya), dev(fb, wba)
    w = dev(ff, rand_codes(rng, ff[0], (F, C, K, K)))
    y, (dx, dw) = run_pair(ff, fb, fg, x, w, None, dy, wb, K, pad, True, raw=False)
    dyg, xg = ops.convert_tensor(dy, fb, fg), ops.convert_tensor(x, ff, fg)
    assert (host(dw) == host(ops.conv2d_weight_grad(fg, dyg, xg, w.shape, 1, pad))).all()
    assert (host(dx) == host(ops.conv2d_input_grad(fb, dy, wb, x.shape, 1, pad))).all()
    assert (host(y) == host(ops.conv2d(ff, x, w, None, 1, pad))).all()


def test_fused_backward_vs_oracle(cuda, po):
    """Config-3 stage formats against the oracle restatement directly."""
    ff, fb, fg = P81, P121, P121
    N, C, H, W, F, K, pad = 2, 32, 8, 8, 32, 3, 1
    rng = np.random.default_rng(11)
    xa = rand_codes(rng, 8, (N, C, H, W))
    dya = rand_codes(rng, 12, (N, F, H, W))
    wba = rand_codes(rng, 12, (F, C, K, K))
    x, dy, wb = dev(ff, xa), dev(fb, dya), dev(fb, wba)
    w = dev(ff, rand_codes(rng, 8, (F, C, K, K)))
    _, (dx, dw) = run_pair(ff, fb, fg, x, w, None, dy, wb, K, pad, True, raw=False)
    xg = po.convert_tensor(8, 1, 12, 1, xa.astype(np.uint64))
    want_dw = po.conv2d_weight_grad(12, 1, dya.astype(np.uint64), xg, (F, C, K, K), 1, pad)
    want_dx = po.conv2d_input_grad(12, 1, dya.astype(np.uint64), wba.astype(np.uint64), (N, C, H, W), 1, pad)
    assert (host(dw).reshape(want_dw.shape) == want_dw).all()
    assert (host(dx).reshape(want_dx.shape) == want_dx).all()


def test_saved_bytes_zero_when_ineligible(cuda):
    # LeNet conv2 (6 -> 16 channels): no implicit pair, the layer uses the per-pass path
    assert ops.conv2d_saved_bytes(P161, (4, 6, 14, 14), (16, 6, 5, 5), 1, 0) == 0
    assert ops.conv2d_backward(P161, P161, P161, torch.zeros((4, 16, 10, 10), dtype=torch.int16).cuda(),
                               None, None, None, (4, 6, 14, 14), (16, 6, 5, 5), 1, 0, False) is None


@pytest.mark.parametrize("cfg", [P80, P81, P121, P161])
@pytest.mark.parametrize("shape", [(2, 32, 8, 8, 32, 3, 1), (2, 3, 32, 32, 32, 3, 1), (1, 256, 4, 4, 32, 3, 1),
                                   (3, 64, 16, 16, 64, 3, 1)])
def test_fused_relu_forward(cuda, cfg, shape):
    """Conv2d + ReLU in one epilogue (pnn_conv2d_fwd_layer) == conv2d then relu_fwd,
    pre-activation output included; NaR rows (relu(NaR) = 0); the small-image /
    deep-K shape runs split-K (finalize + relu pass)."""
    N, C, H, W, F, K, pad = shape
    rng = np.random.default_rng(hash((cfg, shape)) & 0xFFFF)
    xa = rand_codes(rng, cfg[0], (N, C, H, W))
    xa[0, 1, 2, 3] = 1 << (cfg[0] - 1)
    x = dev(cfg, xa)
    w = dev(cfg, rand_codes(rng, cfg[0], (F, C, K, K)))
    b = dev(cfg, rand_codes(rng, cfg[0], (F,)))
    ref = ops.conv2d(cfg, x, w, b, 1, pad)
    n = ops.conv2d_saved_bytes(cfg, x.shape, w.shape, 1, pad)
    saved = torch.empty(n, dtype=torch.uint8, device="cuda") if n else None
    y, pre = ops.conv2d_fwd_layer(cfg, x, w, b, 1, pad, saved, relu=True, want_pre=True)
    assert torch.equal(pre, ref)
    assert torch.equal(y, ops.relu_fwd(cfg, ref))
    y2, none = ops.conv2d_fwd_layer(cfg, x, w, b, 1, pad, None, relu=True, want_pre=False)
    assert none is None and torch.equal(y2, y)


@pytest.mark.parametrize("stages", [(P81, P121, P121), (P80, P80, P80), (P121, P81, P121), (P161, P161, P161)])
@pytest.mark.parametrize("shape", [(2, 32, 8, 8, 32, 3, 1), (2, 3, 32, 32, 32, 3, 1), (3, 64, 16, 16, 64, 3, 1),
                                   (2, 32, 8, 8, 40, 3, 1)])
def test_gated_backward_equals_relu_then_conv(cuda, stages, shape):
    """Conv2d + ReLU backward in one call (gate applied in the digitisers) ==
    relu_bwd followed by the fused conv backward; NaR and zero gates included."""
    ff, fb, fg = stages
    N, C, H, W, F, K, pad = shape
    rng = np.random.default_rng(hash((stages, shape, 1)) & 0xFFFF)
    x = dev(ff, rand_codes(rng, ff[0], (N, C, H, W)))
    w = dev(ff, rand_codes(rng, ff[0], (F, C, K, K)))
    OH, OW = H + 2 * pad - K + 1, W + 2 * pad - K + 1
    gate_a = rand_codes(rng, ff[0], (N, F, OH, OW), nar_ok=True)
    gate_a[0, 0] = 0
    gate = dev(ff, gate_a)
    dy = dev(fb, rand_codes(rng, fb[0], (N, F, OH, OW), nar_ok=True))
    wb = dev(fb, rand_codes(rng, fb[0], (F, C, K, K)))
    need_dx = C % 32 == 0 and F % 32 == 0
    n = ops.conv2d_saved_bytes(ff, x.shape, w.shape, 1, pad)
    saved = torch.empty(n, dtype=torch.uint8, device="cuda") if n else None
    ops.conv2d_fwd_save(ff, x, w, None, 1, pad, saved) if saved is not None else None
    res = ops.conv2d_backward_gated(ff, fb, fg, dy, gate, x, saved, wb, x.shape, w.shape, 1, pad, need_dx)
    assert res is not None
    dx, dw, dyg = res
    want_dyg = ops.relu_bwd(ff, gate, fb, dy)
    assert torch.equal(dyg, want_dyg)
    ref = ops.conv2d_backward(ff, fb, fg, want_dyg, x, saved, wb, x.shape, w.shape, 1, pad, need_dx)
    assert torch.equal(dw, ref[1])
    if need_dx:
        assert torch.equal(dx, ref[0])


def test_fused_relu_backward_step_matches(cuda, po):
    """Sequential with fuse_relu_backward on: a config-3-format CIFAR-CNN step at a
    small batch is bit-identical to the default (two-kernel) backward."""
    from paper_2105_00053_b200 import codec, nn
    st = nn.StagePrecisions(ops.P81, ops.P121, ops.P121, ops.P161, ops.P161)
    rng = np.random.default_rng(4)
    x = codec.from_float64_device(rng.uniform(-1, 1, (8, 3, 32, 32)), st.forward)
    lab = torch.from_numpy(rng.integers(0, 10, 8).astype(np.int32)).cuda()
    outs = []
    for fuse in (False, True):
        model = nn.cifar_cnn(st, seed=3)
        model.fuse_relu_backward = fuse
        loss = nn.train_step(model, nn.CrossEntropyLoss(st), nn.SGD(model.params(), 1 / 16, st), x, lab, 8)
        outs.append([loss] + [p.master for p in model.params()])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("st_fmt", ["config3", "uniform80"])
def test_unrecorded_step_equals_recorded_step(cuda, st_fmt):
    """The fusions the layer path takes only when it does not record (ReLU ->
    MaxPool backward in one pass) leave every parameter bit-identical to the
    recorded (per-layer, oracle-checked) step."""
    from paper_2105_00053_b200 import codec, nn
    st = (nn.StagePrecisions(ops.P81, ops.P121, ops.P121, ops.P161, ops.P161) if st_fmt == "config3"
          else nn.StagePrecisions.uniform(ops.P80))
    rng = np.random.default_rng(9)
    x = codec.from_float64_device(rng.uniform(-1, 1, (8, 3, 32, 32)), st.forward)
    lab = torch.from_numpy(rng.integers(0, 10, 8).astype(np.int32)).cuda()
    outs = []
    for record in ({}, None):
        model = nn.cifar_cnn(st, seed=5)
        loss = nn.train_step(model, nn.CrossEntropyLoss(st), nn.SGD(model.params(), 1 / 16, st), x, lab, 8,
                             record=record)
        outs.append([loss] + [p.master for p in model.params()])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("dy_small", [False, True])
@pytest.mark.parametrize("big", [False, True])
@pytest.mark.parametrize("shape", [(2, 32, 8, 8, 32, 3, 1), (3, 64, 16, 16, 64, 3, 1)])
def test_dgrad_reduced_weight_digits(cuda, po, big, shape, dy_small):
    """posit(12,1) input gradient: weights within 3 digits (|w| < 8) take the
    device-selected reduced-digit kernel (DB = 3); one large weight switches to
    the full kernel.  Both against the oracle."""
    N, C, H, W, F, K, pad = shape
    cfg = P121
    rng = np.random.default_rng(17 + big)
    small = np.array([po.from_float64(12, 1, float(v)) for v in rng.normal(0, 0.3, F * C * K * K)],
                     np.uint64).reshape(F, C, K, K)
    if big:
        small[1, 2, 0, 0] = po.from_float64(12, 1, 100.0)
    dya = rand_codes(rng, 12, (N, F, H, W))
    if dy_small:  # gradient-like values: within 3 digits -> the 3 x 3 digit kernel
        dya = np.array([po.from_float64(12, 1, float(v)) for v in rng.normal(0, 0.01, dya.size)],
                       np.uint64).reshape(dya.shape)
        dya[0, 0, 0, :3] = [0, 1, (1 << 12) - 1]  # zero, minpos, -minpos
    dx = ops.conv2d_input_grad(cfg, dev(cfg, dya), dev(cfg, small), (N, C, H, W), 1, pad)
    want = po.conv2d_input_grad(12, 1, dya, small, (N, C, H, W), 1, pad)
    assert (host(dx).reshape(want.shape) == want).all()


@pytest.mark.parametrize("wide", ["none", "x", "dy"])
@pytest.mark.parametrize("shape", [(2, 32, 8, 8, 32, 3, 1), (3, 64, 16, 16, 64, 3, 1), (2, 3, 32, 32, 32, 3, 1),
                                   # 128 output channels: two 64-column tiles; 96: not a multiple of 64,
                                   # the 32-column kernel
                                   (2, 32, 8, 8, 128, 3, 1), (2, 32, 8, 8, 96, 3, 1)])
def test_wgrad_reduced_digits(cuda, po, wide, shape):
    """Config-3 stages with activation / gradient values within 3 digits: the
    weight gradient takes the device-selected 3 x 3 digit kernel (saved (8,1)
    digits one digit up); one wide value in x or dy switches to the full
    kernel.  Against the per-pass weight gradient (full digits) and the oracle."""
    ff, fb, fg = P81, P121, P121
    N, C, H, W, F, K, pad = shape
    rng = np.random.default_rng(23)
    xa = np.array([po.from_float64(8, 1, float(v)) for v in np.abs(rng.normal(0, 1.0, N * C * H * W))],
                  np.uint64).reshape(N, C, H, W)
    dya = np.array([po.from_float64(12, 1, float(v)) for v in rng.normal(0, 0.01, N * F * H * W)],
                   np.uint64).reshape(N, F, H, W)
    if wide == "x":
        xa[1, 0, 3, 3] = po.from_float64(8, 1, 4000.0)
    if wide == "dy":
        dya[0, 1, 2, 2] = po.from_float64(12, 1, 50.0)
    x, dy = dev(ff, xa), dev(fb, dya)
    w = dev(ff, rand_codes(rng, 8, (F, C, K, K)))
    n = ops.conv2d_saved_bytes(ff, x.shape, w.shape, 1, pad)
    saved = torch.empty(n, dtype=torch.uint8, device="cuda")
    ops.conv2d_fwd_save(ff, x, w, None, 1, pad, saved)
    _, dw = ops.conv2d_backward(ff, fb, fg, dy, x, saved, None, x.shape, w.shape, 1, pad, False)
    want = ops.conv2d_weight_grad(fg, dy, ops.convert_tensor(x, ff, fg), w.shape, 1, pad)
    assert torch.equal(dw, want)
    if N * H * W <= 512:
        ref = po.conv2d_weight_grad(12, 1, dya, po.convert_tensor(8, 1, 12, 1, xa), (F, C, K, K), 1, pad)
        assert (host(dw).reshape(ref.shape) == ref).all()


@pytest.mark.parametrize("wide", ["none", "x", "w"])
@pytest.mark.parametrize("shape", [(2, 32, 8, 8, 32, 3, 1), (3, 64, 16, 16, 64, 3, 1), (2, 3, 32, 32, 32, 3, 1)])
def test_fwd_reduced_digits(cuda, po, wide, shape):
    """posit(8,1) forward with x and w within 3 digits takes the device-selected
    3 x 3 digit kernel; one wide value switches to the full kernel.  Against
    the explicit path and the oracle (with bias, relu fused or not)."""
    N, C, H, W, F, K, pad = shape
    rng = np.random.default_rng(29)
    xa = np.array([po.from_float64(8, 1, float(v)) for v in rng.normal(0, 2.0, N * C * H * W)],
                  np.uint64).reshape(N, C, H, W)
    wa = np.array([po.from_float64(8, 1, float(v)) for v in rng.normal(0, 0.2, F * C * K * K)],
                  np.uint64).reshape(F, C, K, K)
    ba = np.array([po.from_float64(8, 1, float(v)) for v in rng.normal(0, 0.1, F)], np.uint64)
    if wide == "x":
        xa[1, 0, 3, 3] = po.from_float64(8, 1, 3000.0)
    if wide == "w":
        wa[2, 1, 1, 1] = po.from_float64(8, 1, -3000.0)
    x, w, b = dev(P81, xa), dev(P81, wa), dev(P81, ba)
    y = ops.conv2d(P81, x, w, b, 1, pad)
    prev = ops.conv_algo(1)
    try:
        ref = ops.conv2d(P81, x, w, b, 1, pad)
    finally:
        ops.conv_algo(prev)
    assert torch.equal(y, ref)
    yr, pre = ops.conv2d_fwd_layer(P81, x, w, b, 1, pad, None, relu=True, want_pre=True)
    assert torch.equal(pre, ref) and torch.equal(yr, ops.relu_fwd(P81, ref))
    # relu(y) as the only output: the magnitude-only / no-wrap epilogue rounding
    yo, none = ops.conv2d_fwd_layer(P81, x, w, b, 1, pad, None, relu=True, want_pre=False)
    assert none is None and torch.equal(yo, yr)
    if N * H * W <= 128:
        want = po.conv2d(8, 1, xa, wa, ba, 1, pad)
        assert (host(y).reshape(want.shape) == want).all()


@pytest.mark.parametrize("shape", [(2, 32, 8, 8, 32, 3, 1), (1, 64, 8, 8, 64, 3, 1)])
def test_fwd_relu_only_three_digit_extremes(cuda, po, shape):
    """posit(8,1) operands at the edge of the 3-digit variant (|x| <= 1024: X = 2^22)
    with equal or random signs: the largest exact sums the reduced kernel can see
    (K = 288: no W-bit wrap possible, the epilogue skips the sign extension; K = 576:
    it does not), partial cancellations down to minpos terms, relu of negative sums."""
    N, C, H, W, F, K, pad = shape
    big, one = po.from_float64(8, 1, 1024.0), po.from_float64(8, 1, 1.0)
    neg = lambda c: (-c) & 0xFF
    pool = np.array([big, big, neg(big), one, neg(one), 1, neg(1), 0], np.uint64)
    for seed, same_sign in ((1, True), (2, False)):
        rng = np.random.default_rng(seed)
        xa = np.full((N, C, H, W), big, np.uint64) if same_sign else pool[rng.integers(0, 8, (N, C, H, W))]
        wa = pool[rng.integers(0, 8, (F, C, K, K))]
        if same_sign:
            wa[: F // 2] = big        # all-positive sums of K * 2^44
            wa[F // 2:] = neg(big)    # all-negative
        ba = pool[rng.integers(0, 8, (F,))]
        x, w, b = dev(P81, xa), dev(P81, wa), dev(P81, ba)
        prev = ops.conv_algo(1)
        try:
            ref = ops.conv2d(P81, x, w, b, 1, pad)
        finally:
            ops.conv_algo(prev)
        yo, none = ops.conv2d_fwd_layer(P81, x, w, b, 1, pad, None, relu=True, want_pre=False)
        assert none is None and torch.equal(yo, ops.relu_fwd(P81, ref))
        y, pre = ops.conv2d_fwd_layer(P81, x, w, b, 1, pad, None, relu=True, want_pre=True)
        assert torch.equal(pre, ref) and torch.equal(y, yo)
        if C <= 32:
            want = po.conv2d(8, 1, xa, wa, ba, 1, pad)
            assert (host(pre).reshape(want.shape) == want).all()


@pytest.mark.parametrize("cfg", [P80, P81])
@pytest.mark.parametrize("shape", [(2, 32, 8, 8, 32, 3, 1), (1, 64, 8, 8, 64, 3, 1)])
def test_fwd_relu_only_extremes(cuda, po, cfg, shape):
    """The relu-only epilogue on sums far beyond maxpos (|quire| >= 2^53, where
    the FP64 conversion drops bits and the dropped-bit check is skipped because
    the value saturates), on wrapped W-bit quires and on exact cancellations:
    operands drawn from {+-maxpos, +-1, +-minpos, 0, NaR}.  Against the explicit
    path and, on the small shape, the oracle."""
    N, C, H, W, F, K, pad = shape
    n = cfg[0]
    maxpos, minpos, one, nar = (1 << (n - 1)) - 1, 1, 1 << (n - 2), 1 << (n - 1)
    neg = lambda c: (-c) & ((1 << n) - 1)
    pool = np.array([maxpos, neg(maxpos), one, neg(one), minpos, neg(minpos), 0, maxpos, neg(maxpos)], np.uint64)
    rng = np.random.default_rng(n * 131 + C)
    xa = pool[rng.integers(0, len(pool), (N, C, H, W))]
    wa = pool[rng.integers(0, len(pool), (F, C, K, K))]
    ba = pool[rng.integers(0, len(pool), (F,))]
    xa[0, 3, 2, 2] = nar
    x, w, b = dev(cfg, xa), dev(cfg, wa), dev(cfg, ba)
    prev = ops.conv_algo(1)
    try:
        ref = ops.conv2d(cfg, x, w, b, 1, pad)
    finally:
        ops.conv_algo(prev)
    yo, none = ops.conv2d_fwd_layer(cfg, x, w, b, 1, pad, None, relu=True, want_pre=False)
    assert none is None and torch.equal(yo, ops.relu_fwd(cfg, ref))
    y, pre = ops.conv2d_fwd_layer(cfg, x, w, b, 1, pad, None, relu=True, want_pre=True)
    assert torch.equal(pre, ref) and torch.equal(y, yo)
    if C <= 32:
        want = po.conv2d(cfg[0], cfg[1], xa, wa, ba, 1, pad)
        assert (host(pre).reshape(want.shape) == want).all()


@pytest.mark.parametrize("cfg", [P121, P161])
@pytest.mark.parametrize("wide", ["none", "x", "dy", "w"])
def test_uniform_121_reduced_digits(cuda, wide, cfg):
    """Uniform posit(12,1) layer (BASELINE config 4): forward and weight gradient
    take the 3-digit variants for narrow values (same-format saved digits, no
    offset); one wide value selects the full kernels.  Against the explicit /
    per-pass paths."""
    from paper_2105_00053_b200 import codec
    N, C, H, W, F, K, pad = 2, 32, 16, 16, 64, 3, 1
    rng = np.random.default_rng(31)
    x64 = np.abs(rng.normal(0, 1.0, (N, C, H, W)))
    w64 = rng.normal(0, 0.2, (F, C, K, K))
    dy64 = rng.normal(0, 0.01, (N, F, H, W))
    if wide == "x":
        x64[1, 3, 4, 5] = 100.0
    if wide == "w":
        w64[0, 0, 1, 1] = -100.0
    if wide == "dy":
        dy64[0, 2, 3, 3] = 50.0
    x, w, dy = (codec.from_float64_device(a, cfg) for a in (x64, w64, dy64))
    b = codec.from_float64_device(rng.normal(0, 0.1, F), cfg)
    n = ops.conv2d_saved_bytes(cfg, x.shape, w.shape, 1, pad)
    saved = torch.empty(n, dtype=torch.uint8, device="cuda")
    y = ops.conv2d_fwd_save(cfg, x, w, b, 1, pad, saved)
    prev = ops.conv_algo(1)
    try:
        yref = ops.conv2d(cfg, x, w, b, 1, pad)
        dwref = ops.conv2d_weight_grad(cfg, dy, x, w.shape, 1, pad)
        dxref = ops.conv2d_input_grad(cfg, dy, w, x.shape, 1, pad)
    finally:
        ops.conv_algo(prev)
    assert torch.equal(y, yref)
    dx, dw = ops.conv2d_backward(cfg, cfg, cfg, dy, x, saved, w, x.shape, w.shape, 1, pad, True)
    assert torch.equal(dw, dwref)
    assert torch.equal(dx, dxref)


@pytest.mark.parametrize("cfg", [P121, P161])
@pytest.mark.parametrize("wide", ["none", "A", "B"])
@pytest.mark.parametrize("shape", [(256, 512, 384), (130, 4096, 96)])
def test_gemm_reduced_digits(cuda, po, wide, shape, cfg):
    """Explicit quire GEMM in posit(12,1) (the Linear layers' path) with values
    within 3 digits takes the device-selected 3 x 3 digit kernel; one wide value
    selects the full kernel.  Against the oracle."""
    M, K, N = shape
    rng = np.random.default_rng(37)
    A = np.array([po.from_float64(cfg[0], cfg[1], float(v)) for v in rng.normal(0, 0.5, M * K)], np.uint64).reshape(M, K)
    B = np.array([po.from_float64(cfg[0], cfg[1], float(v)) for v in rng.normal(0, 0.05, K * N)], np.uint64).reshape(K, N)
    if wide == "A":
        A[3, 7] = po.from_float64(cfg[0], cfg[1], 300.0)
    if wide == "B":
        B[5, 1] = po.from_float64(cfg[0], cfg[1], -300.0)
    got = ops.quire_gemm(cfg, dev(cfg, A), dev(cfg, B))
    want = po.matmul(cfg[0], cfg[1], A, B)
    assert (host(got) == want).all()


@pytest.mark.parametrize("fmt", ["config3", "uniform161"])
def test_cifar_step_with_variants_vs_oracle(cuda, po, fmt):
    """A whole CIFAR-CNN training step with every reduced-digit variant enabled
    (this module's fixture) -- every activation, gradient, loss and updated
    weight against the CPU oracle step."""
    from test_train_gpu import run_and_compare
    from paper_2105_00053_b200 import nn
    st = (nn.StagePrecisions(ops.P81, ops.P121, ops.P121, ops.P161, ops.P161) if fmt == "config3"
          else nn.StagePrecisions.uniform(ops.P161))
    rng = np.random.default_rng(41)
    x = rng.uniform(-1.0, 1.0, (4, 3, 32, 32))
    labels = rng.integers(0, 10, 4)
    model = nn.cifar_cnn(st, seed=5)
    run_and_compare(po, model, st, x, labels, 1.0 / 16, steps=1)
