// C++ drop-in check: the reference's own tensor-test style (test_tensor.cpp)
// against include/pnn_b200/tensor_ops.hpp, compared bit for bit with the CPU
// oracle restatement (oracle/posit_oracle.h).  Built and run by
// tests/test_cpp_host_gpu.py on the GPU box.
#include <cstdio>
#include <random>
#include <stdexcept>

#include "pnn_b200/tensor_ops.hpp"

extern "C" {
#include "../../oracle/posit_oracle.h"
}

using pnn_b200::PositConfig;
using pnn_b200::Tensor;

static int failures = 0;
#define EXPECT(c)                                                      \
    do {                                                               \
        if (!(c)) {                                                    \
            std::fprintf(stderr, "%s:%d: EXPECT(%s)\n", __FILE__, __LINE__, #c); \
            ++failures;                                                \
        }                                                              \
    } while (0)

static Tensor rand_tensor(PositConfig c, std::vector<int64_t> shape, uint64_t seed) {
    Tensor t(c, std::move(shape));
    std::mt19937_64 rng(seed);
    const uint64_t nar = uint64_t(1) << (c.nbits - 1);
    for (int64_t i = 0; i < t.numel(); ++i) {
        uint64_t v;
        do { v = rng() & ((uint64_t(1) << c.nbits) - 1); } while (v == nar);
        t.set_bits(i, v);
    }
    return t;
}

int main() {
    const PositConfig p80{8, 0}, p161{16, 1}, p121{12, 1};
    // test_tensor.cpp:52-62 -- 1x16 ones . 16x1 ones -> 16 with the quire
    Tensor r(p80, {1, 16}), c(p80, {16, 1});
    for (int i = 0; i < 16; ++i) r.set_bits(i, 0x40), c.set_bits(i, 0x40);
    EXPECT(po_to_float64(8, 0, pnn_b200::matmul(r, c, true).bits_at(0)) == 16.0);
    // test_tensor.cpp:64-74 -- cancellation keeps minpos^2 -> minpos
    Tensor a(p80, {1, 3}), b(p80, {3, 1});
    a.set_bits(0, po_from_float64(8, 0, 64)); a.set_bits(1, 1); a.set_bits(2, po_from_float64(8, 0, -64));
    b.set_bits(0, 0x40); b.set_bits(1, 1); b.set_bits(2, 0x40);
    EXPECT(pnn_b200::matmul(a, b, true).bits_at(0) == 1);
    // errors are std::invalid_argument like the reference (tensor_ops.cpp:17-27)
    bool threw = false;
    try { pnn_b200::matmul(r, r, true); } catch (const std::invalid_argument&) { threw = true; }
    EXPECT(threw);
    threw = false;
    try { pnn_b200::matmul(a, rand_tensor(p161, {3, 1}, 1), true); } catch (const std::invalid_argument&) { threw = true; }
    EXPECT(threw);
    // random parity vs the oracle, every op of the hot path
    for (PositConfig f : {p80, p121, p161}) {
        Tensor A = rand_tensor(f, {37, 53}, 11), B = rand_tensor(f, {53, 29}, 12);
        Tensor Cg = pnn_b200::matmul(A, B, true);
        std::vector<uint64_t> Cw(37 * 29);
        po_matmul(f.nbits, f.es, A.data(), B.data(), Cw.data(), 37, 53, 29);
        for (int i = 0; i < 37 * 29; ++i) EXPECT(Cg.bits_at(i) == Cw[size_t(i)]);
        Tensor x = rand_tensor(f, {2, 3, 9, 8}, 13), w = rand_tensor(f, {4, 3, 3, 3}, 14), bias = rand_tensor(f, {4}, 15);
        Tensor y = pnn_b200::conv2d(x, w, &bias, 1, 1, true);
        std::vector<uint64_t> yw(size_t(y.numel()));
        po_conv2d(f.nbits, f.es, x.data(), 2, 3, 9, 8, w.data(), 4, 3, 3, bias.data(), 1, 1, yw.data());
        for (int64_t i = 0; i < y.numel(); ++i) EXPECT(y.bits_at(i) == yw[size_t(i)]);
        Tensor dy = rand_tensor(f, y.shape(), 16);
        Tensor dx = pnn_b200::conv2d_input_grad(dy, w, x.shape(), 1, 1, true);
        std::vector<uint64_t> dxw(size_t(dx.numel()));
        po_conv2d_input_grad(f.nbits, f.es, dy.data(), 2, 4, 9, 8, w.data(), 3, 3, 3, 9, 8, 1, 1, dxw.data());
        for (int64_t i = 0; i < dx.numel(); ++i) EXPECT(dx.bits_at(i) == dxw[size_t(i)]);
        Tensor dw = pnn_b200::conv2d_weight_grad(dy, x, w.shape(), 1, 1, true);
        std::vector<uint64_t> dww(size_t(dw.numel()));
        po_conv2d_weight_grad(f.nbits, f.es, dy.data(), 2, 4, 9, 8, x.data(), 3, 9, 8, 3, 3, 1, 1, dww.data());
        for (int64_t i = 0; i < dw.numel(); ++i) EXPECT(dw.bits_at(i) == dww[size_t(i)]);
        Tensor db = pnn_b200::conv2d_bias_grad(dy, true);
        std::vector<uint64_t> dbw(4);
        po_conv2d_bias_grad(f.nbits, f.es, dy.data(), 2, 4, 9, 8, dbw.data());
        for (int i = 0; i < 4; ++i) EXPECT(db.bits_at(i) == dbw[size_t(i)]);
        auto mp = pnn_b200::maxpool2d(x, 2, 2);
        std::vector<uint64_t> mpw(size_t(mp.out.numel()));
        std::vector<int64_t> amw(mpw.size());
        po_maxpool2d(f.nbits, f.es, x.data(), 2, 3, 9, 8, 2, 2, mpw.data(), amw.data());
        for (int64_t i = 0; i < mp.out.numel(); ++i) EXPECT(mp.out.bits_at(i) == mpw[size_t(i)] && mp.argmax[size_t(i)] == amw[size_t(i)]);
        Tensor conv = pnn_b200::convert_tensor(x, p80);
        for (int64_t i = 0; i < x.numel(); ++i) EXPECT(conv.bits_at(i) == po_convert(f.nbits, f.es, 8, 0, x.bits_at(i)));
        // use_quire = false: the sequential-rounding kernels (tensor_ops.cpp:145-164, 232-335)
        Tensor Cs = pnn_b200::matmul(A, B, false);
        po_matmul_seq(f.nbits, f.es, A.data(), B.data(), Cw.data(), 37, 53, 29);
        for (int i = 0; i < 37 * 29; ++i) EXPECT(Cs.bits_at(i) == Cw[size_t(i)]);
        Tensor ys = pnn_b200::conv2d(x, w, &bias, 1, 1, false);
        po_conv2d_seq(f.nbits, f.es, x.data(), 2, 3, 9, 8, w.data(), 4, 3, 3, bias.data(), 1, 1, yw.data());
        for (int64_t i = 0; i < ys.numel(); ++i) EXPECT(ys.bits_at(i) == yw[size_t(i)]);
        Tensor dxs = pnn_b200::conv2d_input_grad(dy, w, x.shape(), 1, 1, false);
        po_conv2d_input_grad_seq(f.nbits, f.es, dy.data(), 2, 4, 9, 8, w.data(), 3, 3, 3, 9, 8, 1, 1, dxw.data());
        for (int64_t i = 0; i < dxs.numel(); ++i) EXPECT(dxs.bits_at(i) == dxw[size_t(i)]);
        Tensor dws = pnn_b200::conv2d_weight_grad(dy, x, w.shape(), 1, 1, false);
        po_conv2d_weight_grad_seq(f.nbits, f.es, dy.data(), 2, 4, 9, 8, x.data(), 3, 9, 8, 3, 3, 1, 1, dww.data());
        for (int64_t i = 0; i < dws.numel(); ++i) EXPECT(dws.bits_at(i) == dww[size_t(i)]);
        Tensor dbs = pnn_b200::conv2d_bias_grad(dy, false);
        po_bias_grad_seq(f.nbits, f.es, dy.data(), 2, 4, 9 * 8, dbw.data());
        for (int i = 0; i < 4; ++i) EXPECT(dbs.bits_at(i) == dbw[size_t(i)]);
    }
    // maxpool2d_backward, reference signature (tensor_ops.cpp:658-670): any
    // window -- overlapping 3x3/2 and tiled 3x3/3 -- and an arbitrary argmax
    // with collisions, each vs the oracle's sequential scatter.
    for (PositConfig f : {p80, p121, p161}) {
        for (int k : {2, 3}) {
            for (int s : {1, 2, 3}) {
                Tensor x = rand_tensor(f, {2, 3, 6, 7}, 40 + k * 3 + s);
                auto mp = pnn_b200::maxpool2d(x, k, s);
                std::vector<uint64_t> yw(size_t(mp.out.numel()));
                std::vector<int64_t> amw(size_t(mp.out.numel()));
                po_maxpool2d(f.nbits, f.es, x.data(), 2, 3, 6, 7, k, s, yw.data(), amw.data());
                for (int64_t i = 0; i < mp.out.numel(); ++i) {
                    EXPECT(mp.out.bits_at(i) == yw[size_t(i)]);
                    EXPECT(mp.argmax[size_t(i)] == amw[size_t(i)]);
                }
                Tensor dy = rand_tensor(f, mp.out.shape(), 50 + k * 3 + s);
                std::vector<uint64_t> dxw(size_t(x.numel()));
                po_maxpool2d_backward(f.nbits, f.es, dy.data(), dy.numel(), mp.argmax.data(), x.numel(),
                                      dxw.data());
                Tensor dx = pnn_b200::maxpool2d_backward(dy, mp.argmax, x.shape());
                for (int64_t i = 0; i < x.numel(); ++i) EXPECT(dx.bits_at(i) == dxw[size_t(i)]);
                Tensor dx2 = pnn_b200::maxpool2d_backward(dy, mp.argmax, x.shape(), k, s);
                for (int64_t i = 0; i < x.numel(); ++i) EXPECT(dx2.bits_at(i) == dxw[size_t(i)]);
            }
        }
        // arbitrary argmax: 500 outputs onto 40 targets (many collisions)
        Tensor dy = rand_tensor(f, {500}, 61);
        std::vector<int64_t> am(500);
        std::mt19937_64 rng(62);
        for (auto& t : am) t = int64_t(rng() % 40);
        std::vector<uint64_t> dxw(40);
        po_maxpool2d_backward(f.nbits, f.es, dy.data(), 500, am.data(), 40, dxw.data());
        Tensor dx = pnn_b200::maxpool2d_backward(dy, am, {1, 1, 5, 8});
        for (int i = 0; i < 40; ++i) EXPECT(dx.bits_at(i) == dxw[size_t(i)]);
        // window mismatch / out-of-range targets throw instead of reading past dy
        Tensor x = rand_tensor(f, {1, 2, 6, 6}, 63);
        auto mp = pnn_b200::maxpool2d(x, 3, 3);
        bool threw = false;
        try { pnn_b200::maxpool2d_backward(mp.out, mp.argmax, x.shape(), 2, 2); }
        catch (const std::invalid_argument&) { threw = true; }
        EXPECT(threw);
        threw = false;
        am.assign(500, 40);
        try { pnn_b200::maxpool2d_backward(dy, am, {1, 1, 5, 8}); }
        catch (const std::invalid_argument&) { threw = true; }
        EXPECT(threw);
    }
    // conv gradient shape cross-checks (std::invalid_argument, no device access)
    {
        Tensor x = rand_tensor(p80, {2, 3, 9, 8}, 70), w = rand_tensor(p80, {4, 3, 3, 3}, 71);
        Tensor dy = rand_tensor(p80, {2, 4, 9, 8}, 72), dy_bad = rand_tensor(p80, {2, 5, 9, 8}, 73);
        int throws = 0;
        try { pnn_b200::conv2d_weight_grad(dy, x, {5, 3, 3, 3}, 1, 1, true); } catch (const std::invalid_argument&) { ++throws; }
        try { pnn_b200::conv2d_weight_grad(dy, x, {4, 2, 3, 3}, 1, 1, true); } catch (const std::invalid_argument&) { ++throws; }
        try { pnn_b200::conv2d_weight_grad(rand_tensor(p80, {3, 4, 9, 8}, 74), x, w.shape(), 1, 1, true); } catch (const std::invalid_argument&) { ++throws; }
        try { pnn_b200::conv2d_weight_grad(dy, x, w.shape(), 1, 0, true); } catch (const std::invalid_argument&) { ++throws; }
        try { pnn_b200::conv2d_input_grad(dy_bad, w, x.shape(), 1, 1, true); } catch (const std::invalid_argument&) { ++throws; }
        try { pnn_b200::conv2d_input_grad(dy, w, {2, 2, 9, 8}, 1, 1, true); } catch (const std::invalid_argument&) { ++throws; }
        try { pnn_b200::conv2d_input_grad(dy, w, {2, 3, 9, 8}, 2, 1, true); } catch (const std::invalid_argument&) { ++throws; }
        EXPECT(throws == 7);
    }
    std::printf("host_ops_test: %s (%d failures)\n", failures ? "FAILED" : "ok", failures);
    return failures ? 1 : 0;
}
