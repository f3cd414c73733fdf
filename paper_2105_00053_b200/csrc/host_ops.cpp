// C++ host mirror (include/pnn_b200/tensor_ops.hpp) over the C-ABI.
#include "../../include/pnn_b200/tensor_ops.hpp"

#include <cuda_runtime.h>

#include <mutex>
#include <stdexcept>
#include <string>

#include "../../include/pnn_b200.h"

namespace pnn_b200 {

Tensor::Tensor(PositConfig cfg, std::vector<int64_t> shape) : cfg_(cfg), shape_(std::move(shape)) {
    numel_ = 1;
    for (int64_t d : shape_) {
        if (d < 0) throw std::invalid_argument("Tensor: negative extent");
        numel_ *= d;
    }
    buf_ = std::make_shared<std::vector<uint64_t>>(size_t(numel_), 0);
}

namespace {

void require(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

void check(int rc) {
    if (rc == PNN_OK) return;
    const std::string msg = pnn_last_error();
    if (rc == PNN_EINVAL || rc == PNN_EUNSUPPORTED) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffers + pack/unpack of host uint64 codes.
struct Dev {
    void* p = nullptr;
    size_t bytes = 0;
    explicit Dev(size_t n) : bytes(n) {
        if (n) cuda(cudaMalloc(&p, n), "cudaMalloc");
    }
    ~Dev() {
        if (p) cudaFree(p);
    }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
};

int cb(const PositConfig& c) { return c.nbits <= 8 ? 1 : 2; }

std::unique_ptr<Dev> upload(const Tensor& t) {
    const int b = cb(t.config());
    auto d = std::make_unique<Dev>(size_t(t.numel()) * b);
    std::vector<uint8_t> tmp(size_t(t.numel()) * b);
    const uint64_t m = (uint64_t(1) << t.config().nbits) - 1;
    for (int64_t i = 0; i < t.numel(); ++i) {
        const uint64_t c = t.bits_at(i) & m;
        if (b == 1) tmp[size_t(i)] = uint8_t(c);
        else reinterpret_cast<uint16_t*>(tmp.data())[i] = uint16_t(c);
    }
    if (!tmp.empty()) cuda(cudaMemcpy(d->p, tmp.data(), tmp.size(), cudaMemcpyHostToDevice), "H2D");
    return d;
}

void download(const Dev& d, Tensor& t) {
    const int b = cb(t.config());
    std::vector<uint8_t> tmp(size_t(t.numel()) * b);
    if (!tmp.empty()) cuda(cudaMemcpy(tmp.data(), d.p, tmp.size(), cudaMemcpyDeviceToHost), "D2H");
    for (int64_t i = 0; i < t.numel(); ++i)
        t.set_bits(i, b == 1 ? uint64_t(tmp[size_t(i)])
                             : uint64_t(reinterpret_cast<const uint16_t*>(tmp.data())[i]));
}

void same_cfg(const Tensor& a, const Tensor& b, const char* what) {
    if (!(a.config() == b.config()))
        throw std::invalid_argument(std::string(what) + ": dtype mismatch");
}

void sync() { cuda(cudaDeviceSynchronize(), "sync"); }

}  // namespace

Tensor matmul(const Tensor& a, const Tensor& b, bool use_quire, const void*) {
    require(a.rank() == 2 && b.rank() == 2, "matmul: rank-2 tensors required");
    require(a.dim(1) == b.dim(0), "matmul: inner dimensions disagree");
    same_cfg(a, b, "matmul");
    Tensor c(a.config(), {a.dim(0), b.dim(1)});
    if (!use_quire) {  // matmul_seq: one rounding per term (tensor_ops.cpp:145-164)
        const auto& f = a.config();
        auto da = upload(a), dbb = upload(b);
        Dev out(size_t(c.numel()) * cb(f));
        check(pnn_matmul_seq(f.nbits, f.es, da->p, dbb->p, out.p, a.dim(0), b.dim(1), a.dim(1),
                             nullptr));
        sync();
        download(out, c);
        return c;
    }
    check(pnn_matmul_host(a.config().nbits, a.config().es, a.data(), b.data(), c.data(), a.dim(0),
                          a.dim(1), b.dim(1)));
    return c;
}

Tensor par_matmul(const Tensor& a, const Tensor& b, bool use_quire, int) {
    return matmul(a, b, use_quire, nullptr);
}

Tensor conv2d(const Tensor& x, const Tensor& w, const Tensor* bias, int stride, int pad,
              bool use_quire, const void*) {
    require(x.rank() == 4 && w.rank() == 4, "conv2d: NCHW/FCKK tensors required");
    require(stride >= 1 && pad >= 0, "conv2d: bad stride/pad");
    same_cfg(x, w, "conv2d");
    if (bias) {
        same_cfg(x, *bias, "conv2d bias");
        require(bias->numel() == w.dim(0), "conv2d: bias size mismatch");
    }
    require(w.dim(1) == x.dim(1), "conv2d: channel mismatch");
    const auto& f = x.config();
    const int64_t N = x.dim(0), C = x.dim(1), H = x.dim(2), W = x.dim(3), F = w.dim(0),
                  KH = w.dim(2), KW = w.dim(3);
    require(H + 2 * pad >= KH && W + 2 * pad >= KW, "conv2d: kernel larger than input");
    const int64_t OH = (H + 2 * pad - KH) / stride + 1, OW = (W + 2 * pad - KW) / stride + 1;
    Tensor y(f, {N, F, OH, OW});
    auto dx = upload(x), dw = upload(w);
    std::unique_ptr<Dev> db = bias ? upload(*bias) : nullptr;
    Dev dy(size_t(y.numel()) * cb(f));
    if (!use_quire) {  // conv_seq (tensor_ops.cpp:232-264)
        check(pnn_conv2d_fwd_seq(f.nbits, f.es, dx->p, N, C, H, W, dw->p, F, KH, KW,
                                 db ? db->p : nullptr, stride, pad, dy.p, nullptr));
        sync();
        download(dy, y);
        return y;
    }
    size_t ws = 0;
    check(pnn_conv2d_workspace(0, f.nbits, f.es, N, C, H, W, F, KH, KW, stride, pad, bias != nullptr,
                               &ws));
    Dev work(ws);
    check(pnn_conv2d_fwd(f.nbits, f.es, dx->p, N, C, H, W, dw->p, F, KH, KW, db ? db->p : nullptr,
                         stride, pad, dy.p, work.p, ws, nullptr));
    sync();
    download(dy, y);
    return y;
}

Tensor conv2d_input_grad(const Tensor& dy, const Tensor& w, const std::vector<int64_t>& x_shape,
                         int stride, int pad, bool use_quire, const void*) {
    require(dy.rank() == 4 && w.rank() == 4 && x_shape.size() == 4, "conv2d_input_grad: bad ranks");
    same_cfg(dy, w, "conv2d_input_grad");
    const auto& f = dy.config();
    const int64_t N = x_shape[0], C = x_shape[1], H = x_shape[2], W = x_shape[3];
    require(stride >= 1 && pad >= 0, "conv2d_input_grad: bad stride/pad");
    require(N >= 0 && C >= 1 && H >= 1 && W >= 1, "conv2d_input_grad: bad x_shape");
    require(w.dim(1) == C, "conv2d_input_grad: channel mismatch (w vs x_shape)");
    require(dy.dim(0) == N && dy.dim(1) == w.dim(0), "conv2d_input_grad: dy does not match x_shape / w");
    require(H + 2 * pad >= w.dim(2) && W + 2 * pad >= w.dim(3), "conv2d_input_grad: kernel larger than input");
    require(dy.dim(2) == (H + 2 * pad - w.dim(2)) / stride + 1 && dy.dim(3) == (W + 2 * pad - w.dim(3)) / stride + 1,
            "conv2d_input_grad: dy spatial size does not match the convolution");
    Tensor dx(f, x_shape);
    auto ddy = upload(dy), dw = upload(w);
    Dev out(size_t(dx.numel()) * cb(f));
    if (!use_quire) {  // gather_seq (tensor_ops.cpp:302-318)
        check(pnn_conv2d_dgrad_seq(f.nbits, f.es, ddy->p, N, dy.dim(1), dy.dim(2), dy.dim(3), dw->p,
                                   C, w.dim(2), w.dim(3), H, W, stride, pad, out.p, nullptr));
        sync();
        download(out, dx);
        return dx;
    }
    size_t ws = 0;
    check(pnn_conv2d_workspace(1, f.nbits, f.es, N, C, H, W, w.dim(0), w.dim(2), w.dim(3), stride,
                               pad, 0, &ws));
    Dev work(ws);
    check(pnn_conv2d_dgrad(f.nbits, f.es, ddy->p, N, dy.dim(1), dy.dim(2), dy.dim(3), dw->p, C,
                           w.dim(2), w.dim(3), H, W, stride, pad, out.p, work.p, ws, nullptr));
    sync();
    download(out, dx);
    return dx;
}

Tensor conv2d_weight_grad(const Tensor& dy, const Tensor& x, const std::vector<int64_t>& w_shape,
                          int stride, int pad, bool use_quire, const void*) {
    require(dy.rank() == 4 && x.rank() == 4 && w_shape.size() == 4, "conv2d_weight_grad: bad ranks");
    same_cfg(dy, x, "conv2d_weight_grad");
    const auto& f = dy.config();
    require(stride >= 1 && pad >= 0, "conv2d_weight_grad: bad stride/pad");
    require(w_shape[0] == dy.dim(1) && w_shape[1] == x.dim(1), "conv2d_weight_grad: w_shape does not match dy / x");
    require(dy.dim(0) == x.dim(0), "conv2d_weight_grad: batch mismatch");
    require(w_shape[2] >= 1 && w_shape[3] >= 1 && x.dim(2) + 2 * pad >= w_shape[2] &&
                x.dim(3) + 2 * pad >= w_shape[3],
            "conv2d_weight_grad: kernel larger than input");
    require(dy.dim(2) == (x.dim(2) + 2 * pad - w_shape[2]) / stride + 1 &&
                dy.dim(3) == (x.dim(3) + 2 * pad - w_shape[3]) / stride + 1,
            "conv2d_weight_grad: dy spatial size does not match the convolution");
    Tensor dw(f, w_shape);
    auto ddy = upload(dy), dx = upload(x);
    Dev out(size_t(dw.numel()) * cb(f));
    if (!use_quire) {  // gather_seq over (n, oy, ox) (tensor_ops.cpp:302-318, 586-600)
        check(pnn_conv2d_wgrad_seq(f.nbits, f.es, ddy->p, dy.dim(0), dy.dim(1), dy.dim(2), dy.dim(3),
                                   dx->p, x.dim(1), x.dim(2), x.dim(3), w_shape[2], w_shape[3], stride,
                                   pad, out.p, nullptr));
        sync();
        download(out, dw);
        return dw;
    }
    size_t ws = 0;
    check(pnn_conv2d_workspace(2, f.nbits, f.es, x.dim(0), x.dim(1), x.dim(2), x.dim(3), w_shape[0],
                               w_shape[2], w_shape[3], stride, pad, 0, &ws));
    Dev work(ws);
    check(pnn_conv2d_wgrad(f.nbits, f.es, ddy->p, dy.dim(0), dy.dim(1), dy.dim(2), dy.dim(3), dx->p,
                           x.dim(1), x.dim(2), x.dim(3), w_shape[2], w_shape[3], stride, pad, out.p,
                           nullptr, nullptr, work.p, ws, nullptr));
    sync();
    download(out, dw);
    return dw;
}

static Tensor bias_sum(const Tensor& t, int64_t N, int64_t F, int64_t P, bool use_quire) {
    const auto& f = t.config();
    Tensor db(f, {F});
    auto d = upload(t);
    Dev out(size_t(F) * cb(f));
    if (!use_quire) {  // gather_seq_sum (tensor_ops.cpp:320-335)
        check(pnn_bias_grad_seq(f.nbits, f.es, d->p, N, F, P, out.p, nullptr));
        sync();
        download(out, db);
        return db;
    }
    size_t ws = 0;
    check(pnn_bias_grad_workspace(F, &ws));
    Dev work(ws);
    check(pnn_bias_grad(f.nbits, f.es, d->p, N, F, P, out.p, nullptr, nullptr, work.p, ws, nullptr));
    sync();
    download(out, db);
    return db;
}

Tensor conv2d_bias_grad(const Tensor& dy, bool use_quire) {
    require(dy.rank() == 4, "conv2d_bias_grad: bad rank");
    return bias_sum(dy, dy.dim(0), dy.dim(1), dy.dim(2) * dy.dim(3), use_quire);
}

Tensor column_sum(const Tensor& x, bool use_quire) {
    require(x.rank() == 2, "column_sum: rank-2 tensor required");
    return bias_sum(x, x.dim(0), x.dim(1), 1, use_quire);
}

MaxPoolResult maxpool2d(const Tensor& x, int k, int stride, const void*) {
    require(x.rank() == 4, "maxpool2d: NCHW tensor required");
    require(x.dim(2) >= k && x.dim(3) >= k, "maxpool2d: window larger than input");
    const auto& f = x.config();
    const int64_t OH = (x.dim(2) - k) / stride + 1, OW = (x.dim(3) - k) / stride + 1;
    MaxPoolResult r{Tensor(f, {x.dim(0), x.dim(1), OH, OW}), {}};
    r.argmax.resize(size_t(r.out.numel()));
    auto dx = upload(x);
    Dev y(size_t(r.out.numel()) * cb(f)), am(size_t(r.out.numel()) * 8);
    check(pnn_maxpool2d_fwd(f.nbits, f.es, dx->p, x.dim(0), x.dim(1), x.dim(2), x.dim(3), k, stride,
                            y.p, static_cast<int64_t*>(am.p), nullptr));
    sync();
    download(y, r.out);
    if (!r.argmax.empty())
        cuda(cudaMemcpy(r.argmax.data(), am.p, am.bytes, cudaMemcpyDeviceToHost), "D2H argmax");
    return r;
}

// tensor_ops.cpp:658-670: window-independent, outputs added per target in
// increasing output order (pnn_maxpool2d_bwd_scatter).
Tensor maxpool2d_backward(const Tensor& dy, const std::vector<int64_t>& argmax,
                          const std::vector<int64_t>& x_shape) {
    require(size_t(dy.numel()) == argmax.size(), "maxpool2d_backward: argmax mismatch");
    const auto& f = dy.config();
    Tensor dx(f, x_shape);
    for (int64_t t : argmax)  // undefined behaviour in the reference: rejected here
        require(t >= 0 && t < dx.numel(), "maxpool2d_backward: argmax index out of range");
    auto ddy = upload(dy);
    Dev am(argmax.size() * 8), out(size_t(dx.numel()) * cb(f));
    if (!argmax.empty())
        cuda(cudaMemcpy(am.p, argmax.data(), am.bytes, cudaMemcpyHostToDevice), "H2D argmax");
    size_t ws = 0;
    check(pnn_maxpool2d_bwd_scatter_workspace(dy.numel(), dx.numel(), &ws));
    Dev work(ws);
    check(pnn_maxpool2d_bwd_scatter(f.nbits, f.es, ddy->p, static_cast<const int64_t*>(am.p), dy.numel(),
                                    out.p, dx.numel(), work.p, ws, nullptr));
    sync();
    download(out, dx);
    return dx;
}

Tensor maxpool2d_backward(const Tensor& dy, const std::vector<int64_t>& argmax,
                          const std::vector<int64_t>& x_shape, int k, int stride) {
    require(size_t(dy.numel()) == argmax.size(), "maxpool2d_backward: argmax mismatch");
    require(x_shape.size() == 4, "maxpool2d_backward: NCHW shape required");
    require(k >= 1 && stride >= 1 && x_shape[2] >= k && x_shape[3] >= k, "maxpool2d_backward: bad window");
    const int64_t OH = (x_shape[2] - k) / stride + 1, OW = (x_shape[3] - k) / stride + 1;
    require(dy.rank() == 4 && dy.dim(0) == x_shape[0] && dy.dim(1) == x_shape[1] && dy.dim(2) == OH &&
                dy.dim(3) == OW,
            "maxpool2d_backward: dy is not the (N, C, OH, OW) output of this window");
    // every argmax must lie in its own window (else the 3-argument scatter applies)
    for (int64_t o = 0; o < dy.numel(); ++o) {
        const int64_t ox = o % OW, oy = (o / OW) % OH, nc = o / (OW * OH);
        const int64_t t = argmax[size_t(o)], ix = t % x_shape[3], iy = (t / x_shape[3]) % x_shape[2];
        require(t >= 0 && t / (x_shape[2] * x_shape[3]) == nc && iy >= oy * stride && iy < oy * stride + k &&
                    ix >= ox * stride && ix < ox * stride + k,
                "maxpool2d_backward: argmax outside its window");
    }
    const auto& f = dy.config();
    Tensor dx(f, x_shape);
    auto ddy = upload(dy);
    Dev am(argmax.size() * 8), out(size_t(dx.numel()) * cb(f));
    if (!argmax.empty())
        cuda(cudaMemcpy(am.p, argmax.data(), am.bytes, cudaMemcpyHostToDevice), "H2D argmax");
    check(pnn_maxpool2d_bwd(f.nbits, f.es, ddy->p, static_cast<const int64_t*>(am.p), x_shape[0],
                            x_shape[1], x_shape[2], x_shape[3], k, stride, out.p, nullptr));
    sync();
    download(out, dx);
    return dx;
}

Tensor convert_tensor(const Tensor& t, const PositConfig& target) {
    if (t.config() == target) return t;
    Tensor out(target, t.shape());
    auto d = upload(t);
    Dev o(size_t(t.numel()) * cb(target));
    check(pnn_convert(t.config().nbits, t.config().es, target.nbits, target.es, d->p, o.p, t.numel(),
                      nullptr));
    sync();
    download(o, out);
    return out;
}

}  // namespace pnn_b200
