// C-ABI shim over the UNMODIFIED reference library (TEST INFRASTRUCTURE ONLY).
//
// oracle/Makefile compiles the reference sources where they lie
// (/root/reference/proj/src/{posit,posit_tables,posit_math,quire,tensor,
// tensor_ops}.cpp) together with this file into oracle/_ref/libpnn_ref.so.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg load it: it is the checker and the CPU baseline,
// never the product path.
//
// Every entry point takes posit codes as uint64 (one per element, the
// reference's own Tensor storage, tensor.hpp:74) and calls the reference's
// public API (tensor_ops.hpp:17-61, quire.hpp:18-86, posit.hpp:86-140).
// Errors thrown by the reference (std::invalid_argument) become a nonzero
// return code and a message readable through ref_last_error().
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "pnn/posit.hpp"
#include "pnn/posit_math.hpp"
#include "pnn/posit_tables.hpp"
#include "pnn/quire.hpp"
#include "pnn/tensor.hpp"
#include "pnn/tensor_ops.hpp"
#include "pnn/thread_pool.hpp"

using namespace pnn;

namespace {

thread_local std::string g_err;

PositConfig cfg_of(int nbits, int es) { return PositConfig{nbits, es}; }

Tensor make_tensor(int nbits, int es, std::vector<int64_t> shape, const uint64_t* codes) {
    Tensor t(posit_dtype(cfg_of(nbits, es)), std::move(shape));
    if (t.numel() > 0) std::memcpy(t.data(), codes, size_t(t.numel()) * 8);
    return t;
}

void copy_out(const Tensor& t, uint64_t* out) {
    if (t.numel() > 0) std::memcpy(out, t.data(), size_t(t.numel()) * 8);
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown error";
        return 2;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- scalar layer (posit.hpp) ----

int ref_decode_fixed(int nbits, int es, uint64_t code, int32_t* lsb_scale,
                     uint32_t* sig, uint8_t* neg, uint8_t* nar) {
    return guarded([&] {
        const auto& t = decode_tables(cfg_of(nbits, es));
        const auto& f = t.fixed[code & cfg_of(nbits, es).pattern_mask()];
        *lsb_scale = f.lsb_scale;
        *sig = f.sig;
        *neg = f.neg;
        *nar = f.nar;
    });
}

int ref_unpack(int nbits, int es, uint64_t code, int* cls, int* neg, int* scale,
               uint64_t* sig) {
    return guarded([&] {
        auto u = detail::unpack(cfg_of(nbits, es), code);
        *cls = int(u.cls);
        *neg = u.neg;
        *scale = u.scale;
        *sig = u.sig;
    });
}

uint64_t ref_pack_round(int nbits, int es, int neg, int scale, uint64_t sig, int sticky) {
    return detail::pack_round(cfg_of(nbits, es), neg != 0, scale, sig, sticky != 0);
}

uint64_t ref_convert(int src_nbits, int src_es, int dst_nbits, int dst_es, uint64_t code) {
    return convert(PositValue{cfg_of(src_nbits, src_es), code}, cfg_of(dst_nbits, dst_es)).bits;
}

// op: 0 add, 1 sub, 2 mul, 3 div (posit.hpp:88-95, auto arithmetic path)
uint64_t ref_scalar_op(int nbits, int es, int op, uint64_t a, uint64_t b) {
    PositValue x{cfg_of(nbits, es), a}, y{cfg_of(nbits, es), b};
    switch (op) {
        case 0: return add(x, y).bits;
        case 1: return sub(x, y).bits;
        case 2: return mul(x, y).bits;
        default: return div(x, y).bits;
    }
}

int ref_compare(int nbits, int es, uint64_t a, uint64_t b) {
    return compare(PositValue{cfg_of(nbits, es), a}, PositValue{cfg_of(nbits, es), b});
}

uint64_t ref_from_float64(int nbits, int es, double x) {
    return from_float64(x, cfg_of(nbits, es)).bits;
}

double ref_to_float64(int nbits, int es, uint64_t code) {
    return to_float64(PositValue{cfg_of(nbits, es), code});
}

uint64_t ref_ldexp(int nbits, int es, uint64_t code, int k) {
    return ldexp_posit(PositValue{cfg_of(nbits, es), code}, k).bits;
}

uint64_t ref_round_to_int(int nbits, int es, uint64_t code) {
    return round_to_int(PositValue{cfg_of(nbits, es), code}).bits;
}

int64_t ref_to_int64(int nbits, int es, uint64_t code) {
    return to_int64(PositValue{cfg_of(nbits, es), code});
}

uint64_t ref_exp(int nbits, int es, uint64_t code) {
    return exp_posit(PositValue{cfg_of(nbits, es), code}).bits;
}

uint64_t ref_log(int nbits, int es, uint64_t code) {
    return log_posit(PositValue{cfg_of(nbits, es), code}).bits;
}

uint64_t ref_tanh(int nbits, int es, uint64_t code) {
    return tanh_posit(PositValue{cfg_of(nbits, es), code}).bits;
}

uint64_t ref_sigmoid(int nbits, int es, uint64_t code) {
    return sigmoid_posit(PositValue{cfg_of(nbits, es), code}).bits;
}

uint64_t ref_sqrt(int nbits, int es, uint64_t code) {
    return sqrt_posit(PositValue{cfg_of(nbits, es), code}).bits;
}

uint64_t ref_from_int64(int nbits, int es, int64_t v) {
    return from_int64(v, cfg_of(nbits, es)).bits;
}

// ---- quire (quire.hpp) ----

void* ref_quire_new(int nbits, int es) { return new Quire(cfg_of(nbits, es)); }
void ref_quire_free(void* q) { delete static_cast<Quire*>(q); }
void ref_quire_clear(void* q) { static_cast<Quire*>(q)->clear(); }
void ref_quire_add_posit(void* q, uint64_t a) {
    auto* Q = static_cast<Quire*>(q);
    Q->add_posit(PositValue{Q->config(), a});
}
void ref_quire_add_product(void* q, uint64_t a, uint64_t b) {
    auto* Q = static_cast<Quire*>(q);
    Q->add_product(PositValue{Q->config(), a}, PositValue{Q->config(), b});
}
void ref_quire_sub_product(void* q, uint64_t a, uint64_t b) {
    auto* Q = static_cast<Quire*>(q);
    Q->sub_product(PositValue{Q->config(), a}, PositValue{Q->config(), b});
}
uint64_t ref_quire_to_posit(void* q) { return static_cast<Quire*>(q)->to_posit().bits; }

int ref_fused_dot(int nbits, int es, const uint64_t* a, const uint64_t* b, int64_t len,
                  uint64_t* out) {
    return guarded([&] {
        std::vector<PositValue> va, vb;
        for (int64_t i = 0; i < len; ++i) {
            va.push_back({cfg_of(nbits, es), a[i]});
            vb.push_back({cfg_of(nbits, es), b[i]});
        }
        *out = fused_dot(va, vb).bits;
    });
}

// ---- tensor kernels (tensor_ops.hpp) ----

int ref_matmul(int nbits, int es, const uint64_t* A, const uint64_t* B, uint64_t* C,
               int64_t m, int64_t k, int64_t n, int use_quire, int threads) {
    return guarded([&] {
        Tensor a = make_tensor(nbits, es, {m, k}, A);
        Tensor b = make_tensor(nbits, es, {k, n}, B);
        ThreadPool pool(threads);
        copy_out(matmul(a, b, use_quire != 0, threads > 1 ? &pool : nullptr), C);
    });
}

int ref_conv2d(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H,
               int64_t W, const uint64_t* w, int64_t F, int64_t KH, int64_t KW,
               const uint64_t* bias, int stride, int pad, int use_quire, int threads,
               uint64_t* y) {
    return guarded([&] {
        Tensor xt = make_tensor(nbits, es, {N, C, H, W}, x);
        Tensor wt = make_tensor(nbits, es, {F, C, KH, KW}, w);
        Tensor bt;
        if (bias) bt = make_tensor(nbits, es, {F}, bias);
        ThreadPool pool(threads);
        copy_out(conv2d(xt, wt, bias ? &bt : nullptr, stride, pad, use_quire != 0,
                        threads > 1 ? &pool : nullptr),
                 y);
    });
}

int ref_conv2d_input_grad(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                          int64_t OH, int64_t OW, const uint64_t* w, int64_t C,
                          int64_t KH, int64_t KW, int64_t H, int64_t W, int stride,
                          int pad, int use_quire, int threads, uint64_t* dx) {
    return guarded([&] {
        Tensor dyt = make_tensor(nbits, es, {N, F, OH, OW}, dy);
        Tensor wt = make_tensor(nbits, es, {F, C, KH, KW}, w);
        ThreadPool pool(threads);
        copy_out(conv2d_input_grad(dyt, wt, {N, C, H, W}, stride, pad, use_quire != 0,
                                   threads > 1 ? &pool : nullptr),
                 dx);
    });
}

int ref_conv2d_weight_grad(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                           int64_t OH, int64_t OW, const uint64_t* x, int64_t C,
                           int64_t H, int64_t W, int64_t KH, int64_t KW, int stride,
                           int pad, int use_quire, int threads, uint64_t* dw) {
    return guarded([&] {
        Tensor dyt = make_tensor(nbits, es, {N, F, OH, OW}, dy);
        Tensor xt = make_tensor(nbits, es, {N, C, H, W}, x);
        ThreadPool pool(threads);
        copy_out(conv2d_weight_grad(dyt, xt, {F, C, KH, KW}, stride, pad, use_quire != 0,
                                    threads > 1 ? &pool : nullptr),
                 dw);
    });
}

int ref_conv2d_bias_grad(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                         int64_t OH, int64_t OW, int use_quire, uint64_t* db) {
    return guarded([&] {
        Tensor dyt = make_tensor(nbits, es, {N, F, OH, OW}, dy);
        copy_out(conv2d_bias_grad(dyt, use_quire != 0), db);
    });
}

int ref_column_sum(int nbits, int es, const uint64_t* x, int64_t B, int64_t N,
                   int use_quire, uint64_t* out) {
    return guarded([&] {
        Tensor xt = make_tensor(nbits, es, {B, N}, x);
        copy_out(column_sum(xt, use_quire != 0), out);
    });
}

int ref_maxpool2d(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H,
                  int64_t W, int k, int stride, uint64_t* y, int64_t* argmax) {
    return guarded([&] {
        Tensor xt = make_tensor(nbits, es, {N, C, H, W}, x);
        MaxPoolResult r = maxpool2d(xt, k, stride, nullptr);
        copy_out(r.out, y);
        std::memcpy(argmax, r.argmax.data(), r.argmax.size() * 8);
    });
}

int ref_maxpool2d_backward(int nbits, int es, const uint64_t* dy, int64_t ny,
                           const int64_t* argmax, int64_t N, int64_t C, int64_t H,
                           int64_t W, uint64_t* dx) {
    return guarded([&] {
        Tensor dyt = make_tensor(nbits, es, {ny}, dy);
        std::vector<int64_t> am(argmax, argmax + ny);
        copy_out(maxpool2d_backward(dyt, am, {N, C, H, W}), dx);
    });
}

int ref_avgpool2d(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H,
                  int64_t W, int k, int stride, int use_quire, uint64_t recip, uint64_t* y) {
    return guarded([&] {
        Tensor xt = make_tensor(nbits, es, {N, C, H, W}, x);
        copy_out(avgpool2d(xt, k, stride, use_quire != 0, recip, nullptr), y);
    });
}

int ref_avgpool2d_backward(int nbits, int es, const uint64_t* dy, int64_t N, int64_t C, int64_t H,
                           int64_t W, int k, int stride, uint64_t recip, uint64_t* dx) {
    return guarded([&] {
        const int64_t OH = (H - k) / stride + 1, OW = (W - k) / stride + 1;
        Tensor dyt = make_tensor(nbits, es, {N, C, OH, OW}, dy);
        copy_out(avgpool2d_backward(dyt, k, stride, {N, C, H, W}, recip, nullptr), dx);
    });
}

int ref_convert_tensor(int src_nbits, int src_es, int dst_nbits, int dst_es,
                       const uint64_t* x, int64_t n, uint64_t* y) {
    return guarded([&] {
        Tensor xt = make_tensor(src_nbits, src_es, {n}, x);
        copy_out(convert_tensor(xt, posit_dtype(cfg_of(dst_nbits, dst_es))), y);
    });
}

int ref_ew(int nbits, int es, int op, const uint64_t* a, const uint64_t* b, int64_t n,
           uint64_t* out) {
    return guarded([&] {
        Tensor at = make_tensor(nbits, es, {n}, a);
        Tensor bt = make_tensor(nbits, es, {n}, b);
        Tensor r = op == 0 ? ew_add(at, bt) : op == 1 ? ew_sub(at, bt) : ew_mul(at, bt);
        copy_out(r, out);
    });
}

int ref_scale(int nbits, int es, const uint64_t* a, int64_t n, uint64_t s, uint64_t* out) {
    return guarded([&] { copy_out(scale(make_tensor(nbits, es, {n}, a), s), out); });
}

int ref_ldexp_tensor(int nbits, int es, const uint64_t* a, int64_t n, int k, uint64_t* out) {
    return guarded([&] { copy_out(ldexp_tensor(make_tensor(nbits, es, {n}, a), k), out); });
}

// Wall time (seconds, steady_clock) of one reference quire matmul on
// caller-provided codes -- the CPU baseline timer used by bench.py.
double ref_time_matmul(int nbits, int es, const uint64_t* A, const uint64_t* B,
                       uint64_t* C, int64_t m, int64_t k, int64_t n, int threads) {
    Tensor a = make_tensor(nbits, es, {m, k}, A);
    Tensor b = make_tensor(nbits, es, {k, n}, B);
    ThreadPool pool(threads);
    auto t0 = std::chrono::steady_clock::now();
    Tensor c = matmul(a, b, true, threads > 1 ? &pool : nullptr);
    auto t1 = std::chrono::steady_clock::now();
    copy_out(c, C);
    return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
