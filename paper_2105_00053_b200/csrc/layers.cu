// The remaining SPEC layers on the device: tanh /
// sigmoid layers (forward + backward), dropout, MSE loss, batch
// normalisation, and SGD with momentum.
//
// The reference has no layer code for these (placeholders);
// SPEC.md:326-353 names them.  The rounding sequence of each is written out
// in oracle/layers_oracle.c and mirrored here op for op: every scalar step is
// one correctly rounded posit op (posit_scalar.cuh), every reduction is one
// exact quire (128-bit two's complement at LSB 2^-2R, masked to W bits, one
// rounding) -- so results are bit-identical to the oracle, independent of
// the grid shape.
//
// All of these are HBM-bound elementwise / per-channel reductions: grids are
// sized in SM multiples, each reduction is split over (chunk, channel)
// blocks that write 128-bit partial quires, and the consumers re-reduce the
// partials (<= 64 per channel) instead of launching a separate finalize.
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/pnn_b200.h"
#include "eltwise_common.cuh"
#include "posit_scalar.cuh"
#include "status.h"

namespace pnn_b200 {
namespace {

typedef unsigned __int128 u128;
typedef __int128 i128;

constexpr int kBnMaxSplit = 64;  // partial quires per channel
constexpr int kSms = 148;

bool elt_ok(int nbits, int es) {
    if (nbits < 2 || nbits > 16 || es < 0 || es > 4) return false;
    return 2 * make_fmt(nbits, es).R <= 96;
}
// formats whose quire fits the 128-bit accumulator (W <= 128, 2R <= 56)
bool quire_ok(int nbits, int es) { return elt_ok(nbits, es) && make_fmt(nbits, es).W <= 128; }

int bytes_of(int nbits) { return nbits <= 8 ? 1 : 2; }

int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > kSms * 16) b = kSms * 16;
    return int(b < 1 ? 1 : b);
}

int launched(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return PNN_OK;
    return set_status(PNN_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int unsupported(const char* what) {
    return set_status(PNN_EUNSUPPORTED, std::string(what) + ": format not supported");
}

}  // namespace

// ---- quire helpers (W <= 128) ----------------------------------------------

// Quire::add(posit): X * 2^R at LSB 2^-2R.
__device__ __forceinline__ void q_add(u128& acc, bool& nar, const PositFmt& f, uint32_t c) {
    int64_t X;
    nar |= decode_x(c, f, X);
    acc += (u128)(i128)X << f.R;
}
// Quire::add_product: Xa * Xb at LSB 2^-2R (|X| <= 2^56, product < 2^113).
__device__ __forceinline__ void q_fma(u128& acc, bool& nar, const PositFmt& f, uint32_t a,
                                      uint32_t b) {
    int64_t Xa, Xb;
    nar |= decode_x(a, f, Xa);
    nar |= decode_x(b, f, Xb);
    acc += (u128)((i128)Xa * (i128)Xb);
}

// Block-wide sum of a 128-bit word (result valid in thread 0).
__device__ u128 block_sum(u128 v) {
    __shared__ unsigned long long lo_s[32], hi_s[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t l = __shfl_xor_sync(0xFFFFFFFFu, uint64_t(v), o);
        const uint64_t h = __shfl_xor_sync(0xFFFFFFFFu, uint64_t(v >> 64), o);
        v += ((u128)h << 64) | l;
    }
    __syncthreads();  // lo_s / hi_s reuse across calls
    if (lane == 0) {
        lo_s[warp] = uint64_t(v);
        hi_s[warp] = uint64_t(v >> 64);
    }
    __syncthreads();
    u128 s = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < int(blockDim.x >> 5); ++w) s += ((u128)hi_s[w] << 64) | lo_s[w];
    return s;
}

__device__ __forceinline__ uint32_t q_round(const PositFmt& f, u128 acc, bool nar) {
    return nar ? nar_of(f) : quire_to_posit(f, acc);
}
__device__ __forceinline__ u128 q_word(const PositFmt& f, u128 acc) {
    const u128 one = 1;
    return f.W >= 128 ? acc : (acc & ((one << f.W) - 1));
}

// ---- activations -----------------------------------------------------------

__global__ void act_fwd_kernel(int kind, PositFmt f, int b, const void* x, void* y, int64_t n) {
    GRID_STRIDE(i, n) {
        const uint32_t v = load_any(x, i, b);
        store_any(y, i, b, kind == 1 ? p_tanh(f, v) : p_sigmoid(f, v));
    }
}

// tanh: dx = dy * (1 - yb*yb); sigmoid: dx = dy * (yb * (1 - yb)); all in b.
__global__ void act_bwd_kernel(int kind, PositFmt ff, int fb, const void* y, PositFmt bf, int bb,
                               const void* dy, void* dx, int64_t n) {
    const uint32_t one = p_from_int64(bf, 1);
    GRID_STRIDE(i, n) {
        const uint32_t yb = p_convert(ff, bf, load_any(y, i, fb));
        const uint32_t t =
            kind == 1 ? p_sub(bf, one, p_mul(bf, yb, yb)) : p_mul(bf, yb, p_sub(bf, one, yb));
        store_any(dx, i, bb, p_mul(bf, load_any(dy, i, bb), t));
    }
}

// ---- dropout ----------------------------------------------------------------

__device__ __forceinline__ uint64_t dropout_bits(uint64_t seed, int64_t i) {
    uint64_t z = seed ^ (uint64_t(i) * 0xD1B54A32D192ED03ull);
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void dropout_kernel(PositFmt f, int b, const void* x, void* y, int64_t n, uint64_t seed,
                               const uint64_t* seed_offset, uint32_t thresh, uint32_t scale) {
    if (seed_offset) seed += *seed_offset;
    GRID_STRIDE(i, n) {
        const bool keep = uint32_t(dropout_bits(seed, i) >> 32) >= thresh;
        store_any(y, i, b, keep ? p_mul(f, load_any(x, i, b), scale) : 0u);
    }
}

// ---- MSE loss (one block: the loss is a scalar over B x outputs) -----------

__global__ void mse_kernel(PositFmt f, int b, const void* y, const void* t, int64_t n, int64_t G,
                           int grad_scale_log2, void* grad, void* loss_out) {
    const uint32_t g = p_from_int64(f, G);
    const uint32_t c = p_div(f, p_from_int64(f, 2), g);
    u128 acc = 0;
    bool nar = false;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t d = p_sub(f, load_any(y, i, b), load_any(t, i, b));
        q_fma(acc, nar, f, d, d);
        uint32_t gi = p_mul(f, d, c);
        if (grad_scale_log2) gi = p_ldexp(f, gi, grad_scale_log2);
        store_any(grad, i, b, gi);
    }
    nar = __syncthreads_or(nar);
    const u128 s = block_sum(acc);
    if (threadIdx.x == 0 && loss_out) store_any(loss_out, 0, b, p_div(f, q_round(f, s, nar), g));
}

// ---- batch normalisation ------------------------------------------------------
// x [N, C, HW]; block (s, c) owns elements [s*chunk, (s+1)*chunk) of channel c
// (element e -> n = e / HW, p = e % HW).  Partial quires: ws[q][c][S].

struct BnGeom {
    int64_t N, C, HW;
    int M, S, chunk;
};

__device__ __forceinline__ int64_t bn_index(const BnGeom& g, int c, int e) {
    const int n = e / int(g.HW), p = e - n * int(g.HW);
    return (int64_t(n) * g.C + c) * g.HW + p;
}

// Reduce partial quire q of channel c (thread 0 gets the sum).
__device__ u128 bn_gather(const u128* ws, const uint8_t* wsn, int q, const BnGeom& g, int c,
                          bool& nar) {
    u128 v = 0;
    bool nr = false;
    for (int s = threadIdx.x; s < g.S; s += blockDim.x) {
        v += ws[(int64_t(q) * g.C + c) * g.S + s];
        nr |= wsn[(int64_t(q) * g.C + c) * g.S + s] != 0;
    }
    nar = __syncthreads_or(nr);
    return block_sum(v);
}

// pass 0: partial sum x;  pass 1: partial sum d*d (d = x - mean);
// pass 2: xhat, y (+ running stats, inv by the s == 0 block).
__global__ void bn_fwd_kernel(int pass, PositFmt f, int fb, const void* x, BnGeom g,
                              const void* gamma, const void* beta, uint32_t eps, int training,
                              PositFmt fo, int ob, void* rm, void* rv, uint32_t mom, void* y,
                              void* xhat, void* inv_out, u128* ws, uint8_t* wsn) {
    const int s = blockIdx.x, c = blockIdx.y;
    const int e0 = s * g.chunk, e1 = min(g.M, e0 + g.chunk);
    __shared__ uint32_t sh_mean, sh_inv;
    const uint32_t Mc = p_from_int64(f, g.M);
    if (pass == 0) {
        u128 acc = 0;
        bool nar = false;
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x)
            q_add(acc, nar, f, load_any(x, bn_index(g, c, e), fb));
        nar = __syncthreads_or(nar);
        const u128 t = block_sum(acc);
        if (threadIdx.x == 0) {
            ws[(0 * g.C + c) * g.S + s] = t;
            wsn[(0 * g.C + c) * g.S + s] = nar;
        }
        return;
    }
    // mean (batch or running)
    if (training) {
        bool nar;
        const u128 t = bn_gather(ws, wsn, 0, g, c, nar);
        if (threadIdx.x == 0) sh_mean = p_div(f, q_round(f, t, nar), Mc);
    } else if (threadIdx.x == 0) {
        sh_mean = p_convert(fo, f, load_any(rm, c, ob));
    }
    __syncthreads();
    const uint32_t mean = sh_mean;
    if (pass == 1) {
        u128 acc = 0;
        bool nar = false;
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            const uint32_t d = p_sub(f, load_any(x, bn_index(g, c, e), fb), mean);
            q_fma(acc, nar, f, d, d);
        }
        nar = __syncthreads_or(nar);
        const u128 t = block_sum(acc);
        if (threadIdx.x == 0) {
            ws[(1 * g.C + c) * g.S + s] = t;
            wsn[(1 * g.C + c) * g.S + s] = nar;
        }
        return;
    }
    // pass 2
    uint32_t var = 0;
    if (training) {
        bool nar;
        const u128 t = bn_gather(ws, wsn, 1, g, c, nar);
        if (threadIdx.x == 0) var = p_div(f, q_round(f, t, nar), Mc);
    } else if (threadIdx.x == 0) {
        var = p_convert(fo, f, load_any(rv, c, ob));
    }
    if (threadIdx.x == 0) {
        const uint32_t inv = p_div(f, p_from_int64(f, 1), p_sqrt(f, p_add(f, var, eps)));
        sh_inv = inv;
        if (s == 0) {
            store_any(inv_out, c, fb, inv);
            if (training) {
                const uint32_t m0 = load_any(rm, c, ob), v0 = load_any(rv, c, ob);
                store_any(rm, c, ob,
                          p_add(fo, m0, p_mul(fo, mom, p_sub(fo, p_convert(f, fo, mean), m0))));
                store_any(rv, c, ob,
                          p_add(fo, v0, p_mul(fo, mom, p_sub(fo, p_convert(f, fo, var), v0))));
            }
        }
    }
    __syncthreads();
    const uint32_t inv = sh_inv;
    const uint32_t gm = load_any(gamma, c, fb), bt = load_any(beta, c, fb);
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const int64_t i = bn_index(g, c, e);
        const uint32_t xh = p_mul(f, p_sub(f, load_any(x, i, fb), mean), inv);
        store_any(xhat, i, fb, xh);
        store_any(y, i, fb, p_add(f, p_mul(f, gm, xh), bt));
    }
}

// pass 0: partial quires qg = sum dyg*xhg, qb = sum dyg (gradient format),
//         q1 = sum dxh, q2 = sum dxh*xhb (backward format);
// pass 1: dgamma / dbeta (+ raw words) by the s == 0 block, dx everywhere.
__global__ void bn_bwd_kernel(int pass, PositFmt ff, int fb, const void* xhat, const void* inv,
                              PositFmt bf, int bb, const void* dy, BnGeom g, const void* gamma_b,
                              PositFmt gf, int gb, void* dx, void* dgamma, void* dbeta,
                              u128* raw_g, uint8_t* nar_g, u128* raw_b, uint8_t* nar_b, u128* ws,
                              uint8_t* wsn) {
    const int s = blockIdx.x, c = blockIdx.y;
    const int e0 = s * g.chunk, e1 = min(g.M, e0 + g.chunk);
    const uint32_t gmb = load_any(gamma_b, c, bb);
    if (pass == 0) {
        u128 a[4] = {0, 0, 0, 0};
        bool n[4] = {false, false, false, false};
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            const int64_t i = bn_index(g, c, e);
            const uint32_t d = load_any(dy, i, bb), xh = load_any(xhat, i, fb);
            const uint32_t dyg = p_convert(bf, gf, d);
            q_fma(a[0], n[0], gf, dyg, p_convert(ff, gf, xh));
            q_add(a[1], n[1], gf, dyg);
            const uint32_t dxh = p_mul(bf, d, gmb);
            q_add(a[2], n[2], bf, dxh);
            q_fma(a[3], n[3], bf, dxh, p_convert(ff, bf, xh));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool nr = __syncthreads_or(n[q]);
            const u128 t = block_sum(a[q]);
            if (threadIdx.x == 0) {
                ws[(int64_t(q) * g.C + c) * g.S + s] = t;
                wsn[(int64_t(q) * g.C + c) * g.S + s] = nr;
            }
        }
        return;
    }
    __shared__ uint32_t sh_s1, sh_s2;
    u128 t[4];
    bool nr[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = bn_gather(ws, wsn, q, g, c, nr[q]);
    if (threadIdx.x == 0) {
        const uint32_t Mb = p_from_int64(bf, g.M);
        sh_s1 = p_div(bf, q_round(bf, t[2], nr[2]), Mb);
        sh_s2 = p_div(bf, q_round(bf, t[3], nr[3]), Mb);
        if (s == 0) {
            if (dgamma) store_any(dgamma, c, gb, q_round(gf, t[0], nr[0]));
            if (dbeta) store_any(dbeta, c, gb, q_round(gf, t[1], nr[1]));
            if (raw_g) {
                raw_g[c] = q_word(gf, t[0]);
                nar_g[c] = nr[0];
            }
            if (raw_b) {
                raw_b[c] = q_word(gf, t[1]);
                nar_b[c] = nr[1];
            }
        }
    }
    __syncthreads();
    const uint32_t s1 = sh_s1, s2 = sh_s2;
    const uint32_t ib = p_convert(ff, bf, load_any(inv, c, fb));
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const int64_t i = bn_index(g, c, e);
        const uint32_t xh = p_convert(ff, bf, load_any(xhat, i, fb));
        const uint32_t dxh = p_mul(bf, load_any(dy, i, bb), gmb);
        store_any(dx, i, bb, p_mul(bf, ib, p_sub(bf, p_sub(bf, dxh, s1), p_mul(bf, xh, s2))));
    }
}

// ---- SGD with momentum ----------------------------------------------------------

__global__ void sgd_momentum_kernel(PositFmt fo, int bo, void* master, void* vel, PositFmt fg,
                                    int bg, const void* grad, int64_t n, uint32_t lr, uint32_t mu,
                                    PositFmt f1, int b1, void* copy1, PositFmt f2, int b2,
                                    void* copy2, int grad_scale_log2) {
    GRID_STRIDE(i, n) {
        uint32_t g = p_convert(fg, fo, load_any(grad, i, bg));
        if (grad_scale_log2 != 0) g = p_ldexp(fo, g, -grad_scale_log2);
        const uint32_t v = p_add(fo, p_mul(fo, mu, load_any(vel, i, bo)), g);
        store_any(vel, i, bo, v);
        const uint32_t w = p_sub(fo, load_any(master, i, bo), p_mul(fo, lr, v));
        store_any(master, i, bo, w);
        if (copy1) store_any(copy1, i, b1, p_convert(fo, f1, w));
        if (copy2) store_any(copy2, i, b2, p_convert(fo, f2, w));
    }
}

namespace {

int bn_geom(int64_t N, int64_t C, int64_t HW, BnGeom* g) {
    if (N < 1 || C < 1 || HW < 1 || C > 65535) return set_status(PNN_EINVAL, "batchnorm: bad shape");
    const int64_t M = N * HW;
    if (M >= (int64_t(1) << 31) || N * C * HW >= (int64_t(1) << 40))
        return set_status(PNN_EINVAL, "batchnorm: too many elements per channel");
    int64_t S = (4 * kSms + C - 1) / C;           // ~4 blocks per SM in total
    S = S < (M + 1023) / 1024 ? S : (M + 1023) / 1024;  // >= 1024 elements per block
    if (S > kBnMaxSplit) S = kBnMaxSplit;
    if (S < 1) S = 1;
    g->N = N;
    g->C = C;
    g->HW = HW;
    g->M = int(M);
    g->S = int(S);
    g->chunk = int((M + S - 1) / S);
    return PNN_OK;
}

size_t bn_ws_bytes(int64_t C) { return size_t(C) * kBnMaxSplit * 4 * (sizeof(u128) + 1); }

}  // namespace
}  // namespace pnn_b200

using namespace pnn_b200;

extern "C" {

int pnn_act_fwd(int kind, int nbits, int es, const void* x, void* y, int64_t n, void* stream) {
    if (!elt_ok(nbits, es)) return unsupported("act_fwd");
    if ((kind != 1 && kind != 2) || n < 0 || (n > 0 && (!x || !y)))
        return set_status(PNN_EINVAL, "act_fwd: bad arguments");
    if (n == 0) return PNN_OK;
    act_fwd_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(kind, make_fmt(nbits, es),
                                                                   bytes_of(nbits), x, y, n);
    return launched("act_fwd");
}

int pnn_act_bwd(int kind, int f_nbits, int f_es, const void* y, int b_nbits, int b_es,
                const void* dy, void* dx, int64_t n, void* stream) {
    if (!elt_ok(f_nbits, f_es) || !elt_ok(b_nbits, b_es)) return unsupported("act_bwd");
    if ((kind != 1 && kind != 2) || n < 0 || (n > 0 && (!y || !dy || !dx)))
        return set_status(PNN_EINVAL, "act_bwd: bad arguments");
    if (n == 0) return PNN_OK;
    act_bwd_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
        kind, make_fmt(f_nbits, f_es), bytes_of(f_nbits), y, make_fmt(b_nbits, b_es),
        bytes_of(b_nbits), dy, dx, n);
    return launched("act_bwd");
}

int pnn_dropout(int nbits, int es, const void* x, void* y, int64_t n, uint64_t seed,
                const void* seed_offset, uint32_t thresh, uint32_t scale_code, void* stream) {
    if (!elt_ok(nbits, es)) return unsupported("dropout");
    if (n < 0 || (n > 0 && (!x || !y))) return set_status(PNN_EINVAL, "dropout: bad arguments");
    if (n == 0) return PNN_OK;
    dropout_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
        make_fmt(nbits, es), bytes_of(nbits), x, y, n, seed,
        static_cast<const uint64_t*>(seed_offset), thresh, scale_code);
    return launched("dropout");
}

int pnn_mse(int nbits, int es, const void* y, const void* t, int64_t n, int64_t global_count,
            int grad_scale_log2, void* grad, void* loss_out, void* stream) {
    if (!quire_ok(nbits, es)) return unsupported("mse (quire wider than 128 bits)");
    if (n < 1 || global_count < 1 || !y || !t || !grad)
        return set_status(PNN_EINVAL, "mse: bad arguments");
    mse_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(make_fmt(nbits, es), bytes_of(nbits), y, t, n,
                                                    global_count, grad_scale_log2, grad, loss_out);
    return launched("mse");
}

int pnn_batchnorm_workspace(int64_t C, size_t* bytes) {
    if (C < 1 || !bytes) return set_status(PNN_EINVAL, "batchnorm_workspace: bad arguments");
    *bytes = bn_ws_bytes(C);
    return PNN_OK;
}

int pnn_batchnorm_fwd(int f_nbits, int f_es, const void* x, int64_t N, int64_t C, int64_t HW,
                      const void* gamma, const void* beta, uint32_t eps_code, int training,
                      int o_nbits, int o_es, void* run_mean, void* run_var, uint32_t mom_code,
                      void* y, void* xhat, void* inv, void* workspace, size_t workspace_bytes,
                      void* stream) {
    if (!quire_ok(f_nbits, f_es) || !elt_ok(o_nbits, o_es)) return unsupported("batchnorm_fwd");
    BnGeom g;
    if (int rc = bn_geom(N, C, HW, &g)) return rc;
    if (!x || !gamma || !beta || !run_mean || !run_var || !y || !xhat || !inv)
        return set_status(PNN_EINVAL, "batchnorm_fwd: bad arguments");
    if (training && (!workspace || workspace_bytes < bn_ws_bytes(C)))
        return set_status(PNN_EWORKSPACE, "batchnorm_fwd: workspace too small");
    u128* ws = static_cast<u128*>(workspace);
    uint8_t* wsn = reinterpret_cast<uint8_t*>(ws + size_t(C) * kBnMaxSplit * 4);
    const PositFmt f = make_fmt(f_nbits, f_es), fo = make_fmt(o_nbits, o_es);
    const dim3 grid(g.S, unsigned(C));
    auto st = (cudaStream_t)stream;
    for (int pass = training ? 0 : 2; pass < 3; ++pass)
        bn_fwd_kernel<<<grid, 256, 0, st>>>(pass, f, bytes_of(f_nbits), x, g, gamma, beta, eps_code,
                                            training, fo, bytes_of(o_nbits), run_mean, run_var,
                                            mom_code, y, xhat, inv, ws, wsn);
    return launched("batchnorm_fwd");
}

int pnn_batchnorm_bwd(int f_nbits, int f_es, const void* xhat, const void* inv, int b_nbits,
                      int b_es, const void* dy, int64_t N, int64_t C, int64_t HW,
                      const void* gamma_b, int g_nbits, int g_es, void* dx, void* dgamma,
                      void* dbeta, void* dgamma_raw, void* dgamma_nar, void* dbeta_raw,
                      void* dbeta_nar, void* workspace, size_t workspace_bytes, void* stream) {
    if (!elt_ok(f_nbits, f_es) || !quire_ok(b_nbits, b_es) || !quire_ok(g_nbits, g_es))
        return unsupported("batchnorm_bwd");
    BnGeom g;
    if (int rc = bn_geom(N, C, HW, &g)) return rc;
    if (!xhat || !inv || !dy || !gamma_b || !dx || (dgamma_raw && !dgamma_nar) ||
        (dbeta_raw && !dbeta_nar))
        return set_status(PNN_EINVAL, "batchnorm_bwd: bad arguments");
    if (!workspace || workspace_bytes < bn_ws_bytes(C))
        return set_status(PNN_EWORKSPACE, "batchnorm_bwd: workspace too small");
    u128* ws = static_cast<u128*>(workspace);
    uint8_t* wsn = reinterpret_cast<uint8_t*>(ws + size_t(C) * kBnMaxSplit * 4);
    const dim3 grid(g.S, unsigned(C));
    auto st = (cudaStream_t)stream;
    for (int pass = 0; pass < 2; ++pass)
        bn_bwd_kernel<<<grid, 256, 0, st>>>(
            pass, make_fmt(f_nbits, f_es), bytes_of(f_nbits), xhat, inv, make_fmt(b_nbits, b_es),
            bytes_of(b_nbits), dy, g, gamma_b, make_fmt(g_nbits, g_es), bytes_of(g_nbits), dx,
            dgamma, dbeta, static_cast<u128*>(dgamma_raw), static_cast<uint8_t*>(dgamma_nar),
            static_cast<u128*>(dbeta_raw), static_cast<uint8_t*>(dbeta_nar), ws, wsn);
    return launched("batchnorm_bwd");
}

int pnn_sgd_step_momentum(int opt_nbits, int opt_es, void* master, void* velocity, int g_nbits,
                          int g_es, const void* grad, int64_t n, uint32_t lr_code,
                          uint32_t mu_code, int c1_nbits, int c1_es, void* copy1, int c2_nbits,
                          int c2_es, void* copy2, int grad_scale_log2, void* stream) {
    if (!elt_ok(opt_nbits, opt_es) || !elt_ok(g_nbits, g_es) ||
        (copy1 && !elt_ok(c1_nbits, c1_es)) || (copy2 && !elt_ok(c2_nbits, c2_es)))
        return unsupported("sgd_step_momentum");
    if (n < 0 || (n > 0 && (!master || !velocity || !grad)))
        return set_status(PNN_EINVAL, "sgd_step_momentum: bad arguments");
    if (n == 0) return PNN_OK;
    const PositFmt fo = make_fmt(opt_nbits, opt_es);
    const PositFmt f1 = copy1 ? make_fmt(c1_nbits, c1_es) : fo;
    const PositFmt f2 = copy2 ? make_fmt(c2_nbits, c2_es) : fo;
    sgd_momentum_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
        fo, bytes_of(opt_nbits), master, velocity, make_fmt(g_nbits, g_es), bytes_of(g_nbits), grad,
        n, lr_code, mu_code, f1, bytes_of(f1.nbits), copy1, f2, bytes_of(f2.nbits), copy2,
        grad_scale_log2);
    return launched("sgd_step_momentum");
}

}  // extern "C"
