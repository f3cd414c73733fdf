// Elementwise / small kernels of the training step (HBM-roofline kernels):
// stage conversion, ReLU, max-pool, softmax cross-entropy, SGD update.
//
//   convert_tensor       proj/src/tensor_ops.cpp:807-821
//   maxpool2d (+bwd)     tensor_ops.cpp:620-656, 658-670 (first strict max; the
//                        backward accumulates with scalar add in output order)
//   ReLU / CE / SGD      no reference code (layers are placeholders, SURVEY.md
//                        §0.3); semantics pinned in SURVEY.md Appendix A.2/A.5/A.7
//                        and mirrored by the CPU oracle step (oracle/step.py)
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/pnn_b200.h"
#include "eltwise_common.cuh"
#include "epilogue.cuh"
#include "posit_scalar.cuh"
#include "pdl.cuh"
#include "status.h"
#include "tables.h"

namespace pnn_b200 {

__global__ void convert_kernel(PositFmt s, int sb, const void* src, PositFmt d, int db, void* dst,
                               int64_t n) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(i, n) { store_any(dst, i, db, p_convert(s, d, load_any(src, i, sb))); }
}

// ReLU: x > 0 ? x : 0 by signed-pattern compare (NaR sorts lowest -> 0).
__global__ void relu_fwd_kernel(PositFmt f, int b, const void* x, void* y, int64_t n) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(i, n) {
        const uint32_t c = load_any(x, i, b);
        store_any(y, i, b, p_compare(f, c, 0) > 0 ? c : 0u);
    }
}

// dx = x > 0 ? dy : 0 (x in the forward format, dy/dx in the backward format).
__global__ void relu_bwd_kernel(PositFmt fx, int bx, const void* x, int bg, const void* dy,
                                void* dx, int64_t n) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(i, n) {
        const uint32_t c = load_any(x, i, bx);
        store_any(dx, i, bg, p_compare(fx, c, 0) > 0 ? load_any(dy, i, bg) : 0u);
    }
}

__global__ void maxpool_fwd_kernel(PositFmt f, int b, const void* x, int64_t NC, int64_t H,
                                   int64_t W, int k, int s, int64_t OH, int64_t OW, void* y,
                                   int64_t* argmax) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(o, NC * OH * OW) {
        const int64_t ox = o % OW, oy = (o / OW) % OH, nc = o / (OW * OH);
        const int64_t base = nc * H * W;
        int64_t best = base + (oy * s) * W + ox * s;
        uint32_t bv = load_any(x, best, b);
        for (int ky = 0; ky < k; ++ky)
            for (int kx = 0; kx < k; ++kx) {
                const int64_t idx = base + (oy * s + ky) * W + ox * s + kx;
                const uint32_t v = load_any(x, idx, b);
                if (p_compare(f, v, bv) > 0) {
                    best = idx;
                    bv = v;
                }
            }
        store_any(y, o, b, bv);
        argmax[o] = best;
    }
}

// dx[t] = add(...add(add(0, dy[i1]), dy[i2])...) over outputs i with
// argmax[i] == t in increasing i -- the reference's sequential order.
__global__ void maxpool_bwd_kernel(PositFmt f, int b, const void* dy, const int64_t* argmax,
                                   int64_t NC, int64_t H, int64_t W, int k, int s, int64_t OH,
                                   int64_t OW, void* dx) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(t, NC * H * W) {
        const int64_t ix = t % W, iy = (t / W) % H, nc = t / (W * H);
        const int64_t oy0 = iy - k + 1 > 0 ? (iy - k + 1 + s - 1) / s : 0;
        const int64_t ox0 = ix - k + 1 > 0 ? (ix - k + 1 + s - 1) / s : 0;
        const int64_t oy1 = min(OH - 1, iy / s), ox1 = min(OW - 1, ix / s);
        uint32_t acc = 0;
        for (int64_t oy = oy0; oy <= oy1; ++oy)
            for (int64_t ox = ox0; ox <= ox1; ++ox) {
                const int64_t o = (nc * OH + oy) * OW + ox;
                if (argmax[o] == t) {  // add(0, v) == v exactly (NaR included)
                    const uint32_t v = load_any(dy, o, b);
                    acc = acc == 0 ? v : p_add(f, acc, v);
                }
            }
        store_any(dx, t, b, acc);
    }
}

// Exactly tiled pooling (k == stride, H = OH*k, W = OW*k): each input lies in
// exactly one window, so a thread per window writes its k x k inputs (argmax
// position gets dy, the rest 0 -- the same values as the general kernel).
// 32-bit index math (the callers check the sizes).
__global__ void maxpool_bwd_tiled_kernel(int b, const void* dy, const int64_t* argmax, int NC,
                                         int OH, int OW, int k, void* dx) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const int W = OW * k, H = OH * k;
    const int total = NC * OH * OW;
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
        const int ox = o % OW, t = o / OW, oy = t % OH, nc = t / OH;
        const int64_t base = (int64_t(nc) * H + oy * k) * W + ox * k;
        const int64_t am = argmax[o];
        const uint32_t v = load_any(dy, o, b);
        for (int ky = 0; ky < k; ++ky)
            for (int kx = 0; kx < k; ++kx) {
                const int64_t idx = base + int64_t(ky) * W + kx;
                store_any(dx, idx, b, idx == am ? v : 0u);
            }
    }
}

__global__ void maxpool_fwd_tiled_kernel(PositFmt f, int b, const void* x, int NC, int OH, int OW,
                                         int k, void* y, int64_t* argmax) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const int W = OW * k, H = OH * k;
    const int total = NC * OH * OW;
    for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
        const int ox = o % OW, t = o / OW, oy = t % OH, nc = t / OH;
        const int64_t base = (int64_t(nc) * H + oy * k) * W + ox * k;
        int64_t best = base;
        uint32_t bv = load_any(x, best, b);
        for (int ky = 0; ky < k; ++ky)
            for (int kx = 0; kx < k; ++kx) {
                const int64_t idx = base + int64_t(ky) * W + kx;
                const uint32_t v = load_any(x, idx, b);
                if (p_compare(f, v, bv) > 0) {
                    best = idx;
                    bv = v;
                }
            }
        store_any(y, o, b, bv);
        argmax[o] = best;
    }
}

// ---- 2x2 / stride-2 pooling, 16-byte vectors (the training step's layers) ----
// Posit order is the order of the sign-extended patterns (NaR lowest,
// posit.cpp:514-520), so the first-strict-max of a window (row-major window
// order, tensor_ops.cpp:620-656) is a signed integer compare.  A thread covers
// WPT = 16 / sizeof(TX) / 2 adjacent windows of one output row: two 16-byte x
// loads (the window's two input rows).

template <typename TX>
__device__ __forceinline__ void load_codes16(const TX* p, uint32_t (&c)[16 / sizeof(TX)]) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < int(16 / sizeof(TX)); ++j)
        c[j] = sizeof(TX) == 1 ? (w[j >> 2] >> (8 * (j & 3))) & 0xFFu : (w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
}

__device__ __forceinline__ uint4 pack16_u8(const uint32_t* c) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
        w[q] = (c[4 * q] & 0xFF) | (c[4 * q + 1] & 0xFF) << 8 | (c[4 * q + 2] & 0xFF) << 16 |
               (c[4 * q + 3] & 0xFF) << 24;
    return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ uint4 pack8_u16(const uint32_t* c) {
    return make_uint4((c[0] & 0xFFFF) | c[1] << 16, (c[2] & 0xFFFF) | c[3] << 16,
                      (c[4] & 0xFFFF) | c[5] << 16, (c[6] & 0xFFFF) | c[7] << 16);
}

// window index (0..3, row-major) of the first strict maximum
__device__ __forceinline__ int argmax4(int32_t a, int32_t b, int32_t c, int32_t d) {
    int i = 0;
    int32_t m = a;
    if (b > m) { m = b; i = 1; }
    if (c > m) { m = c; i = 2; }
    if (d > m) { i = 3; }
    return i;
}

template <typename TX>
__global__ void __launch_bounds__(256) maxpool2_fwd_vec_kernel(int nbits, const TX* __restrict__ x,
                                                               TX* __restrict__ y, int rows, int OW) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    constexpr int VE = 16 / sizeof(TX), WPT = VE / 2;
    const int W = 2 * OW, vpr = OW / WPT;  // vectors per output row
    const int total = rows * vpr;          // rows = N * C * OH
    const int sh = 32 - nbits;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int r = i / vpr, v = i - r * vpr;
        const TX* p0 = x + (int64_t(r) * 2) * W + v * VE;
        uint32_t a[VE], b[VE];
        load_codes16<TX>(p0, a);
        load_codes16<TX>(p0 + W, b);
        uint32_t out[WPT];
#pragma unroll
        for (int j = 0; j < WPT; ++j) {
            const uint32_t c[4] = {a[2 * j], a[2 * j + 1], b[2 * j], b[2 * j + 1]};
            const int k = argmax4(int32_t(c[0] << sh), int32_t(c[1] << sh), int32_t(c[2] << sh),
                                  int32_t(c[3] << sh));
            out[j] = c[k];
        }
        TX* q = y + int64_t(r) * OW + v * WPT;
        if constexpr (sizeof(TX) == 1) {
            *reinterpret_cast<uint2*>(q) = make_uint2(out[0] | out[1] << 8 | out[2] << 16 | out[3] << 24,
                                                      out[4] | out[5] << 8 | out[6] << 16 | out[7] << 24);
        } else {
            *reinterpret_cast<uint2*>(q) = make_uint2(out[0] | out[1] << 16, out[2] | out[3] << 16);
        }
    }
}

// dx = maxpool2d_backward(dy, argmax(x)) without a stored argmax: the window's
// first strict max is recomputed from x; dy (format of TG) lands there, zeros
// elsewhere (tiled windows: every input lies in exactly one window).
// relu_gate: also apply the backward of a ReLU whose output x is (x > 0 at the
// argmax, Appendix A.2) -- the ReLU -> MaxPool pair's backward in one pass.
template <typename TX, typename TG>
__global__ void __launch_bounds__(256) maxpool2_bwd_x_kernel(int x_nbits, const TX* __restrict__ x,
                                                             const TG* __restrict__ dy,
                                                             TG* __restrict__ dx, int rows, int OW,
                                                             int relu_gate = 0) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    constexpr int VE = 16 / sizeof(TX), WPT = VE / 2;
    const int W = 2 * OW, vpr = OW / WPT;
    const int total = rows * vpr;
    const int sh = 32 - x_nbits;
    // vector loads of dy when every thread's WPT gradients are aligned
    const bool gvec = (reinterpret_cast<uintptr_t>(dy) % (WPT * sizeof(TG))) == 0 &&
                      (int64_t(OW) * sizeof(TG)) % (WPT * sizeof(TG)) == 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int r = i / vpr, v = i - r * vpr;
        const int64_t in0 = (int64_t(r) * 2) * W + v * VE;
        uint32_t a[VE], b[VE];
        load_codes16<TX>(x + in0, a);
        load_codes16<TX>(x + in0 + W, b);
        uint32_t g[WPT];
        const TG* gp = dy + int64_t(r) * OW + v * WPT;
        if (!gvec) {
#pragma unroll
            for (int j = 0; j < WPT; ++j) g[j] = uint32_t(gp[j]);
        } else if constexpr (WPT * sizeof(TG) == 16 || WPT * sizeof(TG) == 8) {
            // one 16- or 8-byte load of the WPT gradients
            uint32_t gw[4];
            if constexpr (WPT * sizeof(TG) == 16) {
                const uint4 gv = __ldg(reinterpret_cast<const uint4*>(gp));
                gw[0] = gv.x, gw[1] = gv.y, gw[2] = gv.z, gw[3] = gv.w;
            } else {
                const uint2 gv = __ldg(reinterpret_cast<const uint2*>(gp));
                gw[0] = gv.x, gw[1] = gv.y, gw[2] = gw[3] = 0u;
            }
#pragma unroll
            for (int j = 0; j < WPT; ++j)
                g[j] = sizeof(TG) == 2 ? (gw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu
                                       : (gw[j >> 2] >> (8 * (j & 3))) & 0xFFu;
        } else {
#pragma unroll
            for (int j = 0; j < WPT; ++j) g[j] = uint32_t(gp[j]);
        }
        const uint32_t sign = 1u << (x_nbits - 1);
        uint32_t top[16] = {}, bot[16] = {};  // VE used (pack16_u8 reads 16)
#pragma unroll
        for (int j = 0; j < WPT; ++j) {
            const int k = argmax4(int32_t(a[2 * j] << sh), int32_t(a[2 * j + 1] << sh),
                                  int32_t(b[2 * j] << sh), int32_t(b[2 * j + 1] << sh));
            if (relu_gate) {  // the window max is the ReLU output at the argmax
                const uint32_t mx = k == 0 ? a[2 * j] : k == 1 ? a[2 * j + 1] : k == 2 ? b[2 * j] : b[2 * j + 1];
                if (mx == 0 || (mx & sign)) g[j] = 0u;
            }
            top[2 * j] = k == 0 ? g[j] : 0u;
            top[2 * j + 1] = k == 1 ? g[j] : 0u;
            bot[2 * j] = k == 2 ? g[j] : 0u;
            bot[2 * j + 1] = k == 3 ? g[j] : 0u;
        }
        // VE codes of TG per row: 16-byte vector stores (VE * sizeof(TG) bytes)
        TG* o0 = dx + in0;
        TG* o1 = o0 + W;
        if constexpr (sizeof(TG) == 1 && VE == 8) {  // 8 bytes per row
            const uint4 a0 = pack16_u8(top), a1 = pack16_u8(bot);
            *reinterpret_cast<uint2*>(o0) = make_uint2(a0.x, a0.y);
            *reinterpret_cast<uint2*>(o1) = make_uint2(a1.x, a1.y);
        } else if constexpr (sizeof(TG) == 1) {
            *reinterpret_cast<uint4*>(o0) = pack16_u8(top);
            *reinterpret_cast<uint4*>(o1) = pack16_u8(bot);
        } else {
#pragma unroll
            for (int h = 0; h < VE / 8; ++h) {
                reinterpret_cast<uint4*>(o0)[h] = pack8_u16(top + 8 * h);
                reinterpret_cast<uint4*>(o1)[h] = pack8_u16(bot + 8 * h);
            }
        }
    }
}

// ---- vectorised elementwise paths (16-byte accesses, 8 codes per thread-step)

template <typename T>
struct Vec8;  // 8 codes
template <>
struct Vec8<uint8_t> {
    using V = uint2;
};
template <>
struct Vec8<uint16_t> {
    using V = uint4;
};

template <typename T>
__device__ __forceinline__ void unpack8(const typename Vec8<T>::V& v, uint32_t (&c)[8]) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
#pragma unroll
    for (int j = 0; j < 8; ++j)
        c[j] = sizeof(T) == 1 ? (w[j >> 2] >> (8 * (j & 3))) & 0xFFu : (w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
}

template <typename T>
__device__ __forceinline__ typename Vec8<T>::V pack8(const uint32_t (&c)[8]) {
    typename Vec8<T>::V v;
    uint32_t* w = reinterpret_cast<uint32_t*>(&v);
    if constexpr (sizeof(T) == 1) {
        w[0] = (c[0] & 0xFF) | ((c[1] & 0xFF) << 8) | ((c[2] & 0xFF) << 16) | ((c[3] & 0xFF) << 24);
        w[1] = (c[4] & 0xFF) | ((c[5] & 0xFF) << 8) | ((c[6] & 0xFF) << 16) | ((c[7] & 0xFF) << 24);
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) w[j] = (c[2 * j] & 0xFFFF) | ((c[2 * j + 1] & 0xFFFF) << 16);
    }
    return v;
}

__device__ __forceinline__ bool positive_code(uint32_t c, int nbits) {
    return c != 0 && ((c >> (nbits - 1)) & 1u) == 0;
}

// stage conversion; formats up to 12 bits convert through a per-block table
// (persistent grid: building it costs 1 << nbits conversions per block)
template <typename S, typename Dt>
__global__ void __launch_bounds__(256) convert_vec_kernel(PositFmt s, const S* __restrict__ src,
                                                          PositFmt d, Dt* __restrict__ dst,
                                                          int64_t n) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    __shared__ uint16_t lut[1 << 12];
    const bool use_lut = s.nbits <= 12;
    if (use_lut) {
        for (int c = threadIdx.x; c < (1 << s.nbits); c += blockDim.x) lut[c] = uint16_t(p_convert(s, d, uint32_t(c)));
        __syncthreads();
    }
    const int64_t n8 = n / 8;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8;
         i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t c[8];
        unpack8<S>(reinterpret_cast<const typename Vec8<S>::V*>(src)[i], c);
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = use_lut ? uint32_t(lut[c[j]]) : p_convert(s, d, c[j]);
        reinterpret_cast<typename Vec8<Dt>::V*>(dst)[i] = pack8<Dt>(c);
    }
    for (int64_t i = n8 * 8 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = Dt(use_lut ? uint32_t(lut[uint32_t(src[i])]) : p_convert(s, d, uint32_t(src[i])));
}

template <typename T>
__global__ void relu_fwd_vec_kernel(int nbits, const T* __restrict__ x, T* __restrict__ y, int64_t n) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const int64_t n8 = n / 8;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8;
         i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t c[8];
        unpack8<T>(reinterpret_cast<const typename Vec8<T>::V*>(x)[i], c);
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = positive_code(c[j], nbits) ? c[j] : 0u;
        reinterpret_cast<typename Vec8<T>::V*>(y)[i] = pack8<T>(c);
    }
    for (int64_t i = n8 * 8 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        y[i] = positive_code(uint32_t(x[i]), nbits) ? x[i] : T(0);
}

template <typename TX, typename TG>
__global__ void relu_bwd_vec_kernel(int x_nbits, const TX* __restrict__ x,
                                    const TG* __restrict__ dy, TG* __restrict__ dx, int64_t n) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const int64_t n8 = n / 8;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8;
         i += int64_t(gridDim.x) * blockDim.x) {
        uint32_t cx[8], g[8];
        unpack8<TX>(reinterpret_cast<const typename Vec8<TX>::V*>(x)[i], cx);
        unpack8<TG>(reinterpret_cast<const typename Vec8<TG>::V*>(dy)[i], g);
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = positive_code(cx[j], x_nbits) ? g[j] : 0u;
        reinterpret_cast<typename Vec8<TG>::V*>(dx)[i] = pack8<TG>(g);
    }
    for (int64_t i = n8 * 8 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        dx[i] = positive_code(uint32_t(x[i]), x_nbits) ? dy[i] : TG(0);
}

// Softmax cross-entropy in the loss format:
//   m = max z;  e_j = exp(z_j - m);  S = round(quire sum e_j);
// p_j = e_j / S;  loss_i = log(S) - (z_y - m);
// dlogits_j = ldexp(p_j - [j==y], -log2_batch).
// One warp per row, lanes over classes: the max (a total order on codes, so
// any reduction order gives the same value), the exact integer sum of e_j
// (butterfly over 128-bit lanes), one rounding, then p_j per lane.
__global__ void softmax_xent_kernel(PositFmt f, int b, const void* logits, const int32_t* labels,
                                    int64_t B, int64_t Cn, int log2_batch, int grad_scale_log2,
                                    void* dlogits, void* loss_rows, void* s_rows = nullptr,
                                    const uint16_t* __restrict__ exp_lut = nullptr,
                                    const uint16_t* __restrict__ log_lut = nullptr) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    auto pexp = [&](uint32_t x) { return exp_lut ? uint32_t(__ldg(exp_lut + x)) : p_exp(f, x); };
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; i < B; i += nwarps) {
        const int64_t row = i * Cn;
        uint32_t m = load_any(logits, row, b);
        for (int64_t j = lane; j < Cn; j += 32) {
            const uint32_t v = load_any(logits, row + j, b);
            if (p_compare(f, v, m) > 0) m = v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint32_t v = __shfl_xor_sync(0xFFFFFFFFu, m, o);
            if (p_compare(f, v, m) > 0) m = v;
        }
        // S = quire sum of e_j: exact in the integer image, one rounding
        uint64_t lo = 0, hi = 0;
        bool nar = false;
        uint32_t e0 = 0;  // this lane's first e_j, reused below
        for (int64_t j = lane; j < Cn; j += 32) {
            const uint32_t e = pexp(p_sub(f, load_any(logits, row + j, b), m));
            if (j == lane) e0 = e;
            __int128 X;
            nar |= decode_x128(e, f, X);
            const unsigned __int128 s = ((unsigned __int128)hi << 64 | lo) + (unsigned __int128)X;
            lo = uint64_t(s);
            hi = uint64_t(s >> 64);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t l2 = __shfl_xor_sync(0xFFFFFFFFu, lo, o);
            const uint64_t h2 = __shfl_xor_sync(0xFFFFFFFFu, hi, o);
            const unsigned __int128 s = ((unsigned __int128)hi << 64 | lo) + ((unsigned __int128)h2 << 64 | l2);
            lo = uint64_t(s);
            hi = uint64_t(s >> 64);
        }
        nar = __any_sync(0xFFFFFFFFu, nar);
        const __int128 sx = (__int128)((unsigned __int128)hi << 64 | lo);
        uint32_t S;
        if (nar) {
            S = nar_of(f);
        } else {
            const bool neg = sx < 0;
            S = round_mag128(f, neg, (unsigned __int128)(neg ? -sx : sx), -f.R);
        }
        const int32_t y = labels[i];
        const uint32_t one = p_from_int64(f, 1);
        for (int64_t j = lane; j < Cn; j += 32) {
            const uint32_t e = j == lane ? e0 : pexp(p_sub(f, load_any(logits, row + j, b), m));
            const uint32_t pj = p_div(f, e, S);
            const uint32_t g = p_sub(f, pj, j == y ? one : 0u);
            store_any(dlogits, row + j, b, p_ldexp(f, g, grad_scale_log2 - log2_batch));
        }
        if (lane == 0 && s_rows != nullptr) store_any(s_rows, i, b, S);
        if (lane == 0 && loss_rows != nullptr) {
            const uint32_t zy = load_any(logits, row + y, b);
            store_any(loss_rows, i, b, p_sub(f, log_lut ? uint32_t(__ldg(log_lut + S)) : p_log(f, S), p_sub(f, zy, m)));
        }
    }
}

// loss_i = log(S_i) - (z_y - m) from the row sums S the gradient kernel left
// (same operations as softmax_xent_kernel's last step, Appendix A.5): lets the
// loss run beside the backward pass instead of on its critical path.
__global__ void xent_loss_rows_kernel(PositFmt f, int b, const void* logits, const int32_t* labels,
                                      const void* s_rows, int64_t B, int64_t Cn, void* loss_rows,
                                      const uint16_t* __restrict__ log_lut = nullptr) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(i, B) {
        const int64_t row = i * Cn;
        uint32_t m = load_any(logits, row, b);
        for (int64_t j = 1; j < Cn; ++j) {
            const uint32_t v = load_any(logits, row + j, b);
            if (p_compare(f, v, m) > 0) m = v;
        }
        const uint32_t zy = load_any(logits, row + labels[i], b);
        const uint32_t Sv = load_any(s_rows, i, b);
        store_any(loss_rows, i, b, p_sub(f, log_lut ? uint32_t(__ldg(log_lut + Sv)) : p_log(f, Sv), p_sub(f, zy, m)));
    }
}

// Batch loss: quire sum of loss_i (optionally returned as a raw W-bit word
// for the data-parallel reduction), rounded once, then ldexp by -log2_batch.
__global__ void loss_reduce_kernel(PositFmt f, int b, const void* loss_rows, int64_t B,
                                   int log2_batch, void* loss_out, unsigned __int128* raw_word,
                                   uint8_t* raw_nar) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    __shared__ unsigned long long lo_s[256], hi_s[256];
    __shared__ int nar_s;
    if (threadIdx.x == 0) nar_s = 0;
    __syncthreads();
    __int128 acc = 0;
    for (int64_t i = threadIdx.x; i < B; i += blockDim.x) {
        __int128 X;
        if (decode_x128(load_any(loss_rows, i, b), f, X)) nar_s = 1;
        acc += X;
    }
    lo_s[threadIdx.x] = (unsigned long long)uint64_t(acc);
    hi_s[threadIdx.x] = (unsigned long long)uint64_t((unsigned __int128)acc >> 64);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned __int128 s = 0;
        for (int t = 0; t < blockDim.x; ++t)
            s += (unsigned __int128)lo_s[t] | ((unsigned __int128)hi_s[t] << 64);
        if (raw_word) {  // W <= 128 (host-checked)
            const unsigned __int128 one = 1;
            const unsigned __int128 wmask = f.W >= 128 ? ~(unsigned __int128)0 : ((one << f.W) - 1);
            *raw_word = (s << f.R) & wmask;
            *raw_nar = nar_s ? 1 : 0;
        }
        if (loss_out) {
            // the same exact sum rounded once, from the image (LSB 2^-R)
            const __int128 sx = (__int128)s;
            const bool neg = sx < 0;
            const uint32_t c =
                nar_s ? nar_of(f)
                      : (sx == 0 ? 0u
                                 : round_mag128(f, neg, (unsigned __int128)(neg ? -sx : sx), -f.R));
            store_any(loss_out, 0, b, p_ldexp(f, c, -log2_batch));
        }
    }
}

// SGD: w = sub(w, mul(lr, convert(g -> p_opt))) in
// the optimizer format, then refresh the stage copies (convert, SPEC §3.3).
__global__ void sgd_kernel(PositFmt fo, int bo, void* master, PositFmt fg, int bg, const void* grad,
                           int64_t n, uint32_t lr, PositFmt f1, int b1, void* copy1, PositFmt f2,
                           int b2, void* copy2, int grad_scale_log2) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(i, n) {
        uint32_t g = p_convert(fg, fo, load_any(grad, i, bg));
        if (grad_scale_log2 != 0) g = p_ldexp(fo, g, -grad_scale_log2);  // loss-scale undo
        const uint32_t w = p_sub(fo, load_any(master, i, bo), p_mul(fo, lr, g));
        store_any(master, i, bo, w);
        if (copy1) store_any(copy1, i, b1, p_convert(fo, f1, w));
        if (copy2) store_any(copy2, i, b2, p_convert(fo, f2, w));
    }
}

// The optimizer step of a whole model in one launch: segments = parameter
// tensors (same formats), a grid-stride loop over their concatenation, the
// segment found by binary search in the prefix table (kernel parameter, so the
// launch needs no host->device copy and is CUDA-graph capturable).
constexpr int kSgdMaxSeg = 48;
struct SgdSegs {
    int count;
    int64_t start[kSgdMaxSeg + 1];  // prefix offsets
    void* master[kSgdMaxSeg];
    const void* grad[kSgdMaxSeg];
    void* copy1[kSgdMaxSeg];
    void* copy2[kSgdMaxSeg];
};

// The SGD update on integer images (exact), each rounding by the quire
// rounding table -- the same correctly rounded results as the scalar ops
// p_convert, p_mul, p_sub (posit arithmetic rounds the exact value once, like
// the quire's to_posit): g' = round_o(X_g 2^-R_g), m = round_o(lr g'),
// w' = round_o(w - m).  Valid when every image fits 64 bits and every exact
// intermediate its quire word (sgd_fast_ok).
__device__ __forceinline__ uint32_t sgd_fast(const PositFmt& fo, const PositFmt& fg, int64_t X_lr,
                                             uint32_t w, uint32_t gcode, const uint4* lut) {
    int64_t Xg, Xw;
    const bool gnar = decode_x(gcode, fg, Xg);
    const bool wnar = decode_x(w, fo, Xw);
    if (gnar || wnar) return 1u << (fo.nbits - 1);
    const unsigned __int128 qg = (unsigned __int128)((__int128)Xg << (2 * fo.R - fg.R));
    int64_t Xg16;
    decode_x(q_to_posit_lut(fo, qg, lut), fo, Xg16);
    int64_t Xm;
    decode_x(q_to_posit_lut(fo, (unsigned __int128)((__int128)X_lr * Xg16), lut), fo, Xm);
    return q_to_posit_lut(fo, (unsigned __int128)((__int128)(Xw - Xm) << fo.R), lut);
}

// Stage copy of an optimizer-format value by its integer image: round
// X_w 2^-R_o into format fc -- X shifted to fc's quire units, bits shifted out
// jammed into the LSB (they lie below every rounding position, or the value
// is below minpos and rounds to +-minpos either way), then the quire rounding
// (= p_convert, a correctly rounded conversion).
__device__ __forceinline__ uint32_t copy_fast(const PositFmt& fo, const PositFmt& fc, uint32_t w, int64_t Xw,
                                              const uint4* lut) {
    if (w == (1u << (fo.nbits - 1))) return 1u << (fc.nbits - 1);
    const int sh = 2 * fc.R - fo.R;
    __int128 q;
    if (sh >= 0) {
        q = (__int128)Xw << sh;
    } else {
        const int64_t a = Xw < 0 ? -Xw : Xw;
        const int64_t m = (a >> -sh) | ((a & ((int64_t(1) << -sh) - 1)) != 0 ? 1 : 0);
        q = Xw < 0 ? -(__int128)m : (__int128)m;
    }
    // (the 128-bit rounding takes W > 64; narrower words hold the value in 64 bits)
    return fc.W <= 64 ? q_to_posit_lut(fc, uint64_t(int64_t(q)), lut)
                      : q_to_posit_lut(fc, (unsigned __int128)q, lut);
}

__global__ void sgd_multi_kernel(PositFmt fo, int bo, PositFmt fg, int bg, uint32_t lr, PositFmt f1,
                                 int b1, PositFmt f2, int b2, int grad_scale_log2,
                                 const __grid_constant__ SgdSegs segs, int fast) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    __shared__ uint4 s_lut[kPackLutEntries], s_lut1[kPackLutEntries], s_lut2[kPackLutEntries];
    int64_t X_lr = 0;
    if (fast) {
        build_pack_lut(fo, s_lut, threadIdx.x, blockDim.x);
        if (fast & 2) build_pack_lut(f1, s_lut1, threadIdx.x, blockDim.x);
        if (fast & 4) build_pack_lut(f2, s_lut2, threadIdx.x, blockDim.x);
        decode_x(lr, fo, X_lr);
        __syncthreads();
    }
    // the segment table in shared memory: lane-divergent indexing of the kernel
    // parameter space would serialise on the constant cache
    __shared__ int64_t s_start[kSgdMaxSeg + 1];
    __shared__ const void* s_ptr[4][kSgdMaxSeg];
    for (int t = threadIdx.x; t <= segs.count; t += blockDim.x) s_start[t] = segs.start[t];
    for (int t = threadIdx.x; t < segs.count; t += blockDim.x) {
        s_ptr[0][t] = segs.master[t];
        s_ptr[1][t] = segs.grad[t];
        s_ptr[2][t] = segs.copy1[t];
        s_ptr[3][t] = segs.copy2[t];
    }
    __syncthreads();
    const int64_t total = s_start[segs.count];
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        int lo = 0, hi = segs.count - 1;  // last segment with start <= i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_start[mid] <= i) lo = mid;
            else hi = mid - 1;
        }
        const int64_t k = i - s_start[lo];
        void* const master = const_cast<void*>(s_ptr[0][lo]);
        const void* const grad = s_ptr[1][lo];
        void* const copy1 = const_cast<void*>(s_ptr[2][lo]);
        void* const copy2 = const_cast<void*>(s_ptr[3][lo]);
        uint32_t w;
        if (fast) {
            w = sgd_fast(fo, fg, X_lr, load_any(master, k, bo), load_any(grad, k, bg), s_lut);
        } else {
            uint32_t g = p_convert(fg, fo, load_any(grad, k, bg));
            if (grad_scale_log2 != 0) g = p_ldexp(fo, g, -grad_scale_log2);
            w = p_sub(fo, load_any(master, k, bo), p_mul(fo, lr, g));
        }
        store_any(master, k, bo, w);
        int64_t Xw = 0;
        if (fast & 6) decode_x(w, fo, Xw);
        if (copy1)
            store_any(copy1, k, b1, (fast & 2) ? copy_fast(fo, f1, w, Xw, s_lut1) : p_convert(fo, f1, w));
        if (copy2)
            store_any(copy2, k, b2, (fast & 4) ? copy_fast(fo, f2, w, Xw, s_lut2) : p_convert(fo, f2, w));
    }
}

// ---- SGD through per-format tables (the optimizer step's rounding work is
// per element ALU-bound, not HBM-bound: a table per format pair replaces the
// two code-only operations and leaves one exact subtraction + one rounding):
//   xm_lut[g] = X(p_mul(fo, lr, p_convert(fg, fo, g)))  (lr fixed per call;
//               the integer image of m, INT64_MIN for NaR)
//   c_lut[w]  = p_convert(fo, fc, w)                     (stage copies)
//   w' = p_sub(fo, w, m) = round_o(X_w - X_m), the exact difference of the
//   integer images (|X| <= 2^2R, 2R + 1 <= 63) rounded once (posit.cpp:437-457
//   rounds the exact result of every op once; x_to_posit_lut = pack_round).
// Each table entry is computed by the scalar ops themselves, so the path is
// the sgd_kernel arithmetic, entry for entry.
__global__ void sgd_xm_lut_kernel(PositFmt fo, PositFmt fg, uint32_t lr, int64_t* __restrict__ lut) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(c, int64_t(1) << fg.nbits) {
        int64_t X;
        const bool nar = decode_x(p_mul(fo, lr, p_convert(fg, fo, uint32_t(c))), fo, X);
        lut[c] = nar ? INT64_MIN : X;
    }
}
__global__ void copy_lut_kernel(PositFmt fo, PositFmt fc, uint16_t* __restrict__ lut) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(c, int64_t(1) << fo.nbits) { lut[c] = uint16_t(p_convert(fo, fc, uint32_t(c))); }
}
// exp / log of every code (posit_math.cpp:67-107 through p_exp / p_log): the
// softmax cross-entropy's transcendental steps by table
__global__ void fn_lut_kernel(PositFmt f, int which, uint16_t* __restrict__ lut) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(c, int64_t(1) << f.nbits) {
        lut[c] = uint16_t(which == 0 ? p_exp(f, uint32_t(c)) : p_log(f, uint32_t(c)));
    }
}

// round(X 2^-R) for an int64 integer image (|X| < 2^63) through the rounding table
__device__ __forceinline__ uint32_t x_to_posit_lut(const PositFmt& f, int64_t X, const uint4* lut) {
    uint32_t lo = uint32_t(uint64_t(X)), hi = uint32_t(uint64_t(X) >> 32);
    const uint32_t s = uint32_t(int32_t(hi) >> 31);
    uint32_t ml = lo ^ s, mh = hi ^ s;
    asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(ml), "+r"(mh) : "r"(s & 1u));
    const bool hz = mh == 0;
    const int lzh = __clz(mh), lzl = __clz(ml);
    const uint32_t sig = hz ? (ml << (lzl & 31)) : __funnelshift_l(ml, mh, lzh);
    const bool sticky = !hz && (ml << (lzh & 31)) != 0;
    const int top = hz ? 31 - lzl : 63 - lzh;
    const uint32_t c = pack_lut(f, lut, top - f.R, sig, sticky, s != 0);
    return (ml | mh) == 0 ? 0u : c;
}

struct SgdLuts {
    const int64_t* m;    // [2^fg.nbits] X_m (INT64_MIN = NaR)
    const uint16_t* c1;  // [2^fo.nbits] or null
    const uint16_t* c2;
};

// U elements per thread per grid-stride round (independent load -> table ->
// round chains in flight); a few blocks per SM, each looping (the per-block
// setup -- rounding table, segment table -- is paid once per block).
constexpr int kSgdU = 4;
// TO / TG / T1 / T2: code types of master, gradient, copies (compile-time
// widths: no per-element width branches); FMT: fixed_fmt id of the optimizer
// format (compile-time decode / rounding) or 0.  Segment pointers are global
// memory: loads by __ldg, stores by st.global (no generic LD/ST).
template <typename TO, typename TG, typename T1, typename T2, int FMT>
__global__ void __launch_bounds__(256) sgd_lut_kernel(PositFmt fo_rt, const __grid_constant__ SgdSegs segs,
                                                      SgdLuts t) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const PositFmt fo = fixed_fmt<FMT>(fo_rt);
    __shared__ uint4 s_lut[kPackLutEntries];
    build_pack_lut(fo, s_lut, threadIdx.x, blockDim.x);
    __shared__ int64_t s_start[kSgdMaxSeg + 1];
    for (int i = threadIdx.x; i <= segs.count; i += blockDim.x) s_start[i] = segs.start[i];
    __syncthreads();
    const uint32_t nar = 1u << (fo.nbits - 1);
    const int64_t total = s_start[segs.count];
    // a contiguous range per block, walked in rounds of kSgdU x blockDim
    // elements: the thread's segment only moves forward (no search per element)
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = blockIdx.x * per, r1 = min(total, r0 + per);
    int seg = 0;
    while (seg + 1 < segs.count && s_start[seg + 1] <= r0 + threadIdx.x) ++seg;
    for (int64_t i0 = r0 + threadIdx.x; i0 < r1; i0 += kSgdU * int64_t(blockDim.x)) {
        TO* mp[kSgdU];
        T1* c1p[kSgdU];
        T2* c2p[kSgdU];
        uint32_t w[kSgdU];
        int64_t xm[kSgdU];
        bool on[kSgdU];
#pragma unroll
        for (int u = 0; u < kSgdU; ++u) {
            const int64_t i = i0 + u * int64_t(blockDim.x);
            while (seg + 1 < segs.count && s_start[seg + 1] <= i) ++seg;
            on[u] = i < r1;
            const int64_t k = i - s_start[seg];
            mp[u] = static_cast<TO*>(segs.master[seg]) + k;
            c1p[u] = segs.copy1[seg] ? static_cast<T1*>(segs.copy1[seg]) + k : nullptr;
            c2p[u] = segs.copy2[seg] ? static_cast<T2*>(segs.copy2[seg]) + k : nullptr;
            if (on[u]) {
                xm[u] = __ldg(t.m + uint32_t(__ldg(static_cast<const TG*>(segs.grad[seg]) + k)));
                w[u] = uint32_t(__ldg(mp[u]));
            }
        }
#pragma unroll
        for (int u = 0; u < kSgdU; ++u) {
            if (!on[u]) continue;
            uint32_t r;
            if (w[u] == nar || xm[u] == INT64_MIN) {
                r = nar;
            } else {
                int64_t Xw;
                decode_x(w[u], fo, Xw);
                r = x_to_posit_lut(fo, Xw - xm[u], s_lut);
            }
            w[u] = r;
            __stcg(mp[u], TO(r));
        }
#pragma unroll
        for (int u = 0; u < kSgdU; ++u) {
            if (!on[u]) continue;
            if (c1p[u]) __stcg(c1p[u], T1(__ldg(t.c1 + w[u])));
            if (c2p[u]) __stcg(c2p[u], T2(__ldg(t.c2 + w[u])));
        }
    }
}

template <typename TO, typename TG, typename T1, typename T2>
void launch_sgd_lut(int grid, cudaStream_t st, const PositFmt& fo, const SgdSegs& sg, const SgdLuts& t) {
    if (fixed_fmt_id(fo) == 4) launch_pdl(sgd_lut_kernel<TO, TG, T1, T2, 4>, dim3(grid), dim3(256), 0, st, fo, sg, t);
    else if (fixed_fmt_id(fo) == 3) launch_pdl(sgd_lut_kernel<TO, TG, T1, T2, 3>, dim3(grid), dim3(256), 0, st, fo, sg, t);
    else launch_pdl(sgd_lut_kernel<TO, TG, T1, T2, 0>, dim3(grid), dim3(256), 0, st, fo, sg, t);
}

template <typename TO, typename TG>
void launch_sgd_lut_c(int b1, int b2, int grid, cudaStream_t st, const PositFmt& fo, const SgdSegs& sg,
                      const SgdLuts& t) {
    if (b1 == 1 && b2 == 1) launch_sgd_lut<TO, TG, uint8_t, uint8_t>(grid, st, fo, sg, t);
    else if (b1 == 1) launch_sgd_lut<TO, TG, uint8_t, uint16_t>(grid, st, fo, sg, t);
    else if (b2 == 1) launch_sgd_lut<TO, TG, uint16_t, uint8_t>(grid, st, fo, sg, t);
    else launch_sgd_lut<TO, TG, uint16_t, uint16_t>(grid, st, fo, sg, t);
}

// avgpool2d, tensor_ops.cpp:672-691: window sum (quire: exact, one rounding;
// sequential: add chain in (ky,kx) order) then mul by the caller-quantized
// reciprocal (scale, :763-769).
__global__ void avgpool_fwd_kernel(PositFmt f, int b, const void* x, int64_t NC, int64_t H,
                                   int64_t W, int k, int s, int64_t OH, int64_t OW, int use_quire,
                                   uint32_t recip, void* y) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(o, NC * OH * OW) {
        const int64_t ox = o % OW, oy = (o / OW) % OH, nc = o / (OW * OH);
        const int64_t base = nc * H * W + (oy * s) * W + ox * s;
        uint32_t sum = 0;
        if (use_quire) {
            __int128 acc = 0;
            bool nar = false;
            for (int ky = 0; ky < k; ++ky)
                for (int kx = 0; kx < k; ++kx) {
                    __int128 X;
                    nar |= decode_x128(load_any(x, base + ky * W + kx, b), f, X);
                    acc += X;
                }
            const bool neg = acc < 0;
            sum = nar ? nar_of(f)
                      : round_mag128(f, neg, (unsigned __int128)(neg ? -acc : acc), -f.R);
        } else {
            bool first = true;
            for (int ky = 0; ky < k; ++ky)
                for (int kx = 0; kx < k; ++kx) {
                    const uint32_t v = load_any(x, base + ky * W + kx, b);
                    sum = first ? v : p_add(f, sum, v);
                    first = false;
                }
        }
        store_any(y, o, b, p_mul(f, sum, recip));
    }
}

// avgpool2d_backward, tensor_ops.cpp:693-720: g = mul(dy, recip); each input
// accumulates add(dx, g) over the windows containing it in output order.
__global__ void avgpool_bwd_kernel(PositFmt f, int b, const void* dy, int64_t NC, int64_t H,
                                   int64_t W, int k, int s, int64_t OH, int64_t OW, uint32_t recip,
                                   void* dx) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(t, NC * H * W) {
        const int64_t ix = t % W, iy = (t / W) % H, nc = t / (W * H);
        const int64_t oy0 = iy - k + 1 > 0 ? (iy - k + 1 + s - 1) / s : 0;
        const int64_t ox0 = ix - k + 1 > 0 ? (ix - k + 1 + s - 1) / s : 0;
        const int64_t oy1 = min(OH - 1, iy / s), ox1 = min(OW - 1, ix / s);
        uint32_t acc = 0;
        for (int64_t oy = oy0; oy <= oy1; ++oy)
            for (int64_t ox = ox0; ox <= ox1; ++ox)
                acc = p_add(f, acc, p_mul(f, load_any(dy, (nc * OH + oy) * OW + ox, b), recip));
        store_any(dx, t, b, acc);
    }
}

__global__ void from_float64_kernel(PositFmt f, int b, const double* x, void* out, int64_t n) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(i, n) { store_any(out, i, b, p_from_float64(f, x[i])); }
}

__global__ void scalar_eval_kernel(PositFmt f, int op, const uint32_t* a, const uint32_t* b,
                                   uint32_t* out, int64_t n) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    GRID_STRIDE(i, n) {
        const uint32_t x = a[i], y = b ? b[i] : 0u;
        uint32_t r;
        switch (op) {
            case 0: case 1: case 2: case 3: r = p_op(f, op, x, y); break;
            case 4: r = p_exp(f, x); break;
            case 5: r = p_log(f, x); break;
            case 6: r = p_round_to_int(f, x); break;
            case 7: r = p_ldexp(f, x, int32_t(y)); break;
            case 8: r = uint32_t(p_compare(f, x, y)); break;
            case 10: r = p_tanh(f, x); break;
            case 11: r = p_sigmoid(f, x); break;
            case 12: r = p_sqrt(f, x); break;
            default: r = uint32_t(p_to_int64(f, x)); break;
        }
        out[i] = r;
    }
}

}  // namespace pnn_b200

// =========================================================================
// C-ABI
// =========================================================================

using namespace pnn_b200;

namespace {

bool elt_fmt_ok(int nbits, int es) {
    if (nbits < 2 || nbits > 16 || es < 0 || es > 4) return false;
    return 2 * make_fmt(nbits, es).R <= 96;  // 128-bit images; up to posit(12,2)
}

int bytes_of(int nbits) { return nbits <= 8 ? 1 : 2; }

int grid1(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    return int(b < 1 ? 1 : b);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Code tables (one uint16 entry per source code), device-resident for the life
// of the process: kind 0 = SGD X_m[g] (int64 entries) per (fo, fg, lr), 1 = convert per (fo, fc),
// 2 = exp / 3 = log per format.  Built synchronously on the caller's stream the
// first time; during stream capture a missing table returns null ("use the
// scalar path"), so a CUDA graph replays launches with the tables resident.
uint16_t* code_table(int kind, const PositFmt& a, const PositFmt& b, uint32_t l, cudaStream_t st) {
    const int64_t n = int64_t(1) << (kind == 0 ? b.nbits : a.nbits);
    return static_cast<uint16_t*>(persistent_table(
        table_key(16 + kind, a.nbits, a.es, b.nbits, b.es, 0, l), size_t(n) * (kind == 0 ? 8 : 2), st,
        [&](void* p, cudaStream_t s) {
            if (kind == 0) launch_pdl(sgd_xm_lut_kernel, dim3(grid1(n)), dim3(256), 0, s, a, b, l, static_cast<int64_t*>(p));
            else if (kind == 1) launch_pdl(copy_lut_kernel, dim3(grid1(n)), dim3(256), 0, s, a, b, static_cast<uint16_t*>(p));
            else launch_pdl(fn_lut_kernel, dim3(grid1(n)), dim3(256), 0, s, a, kind - 2, static_cast<uint16_t*>(p));
        }));
}

bool sgd_luts(const PositFmt& fo, const PositFmt& fg, uint32_t lr, const PositFmt* f1, const PositFmt* f2,
              cudaStream_t st, SgdLuts* out) {
    auto get = [&](int kind, const PositFmt& a, const PositFmt& b, uint32_t l) {
        return code_table(kind, a, b, l, st);
    };
    out->m = reinterpret_cast<const int64_t*>(get(0, fo, fg, lr));
    out->c1 = f1 ? get(1, fo, *f1, 0) : nullptr;
    out->c2 = f2 ? get(1, fo, *f2, 0) : nullptr;
    return out->m && (!f1 || out->c1) && (!f2 || out->c2);
}

int launched(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return PNN_OK;
    return set_status(PNN_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CHECK_FMT(n, e)                                                               \
    if (!elt_fmt_ok(n, e)) return set_status(PNN_EUNSUPPORTED, "format not supported")

}  // namespace

extern "C" {

int pnn_convert(int src_nbits, int src_es, int dst_nbits, int dst_es, const void* src, void* dst,
                int64_t n, void* stream) {
    CHECK_FMT(src_nbits, src_es);
    CHECK_FMT(dst_nbits, dst_es);
    if (n < 0 || (n > 0 && (!src || !dst))) return set_status(PNN_EINVAL, "convert: bad arguments");
    if (n == 0) return PNN_OK;
    const PositFmt s = make_fmt(src_nbits, src_es), d = make_fmt(dst_nbits, dst_es);
    auto st = (cudaStream_t)stream;
    if (aligned16(src) && aligned16(dst)) {
        const int grid = grid1(n / 8 + 1) < 148 * 4 ? grid1(n / 8 + 1) : 148 * 4;
        const int sb = bytes_of(src_nbits), db = bytes_of(dst_nbits);
        if (sb == 1 && db == 1)
            launch_pdl(convert_vec_kernel<uint8_t, uint8_t>, dim3(grid), dim3(256), 0, st, s, (const uint8_t*)src, d, (uint8_t*)dst, n);
        else if (sb == 1)
            launch_pdl(convert_vec_kernel<uint8_t, uint16_t>, dim3(grid), dim3(256), 0, st, s, (const uint8_t*)src, d, (uint16_t*)dst, n);
        else if (db == 1)
            launch_pdl(convert_vec_kernel<uint16_t, uint8_t>, dim3(grid), dim3(256), 0, st, s, (const uint16_t*)src, d, (uint8_t*)dst, n);
        else
            launch_pdl(convert_vec_kernel<uint16_t, uint16_t>, dim3(grid), dim3(256), 0, st, s, (const uint16_t*)src, d, (uint16_t*)dst, n);
    } else {
        launch_pdl(convert_kernel, dim3(grid1(n)), dim3(256), 0, st, s, bytes_of(src_nbits), src, d, bytes_of(dst_nbits),
                                                 dst, n);
    }
    return launched("convert");
}

int pnn_relu_fwd(int nbits, int es, const void* x, void* y, int64_t n, void* stream) {
    CHECK_FMT(nbits, es);
    if (n < 0) return set_status(PNN_EINVAL, "relu: bad size");
    if (n == 0) return PNN_OK;
    auto st = (cudaStream_t)stream;
    if (aligned16(x) && aligned16(y)) {
        if (bytes_of(nbits) == 1)
            launch_pdl(relu_fwd_vec_kernel<uint8_t>, dim3(grid1(n / 8 + 1)), dim3(256), 0, st, nbits, (const uint8_t*)x, (uint8_t*)y, n);
        else
            launch_pdl(relu_fwd_vec_kernel<uint16_t>, dim3(grid1(n / 8 + 1)), dim3(256), 0, st, nbits, (const uint16_t*)x, (uint16_t*)y, n);
    } else {
        launch_pdl(relu_fwd_kernel, dim3(grid1(n)), dim3(256), 0, st, make_fmt(nbits, es), bytes_of(nbits), x, y, n);
    }
    return launched("relu_fwd");
}

int pnn_relu_bwd(int x_nbits, int x_es, const void* x, int g_nbits, int g_es, const void* dy,
                 void* dx, int64_t n, void* stream) {
    CHECK_FMT(x_nbits, x_es);
    CHECK_FMT(g_nbits, g_es);
    if (n < 0) return set_status(PNN_EINVAL, "relu: bad size");
    if (n == 0) return PNN_OK;
    auto st = (cudaStream_t)stream;
    if (aligned16(x) && aligned16(dy) && aligned16(dx)) {
        const int grid = grid1(n / 8 + 1);
        const int xb = bytes_of(x_nbits), gb = bytes_of(g_nbits);
        if (xb == 1 && gb == 1)
            launch_pdl(relu_bwd_vec_kernel<uint8_t, uint8_t>, dim3(grid), dim3(256), 0, st, x_nbits, (const uint8_t*)x, (const uint8_t*)dy, (uint8_t*)dx, n);
        else if (xb == 1)
            launch_pdl(relu_bwd_vec_kernel<uint8_t, uint16_t>, dim3(grid), dim3(256), 0, st, x_nbits, (const uint8_t*)x, (const uint16_t*)dy, (uint16_t*)dx, n);
        else if (gb == 1)
            launch_pdl(relu_bwd_vec_kernel<uint16_t, uint8_t>, dim3(grid), dim3(256), 0, st, x_nbits, (const uint16_t*)x, (const uint8_t*)dy, (uint8_t*)dx, n);
        else
            launch_pdl(relu_bwd_vec_kernel<uint16_t, uint16_t>, dim3(grid), dim3(256), 0, st, x_nbits, (const uint16_t*)x, (const uint16_t*)dy, (uint16_t*)dx, n);
    } else {
        launch_pdl(relu_bwd_kernel, dim3(grid1(n)), dim3(256), 0, st, make_fmt(x_nbits, x_es), bytes_of(x_nbits), x,
                                                  bytes_of(g_nbits), dy, dx, n);
    }
    return launched("relu_bwd");
}

// 2x2 / stride 2 exactly tiled, 16-byte vectors of x fit whole output rows
static bool pool2_vec_ok(int nbits, int64_t N, int64_t C, int64_t H, int64_t W, int k, int stride,
                         const void* x) {
    const int64_t wpt = nbits <= 8 ? 8 : 4;
    return k == 2 && stride == 2 && H % 2 == 0 && W % (2 * wpt) == 0 && aligned16(x) &&
           N * C * H * W < (int64_t(1) << 31);
}

int pnn_maxpool2d_fwd(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H,
                      int64_t W, int k, int stride, void* y, int64_t* argmax, void* stream) {
    CHECK_FMT(nbits, es);
    if (N < 0 || C < 1 || k < 1 || stride < 1 || H < k || W < k)
        return set_status(PNN_EINVAL, "maxpool2d: window larger than input");
    const int64_t OH = (H - k) / stride + 1, OW = (W - k) / stride + 1;
    if (N == 0) return PNN_OK;
    if (argmax == nullptr && pool2_vec_ok(nbits, N, C, H, W, k, stride, x) && aligned16(y)) {
        // no argmax wanted (the layer recomputes it in pnn_maxpool2d_bwd_x)
        const int rows = int(N * C * OH), wpt = nbits <= 8 ? 8 : 4;
        const int grid = grid1(int64_t(rows) * (OW / wpt));
        if (nbits <= 8)
            launch_pdl(maxpool2_fwd_vec_kernel<uint8_t>, dim3(grid), dim3(256), 0, (cudaStream_t)stream, 
                nbits, (const uint8_t*)x, (uint8_t*)y, rows, int(OW));
        else
            launch_pdl(maxpool2_fwd_vec_kernel<uint16_t>, dim3(grid), dim3(256), 0, (cudaStream_t)stream, 
                nbits, (const uint16_t*)x, (uint16_t*)y, rows, int(OW));
        return launched("maxpool2d_fwd");
    }
    if (argmax == nullptr) return set_status(PNN_EINVAL, "maxpool2d: argmax output required");
    if (k == stride && H == OH * k && W == OW * k && N * C * H * W < (int64_t(1) << 31))
        launch_pdl(maxpool_fwd_tiled_kernel, dim3(grid1(N * C * OH * OW)), dim3(256), 0, (cudaStream_t)stream, 
            make_fmt(nbits, es), bytes_of(nbits), x, int(N * C), int(OH), int(OW), k, y, argmax);
    else
        launch_pdl(maxpool_fwd_kernel, dim3(grid1(N * C * OH * OW)), dim3(256), 0, (cudaStream_t)stream, 
            make_fmt(nbits, es), bytes_of(nbits), x, N * C, H, W, k, stride, OH, OW, y, argmax);
    return launched("maxpool2d_fwd");
}

int pnn_maxpool2d_bwd_x(int x_nbits, int x_es, const void* x, int g_nbits, int g_es, const void* dy,
                        int64_t N, int64_t C, int64_t H, int64_t W, int k, int stride, void* dx,
                        void* stream) {
    return pnn_maxpool2d_relu_bwd_x(x_nbits, x_es, x, g_nbits, g_es, dy, N, C, H, W, k, stride, 0, dx,
                                    stream);
}

int pnn_maxpool2d_relu_bwd_x(int x_nbits, int x_es, const void* x, int g_nbits, int g_es, const void* dy,
                             int64_t N, int64_t C, int64_t H, int64_t W, int k, int stride, int relu_gate,
                             void* dx, void* stream) {
    CHECK_FMT(x_nbits, x_es);
    CHECK_FMT(g_nbits, g_es);
    if (N < 0 || C < 1 || k < 1 || stride < 1 || H < k || W < k || !x || !dy || !dx)
        return set_status(PNN_EINVAL, "maxpool2d_backward: bad shape");
    if (N == 0) return PNN_OK;
    if (!pool2_vec_ok(x_nbits, N, C, H, W, k, stride, x))
        return set_status(PNN_EUNSUPPORTED, "maxpool2d_bwd_x: 2x2/2 tiled, W a multiple of the vector");
    const int rows = int(N * C * (H / 2)), OW = int(W / 2), wpt = x_nbits <= 8 ? 8 : 4;
    const int grid = grid1(int64_t(rows) * (OW / wpt));
    auto st = (cudaStream_t)stream;
    const bool x8 = x_nbits <= 8, g8 = g_nbits <= 8;
#define PNN_MPB(TX, TG)                                                                    \
    launch_pdl(maxpool2_bwd_x_kernel<TX, TG>, dim3(grid), dim3(256), 0, st, x_nbits, (const TX*)x, (const TG*)dy, \
                                                        (TG*)dx, rows, OW, relu_gate)
    if (x8 && g8) PNN_MPB(uint8_t, uint8_t);
    else if (x8) PNN_MPB(uint8_t, uint16_t);
    else if (g8) PNN_MPB(uint16_t, uint8_t);
    else PNN_MPB(uint16_t, uint16_t);
#undef PNN_MPB
    return launched("maxpool2d_bwd_x");
}

int pnn_maxpool2d_bwd(int nbits, int es, const void* dy, const int64_t* argmax, int64_t N,
                      int64_t C, int64_t H, int64_t W, int k, int stride, void* dx, void* stream) {
    CHECK_FMT(nbits, es);
    if (N < 0 || C < 1 || k < 1 || stride < 1 || H < k || W < k)
        return set_status(PNN_EINVAL, "maxpool2d_backward: bad shape");
    const int64_t OH = (H - k) / stride + 1, OW = (W - k) / stride + 1;
    if (N == 0) return PNN_OK;
    if (k == stride && H == OH * k && W == OW * k && N * C * H * W < (int64_t(1) << 31))
        launch_pdl(maxpool_bwd_tiled_kernel, dim3(grid1(N * C * OH * OW)), dim3(256), 0, (cudaStream_t)stream, 
            bytes_of(nbits), dy, argmax, int(N * C), int(OH), int(OW), k, dx);
    else
        launch_pdl(maxpool_bwd_kernel, dim3(grid1(N * C * H * W)), dim3(256), 0, (cudaStream_t)stream, 
            make_fmt(nbits, es), bytes_of(nbits), dy, argmax, N * C, H, W, k, stride, OH, OW, dx);
    return launched("maxpool2d_bwd");
}

int pnn_softmax_xent(int nbits, int es, const void* logits, const int32_t* labels, int64_t B,
                     int64_t classes, int log2_batch, void* dlogits, void* loss_rows,
                     void* loss_out, void* raw_word, void* raw_nar, void* stream) {
    return pnn_softmax_xent_scaled(nbits, es, logits, labels, B, classes, log2_batch, 0, dlogits,
                                   loss_rows, loss_out, raw_word, raw_nar, stream);
}

int pnn_softmax_xent_scaled(int nbits, int es, const void* logits, const int32_t* labels,
                            int64_t B, int64_t classes, int log2_batch, int grad_scale_log2,
                            void* dlogits, void* loss_rows, void* loss_out, void* raw_word,
                            void* raw_nar, void* stream) {
    CHECK_FMT(nbits, es);
    if (B < 1 || classes < 1 || !logits || !labels || !dlogits || !loss_rows)
        return set_status(PNN_EINVAL, "softmax_xent: bad arguments");
    const PositFmt f = make_fmt(nbits, es);
    if (raw_word && f.W > 128)
        return set_status(PNN_EUNSUPPORTED, "softmax_xent: raw loss words need a quire of <= 128 bits");
    auto st = (cudaStream_t)stream;
    launch_pdl(softmax_xent_kernel, dim3(grid1(B * 32)), dim3(256), 0, st, f, bytes_of(nbits), logits, labels, B, classes,
                                                      log2_batch, grad_scale_log2, dlogits,
                                                      loss_rows, nullptr, code_table(2, f, f, 0, st),
                                                      code_table(3, f, f, 0, st));
    if (loss_out || raw_word)
        launch_pdl(loss_reduce_kernel, dim3(1), dim3(256), 0, st, f, bytes_of(nbits), loss_rows, B, log2_batch,
                                              loss_out, (unsigned __int128*)raw_word,
                                              (uint8_t*)raw_nar);
    return launched("softmax_xent");
}

int pnn_softmax_xent_grad(int nbits, int es, const void* logits, const int32_t* labels, int64_t B,
                          int64_t classes, int log2_batch, int grad_scale_log2, void* dlogits,
                          void* s_rows, void* stream) {
    CHECK_FMT(nbits, es);
    if (B < 1 || classes < 1 || !logits || !labels || !dlogits || !s_rows)
        return set_status(PNN_EINVAL, "softmax_xent_grad: bad arguments");
    const PositFmt f = make_fmt(nbits, es);
    launch_pdl(softmax_xent_kernel, dim3(grid1(B * 32)), dim3(256), 0, (cudaStream_t)stream, 
        f, bytes_of(nbits), logits, labels, B, classes, log2_batch, grad_scale_log2,
        dlogits, nullptr, s_rows, code_table(2, f, f, 0, (cudaStream_t)stream),
        static_cast<const uint16_t*>(nullptr));
    return launched("softmax_xent_grad");
}

int pnn_softmax_xent_loss(int nbits, int es, const void* logits, const int32_t* labels,
                          const void* s_rows, int64_t B, int64_t classes, int log2_batch,
                          void* loss_rows, void* loss_out, void* raw_word, void* raw_nar, void* stream) {
    CHECK_FMT(nbits, es);
    if (B < 1 || classes < 1 || !logits || !labels || !s_rows || !loss_rows)
        return set_status(PNN_EINVAL, "softmax_xent_loss: bad arguments");
    const PositFmt f = make_fmt(nbits, es);
    if (raw_word && f.W > 128)
        return set_status(PNN_EUNSUPPORTED, "softmax_xent: raw loss words need a quire of <= 128 bits");
    auto st = (cudaStream_t)stream;
    launch_pdl(xent_loss_rows_kernel, dim3(grid1(B)), dim3(256), 0, st, f, bytes_of(nbits), logits, labels, s_rows, B,
                                                     classes, loss_rows, code_table(3, f, f, 0, st));
    if (loss_out || raw_word)
        launch_pdl(loss_reduce_kernel, dim3(1), dim3(256), 0, st, f, bytes_of(nbits), loss_rows, B, log2_batch, loss_out,
                                              (unsigned __int128*)raw_word, (uint8_t*)raw_nar);
    return launched("softmax_xent_loss");
}

int pnn_loss_reduce(int nbits, int es, const void* loss_rows, int64_t B, int log2_batch,
                    void* loss_out, void* stream) {
    CHECK_FMT(nbits, es);
    if (B < 1 || !loss_rows || !loss_out) return set_status(PNN_EINVAL, "loss_reduce: bad arguments");
    launch_pdl(loss_reduce_kernel, dim3(1), dim3(256), 0, (cudaStream_t)stream, make_fmt(nbits, es), bytes_of(nbits),
                                                            loss_rows, B, log2_batch, loss_out,
                                                            nullptr, nullptr);
    return launched("loss_reduce");
}

int pnn_sgd_step(int opt_nbits, int opt_es, void* master, int g_nbits, int g_es, const void* grad,
                 int64_t n, uint32_t lr_code, int c1_nbits, int c1_es, void* copy1, int c2_nbits,
                 int c2_es, void* copy2, void* stream) {
    return pnn_sgd_step_scaled(opt_nbits, opt_es, master, g_nbits, g_es, grad, n, lr_code, c1_nbits,
                               c1_es, copy1, c2_nbits, c2_es, copy2, 0, stream);
}

int pnn_sgd_step_scaled(int opt_nbits, int opt_es, void* master, int g_nbits, int g_es,
                        const void* grad, int64_t n, uint32_t lr_code, int c1_nbits, int c1_es,
                        void* copy1, int c2_nbits, int c2_es, void* copy2, int grad_scale_log2,
                        void* stream) {
    CHECK_FMT(opt_nbits, opt_es);
    CHECK_FMT(g_nbits, g_es);
    if (copy1) CHECK_FMT(c1_nbits, c1_es);
    if (copy2) CHECK_FMT(c2_nbits, c2_es);
    if (n < 0 || (n > 0 && (!master || !grad))) return set_status(PNN_EINVAL, "sgd: bad arguments");
    if (n == 0) return PNN_OK;
    const PositFmt f1 = copy1 ? make_fmt(c1_nbits, c1_es) : make_fmt(opt_nbits, opt_es);
    const PositFmt f2 = copy2 ? make_fmt(c2_nbits, c2_es) : make_fmt(opt_nbits, opt_es);
    launch_pdl(sgd_kernel, dim3(grid1(n)), dim3(256), 0, (cudaStream_t)stream, 
        make_fmt(opt_nbits, opt_es), bytes_of(opt_nbits), master, make_fmt(g_nbits, g_es),
        bytes_of(g_nbits), grad, n, lr_code, f1, bytes_of(f1.nbits), copy1, f2,
        bytes_of(f2.nbits), copy2, grad_scale_log2);
    return launched("sgd_step");
}

int pnn_sgd_step_multi(int opt_nbits, int opt_es, int g_nbits, int g_es, uint32_t lr_code, int c1_nbits,
                       int c1_es, int c2_nbits, int c2_es, int grad_scale_log2, int count,
                       void* const* masters, const void* const* grads, void* const* copy1s,
                       void* const* copy2s, const int64_t* ns, void* stream) {
    CHECK_FMT(opt_nbits, opt_es);
    CHECK_FMT(g_nbits, g_es);
    if (count < 0 || (count > 0 && (!masters || !grads || !ns)))
        return set_status(PNN_EINVAL, "sgd_multi: bad arguments");
    const bool has1 = copy1s != nullptr, has2 = copy2s != nullptr;
    if (has1) CHECK_FMT(c1_nbits, c1_es);
    if (has2) CHECK_FMT(c2_nbits, c2_es);
    const PositFmt fo = make_fmt(opt_nbits, opt_es), fg = make_fmt(g_nbits, g_es);
    const PositFmt f1 = has1 ? make_fmt(c1_nbits, c1_es) : fo, f2 = has2 ? make_fmt(c2_nbits, c2_es) : fo;
    // integer-image update (sgd_fast): images within 64 bits, exact intermediates
    // within the optimizer quire word (|X_g| 2^(2Ro-Rg), lr * g', (w - m) 2^Ro)
    const bool lr_nar = lr_code == (1u << (opt_nbits - 1));
    // copies by integer image: the shifted image stays within the copy format's quire word
    auto copy_ok = [&](const PositFmt& fc) {
        return 2 * fc.R <= 60 && fc.W <= 128 && fo.R + 2 * fc.R + 1 < fc.W && 2 * fo.R <= 60;
    };
    int fast = grad_scale_log2 == 0 && !lr_nar && fo.W > 64 && 2 * fo.R <= 62 && 2 * fg.R <= 62 &&
                     2 * fo.R >= fg.R && 2 * fo.R <= 60 && fo.W <= 128 && fg.R + 2 * fo.R + 1 < fo.W &&
                     4 * fo.R + 1 < fo.W && 3 * fo.R + 2 < fo.W;
    if (fast) fast |= (has1 && copy_ok(f1) ? 2 : 0) | (has2 && copy_ok(f2) ? 4 : 0);
    // table path: images within int64 (2R_o + 1 <= 63), 16-bit tables; the
    // tables are built on first use outside stream capture (a CUDA graph
    // replays the launch with the tables already resident)
    SgdLuts luts{};
    const bool lut_path = grad_scale_log2 == 0 && 2 * fo.R + 1 <= 63 &&
                          sgd_luts(fo, fg, lr_code, has1 ? &f1 : nullptr, has2 ? &f2 : nullptr,
                                   (cudaStream_t)stream, &luts);
    for (int base = 0; base < count; base += kSgdMaxSeg) {
        SgdSegs sg{};
        sg.count = 0;
        int64_t tot = 0;
        for (int i = base; i < count && i < base + kSgdMaxSeg; ++i) {
            if (ns[i] < 0 || (ns[i] > 0 && (!masters[i] || !grads[i])))
                return set_status(PNN_EINVAL, "sgd_multi: bad arguments");
            const int j = sg.count++;
            sg.start[j] = tot;
            sg.master[j] = masters[i];
            sg.grad[j] = grads[i];
            sg.copy1[j] = has1 ? copy1s[i] : nullptr;
            sg.copy2[j] = has2 ? copy2s[i] : nullptr;
            tot += ns[i];
        }
        sg.start[sg.count] = tot;
        if (tot == 0) continue;
        if (lut_path) {
            int gr = grid1((tot + kSgdU - 1) / kSgdU);
            gr = gr < 148 * 4 ? gr : 148 * 4;
            const int b1 = bytes_of(f1.nbits), b2 = bytes_of(f2.nbits);
            const auto st = (cudaStream_t)stream;
            if (bytes_of(opt_nbits) == 2 && bytes_of(g_nbits) == 2)
                launch_sgd_lut_c<uint16_t, uint16_t>(b1, b2, gr, st, fo, sg, luts);
            else if (bytes_of(opt_nbits) == 2)
                launch_sgd_lut_c<uint16_t, uint8_t>(b1, b2, gr, st, fo, sg, luts);
            else if (bytes_of(g_nbits) == 2)
                launch_sgd_lut_c<uint8_t, uint16_t>(b1, b2, gr, st, fo, sg, luts);
            else
                launch_sgd_lut_c<uint8_t, uint8_t>(b1, b2, gr, st, fo, sg, luts);
            continue;
        }
        launch_pdl(sgd_multi_kernel, dim3(grid1(tot)), dim3(256), 0, (cudaStream_t)stream, 
            fo, bytes_of(opt_nbits), fg, bytes_of(g_nbits), lr_code, f1, bytes_of(f1.nbits), f2,
            bytes_of(f2.nbits), grad_scale_log2, sg, fast);
    }
    return launched("sgd_step_multi");
}

int pnn_avgpool2d_fwd(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H,
                      int64_t W, int k, int stride, int use_quire, uint32_t recip_code, void* y,
                      void* stream) {
    CHECK_FMT(nbits, es);
    if (N < 0 || C < 1 || k < 1 || stride < 1 || H < k || W < k)
        return set_status(PNN_EINVAL, "avgpool2d: window larger than input");
    const int64_t OH = (H - k) / stride + 1, OW = (W - k) / stride + 1;
    if (N == 0) return PNN_OK;
    launch_pdl(avgpool_fwd_kernel, dim3(grid1(N * C * OH * OW)), dim3(256), 0, (cudaStream_t)stream, 
        make_fmt(nbits, es), bytes_of(nbits), x, N * C, H, W, k, stride, OH, OW, use_quire,
        recip_code, y);
    return launched("avgpool2d_fwd");
}

int pnn_avgpool2d_bwd(int nbits, int es, const void* dy, int64_t N, int64_t C, int64_t H,
                      int64_t W, int k, int stride, uint32_t recip_code, void* dx, void* stream) {
    CHECK_FMT(nbits, es);
    if (N < 0 || C < 1 || k < 1 || stride < 1 || H < k || W < k)
        return set_status(PNN_EINVAL, "avgpool2d_backward: bad shape");
    const int64_t OH = (H - k) / stride + 1, OW = (W - k) / stride + 1;
    if (N == 0) return PNN_OK;
    launch_pdl(avgpool_bwd_kernel, dim3(grid1(N * C * H * W)), dim3(256), 0, (cudaStream_t)stream, 
        make_fmt(nbits, es), bytes_of(nbits), dy, N * C, H, W, k, stride, OH, OW, recip_code, dx);
    return launched("avgpool2d_bwd");
}

int pnn_from_float64(int nbits, int es, const double* x, void* codes, int64_t n, void* stream) {
    CHECK_FMT(nbits, es);
    if (n < 0 || (n > 0 && (!x || !codes))) return set_status(PNN_EINVAL, "from_float64: bad args");
    if (n == 0) return PNN_OK;
    launch_pdl(from_float64_kernel, dim3(grid1(n)), dim3(256), 0, (cudaStream_t)stream, make_fmt(nbits, es),
                                                                    bytes_of(nbits), x, codes, n);
    return launched("from_float64");
}

int pnn_scalar_eval(int nbits, int es, int op, const uint32_t* a, const uint32_t* b,
                    uint32_t* out, int64_t n, void* stream) {
    CHECK_FMT(nbits, es);
    if (n <= 0) return PNN_OK;
    launch_pdl(scalar_eval_kernel, dim3(grid1(n)), dim3(256), 0, (cudaStream_t)stream, make_fmt(nbits, es), op, a, b,
                                                                   out, n);
    return launched("scalar_eval");
}

}  // extern "C"
