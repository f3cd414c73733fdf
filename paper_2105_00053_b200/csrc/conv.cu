// Conv2d / Linear passes as implicit GEMMs on the tcgen05 quire core.
//
//   forward      conv2d -> conv_quire            proj/src/tensor_ops.cpp:494-525, 266-297
//                  GEMM  M = N*OH*OW pixels, N = F, K = C*KH*KW (+1: bias * 1.0 inside the quire, :292)
//   input grad   conv2d_input_grad               tensor_ops.cpp:527-574
//                  GEMM  M = N*H*W, N = C, K = F*KH*KW (taps that fail the divisibility /
//                        range tests of :546-554 are zero and carry no NaR)
//   weight grad  conv2d_weight_grad              tensor_ops.cpp:576-603
//                  GEMM  M = C*KH*KW, N = F, K = N*OH*OW (batch reduction; split-K)
//   bias grad    conv2d_bias_grad / column_sum   tensor_ops.cpp:605-618, 722-731
//                  CUDA-core exact 128-bit reduction (quire sum of X * 2^R)
//
// A Linear layer is the 1x1 convolution of [B, in, 1, 1].
// NaR: an output is NaR iff one of ITS terms has a NaR operand (quire.hpp:55,
// NaR * 0 included).  For forward and weight-grad every k of the GEMM is a
// term, so operand row/column flags are exact; for input-grad the weight-side
// flag is applied per output over its valid taps only (dgrad_weight_nar).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <type_traits>

#include "../../include/pnn_b200.h"
#include "igemm.h"
#include "igemm_core.cuh"
#include "pdl.cuh"
#include "status.h"
#include "tables.h"

namespace pnn_b200 {

// ---- forward ---------------------------------------------------------------

template <typename CodeT>
struct FetchIm2colFwd {  // X[r = (n,oy,ox)][k = (c,ky,kx) | bias col]
    const CodeT* x;
    ConvGeom g;
    int64_t kconv;
    uint32_t one_code;
    static constexpr bool kRowFastest = true;
    static constexpr bool kVecK = false, kVecR = false, kSep = true;
    __device__ const CodeT* ptr(int64_t, int64_t) const { return nullptr; }
    // separable form: row -> (image base + window origin), k -> (tap offset, tap)
    struct RI { int64_t base; int iy0, ix0; };
    struct KI { int64_t off; int ky, kx; };
    __device__ __forceinline__ RI row(int64_t r) const {
        const int64_t ohw = g.OH * g.OW;
        const int64_t n = r / ohw, p = r - n * ohw, oy = p / g.OW, ox = p - oy * g.OW;
        const int iy0 = int(oy * g.stride - g.pad), ix0 = int(ox * g.stride - g.pad);
        return RI{n * g.C * g.H * g.W + int64_t(iy0) * g.W + ix0, iy0, ix0};
    }
    __device__ __forceinline__ KI kin(int64_t k) const {
        if (k >= kconv) return KI{0, 1 << 30, 0};  // bias column
        const int64_t khw = g.KH * g.KW;
        const int64_t c = k / khw, t = k - c * khw, ky = t / g.KW, kx = t - ky * g.KW;
        return KI{c * g.H * g.W + ky * g.W + kx, int(ky), int(kx)};
    }
    __device__ __forceinline__ uint32_t at(const RI& ri, const KI& ki) const {
        if (ki.ky == (1 << 30)) return one_code;
        const int iy = ri.iy0 + ki.ky, ix = ri.ix0 + ki.kx;
        if (unsigned(iy) >= unsigned(g.H) || unsigned(ix) >= unsigned(g.W)) return 0;
        return uint32_t(x[ri.base + ki.off]);
    }
    __device__ __forceinline__ uint32_t operator()(int64_t r, int64_t k) const {
        if (k >= kconv) return one_code;
        const int64_t ohw = g.OH * g.OW;
        const int64_t n = r / ohw, p = r - n * ohw, oy = p / g.OW, ox = p - oy * g.OW;
        const int64_t khw = g.KH * g.KW;
        const int64_t c = k / khw, t = k - c * khw, ky = t / g.KW, kx = t - ky * g.KW;
        const int64_t iy = oy * g.stride + ky - g.pad, ix = ox * g.stride + kx - g.pad;
        if (iy < 0 || iy >= g.H || ix < 0 || ix >= g.W) return 0;
        return uint32_t(x[((n * g.C + c) * g.H + iy) * g.W + ix]);
    }
};

template <typename CodeT>
struct FetchWeightFwd {  // X[r = f][k = (c,ky,kx) | bias col]
    const CodeT* w;
    const CodeT* bias;
    int64_t kconv;
    static constexpr bool kRowFastest = false;
    static constexpr bool kVecK = false, kVecR = false, kSep = true;
    __device__ const CodeT* ptr(int64_t, int64_t) const { return nullptr; }
    struct RI { int64_t base; int f, pad_; };
    struct KI { int64_t off; int is_bias, pad_; };
    __device__ __forceinline__ RI row(int64_t r) const { return RI{r * kconv, int(r), 0}; }
    __device__ __forceinline__ KI kin(int64_t k) const { return KI{k, k >= kconv ? 1 : 0, 0}; }
    __device__ __forceinline__ uint32_t at(const RI& ri, const KI& ki) const {
        return ki.is_bias ? uint32_t(bias[ri.f]) : uint32_t(w[ri.base + ki.off]);
    }
    __device__ __forceinline__ uint32_t operator()(int64_t r, int64_t k) const {
        return k < kconv ? uint32_t(w[r * kconv + k]) : uint32_t(bias[r]);
    }
};

// ---- input grad --------------------------------------------------------------

template <typename CodeT>
struct FetchDgradDy {  // X[r = (n,iy,ix)][k = (f,ky,kx)]
    const CodeT* dy;
    ConvGeom g;
    static constexpr bool kRowFastest = true;
    static constexpr bool kVecK = false, kVecR = false, kSep = true;
    __device__ const CodeT* ptr(int64_t, int64_t) const { return nullptr; }
    struct RI { int64_t base; int ty0, tx0; };  // dy image base, padded input position
    struct KI { int64_t off; int ky, kx; };     // channel-f plane offset, tap
    __device__ __forceinline__ RI row(int64_t r) const {
        const int64_t hw = g.H * g.W;
        const int64_t n = r / hw, p = r - n * hw, iy = p / g.W, ix = p - iy * g.W;
        return RI{n * g.F * g.OH * g.OW, int(iy + g.pad), int(ix + g.pad)};
    }
    __device__ __forceinline__ KI kin(int64_t k) const {
        const int64_t khw = g.KH * g.KW;
        const int64_t f = k / khw, t = k - f * khw, ky = t / g.KW, kx = t - ky * g.KW;
        return KI{f * g.OH * g.OW, int(ky), int(kx)};
    }
    __device__ __forceinline__ uint32_t at(const RI& ri, const KI& ki) const {
        int oy = ri.ty0 - ki.ky, ox = ri.tx0 - ki.kx;  // taps of tensor_ops.cpp:546-554
        if (oy < 0 || ox < 0) return 0;
        if (g.stride != 1) {
            if (oy % g.stride || ox % g.stride) return 0;
            oy /= g.stride;
            ox /= g.stride;
        }
        if (oy >= g.OH || ox >= g.OW) return 0;
        return uint32_t(dy[ri.base + ki.off + int64_t(oy) * g.OW + ox]);
    }
    __device__ __forceinline__ uint32_t operator()(int64_t r, int64_t k) const {
        const int64_t hw = g.H * g.W;
        const int64_t n = r / hw, p = r - n * hw, iy = p / g.W, ix = p - iy * g.W;
        const int64_t khw = g.KH * g.KW;
        const int64_t f = k / khw, t = k - f * khw, ky = t / g.KW, kx = t - ky * g.KW;
        const int64_t ty = iy + g.pad - ky, tx = ix + g.pad - kx;
        if (ty < 0 || tx < 0 || ty % g.stride || tx % g.stride) return 0;
        const int64_t oy = ty / g.stride, ox = tx / g.stride;
        if (oy >= g.OH || ox >= g.OW) return 0;
        return uint32_t(dy[((n * g.F + f) * g.OH + oy) * g.OW + ox]);
    }
};

template <typename CodeT>
struct FetchDgradW {  // X[r = c][k = (f,ky,kx)] = w[f][c][ky][kx]
    const CodeT* w;
    ConvGeom g;
    static constexpr bool kRowFastest = false;
    static constexpr bool kVecK = false, kVecR = false, kSep = true;
    __device__ const CodeT* ptr(int64_t, int64_t) const { return nullptr; }
    struct RI { int64_t base; int pad0, pad1; };
    struct KI { int64_t off; int pad0, pad1; };
    __device__ __forceinline__ RI row(int64_t r) const { return RI{r * g.KH * g.KW, 0, 0}; }
    __device__ __forceinline__ KI kin(int64_t k) const {
        const int64_t khw = g.KH * g.KW;
        const int64_t f = k / khw, t = k - f * khw;
        return KI{f * g.C * khw + t, 0, 0};
    }
    __device__ __forceinline__ uint32_t at(const RI& ri, const KI& ki) const {
        return uint32_t(w[ri.base + ki.off]);
    }
    __device__ __forceinline__ uint32_t operator()(int64_t r, int64_t k) const {
        const int64_t khw = g.KH * g.KW;
        const int64_t f = k / khw, t = k - f * khw;
        return uint32_t(w[(f * g.C + r) * khw + t]);
    }
};

// ---- weight grad -------------------------------------------------------------

template <typename CodeT>
struct FetchWgradX {  // X[r = (c,ky,kx)][k = (n,oy,ox)] = x_pad[n][c][oy*s+ky][ox*s+kx]
    const CodeT* x;
    ConvGeom g;
    static constexpr bool kRowFastest = false;
    static constexpr bool kVecK = false, kVecR = false, kSep = true;
    __device__ const CodeT* ptr(int64_t, int64_t) const { return nullptr; }
    struct RI { int64_t base; int ky_p, kx_p; };  // channel plane, tap - pad
    struct KI { int64_t off; int oys, oxs; };     // image base, output position * stride
    __device__ __forceinline__ RI row(int64_t r) const {
        const int64_t khw = g.KH * g.KW;
        const int64_t c = r / khw, t = r - c * khw, ky = t / g.KW, kx = t - ky * g.KW;
        return RI{c * g.H * g.W, int(ky - g.pad), int(kx - g.pad)};
    }
    __device__ __forceinline__ KI kin(int64_t k) const {
        const int64_t ohw = g.OH * g.OW;
        const int64_t n = k / ohw, p = k - n * ohw, oy = p / g.OW, ox = p - oy * g.OW;
        return KI{n * g.C * g.H * g.W, int(oy * g.stride), int(ox * g.stride)};
    }
    __device__ __forceinline__ uint32_t at(const RI& ri, const KI& ki) const {
        const int iy = ki.oys + ri.ky_p, ix = ki.oxs + ri.kx_p;
        if (unsigned(iy) >= unsigned(g.H) || unsigned(ix) >= unsigned(g.W)) return 0;
        return uint32_t(x[ri.base + ki.off + int64_t(iy) * g.W + ix]);
    }
    __device__ __forceinline__ uint32_t operator()(int64_t r, int64_t k) const {
        const int64_t khw = g.KH * g.KW;
        const int64_t c = r / khw, t = r - c * khw, ky = t / g.KW, kx = t - ky * g.KW;
        const int64_t ohw = g.OH * g.OW;
        const int64_t n = k / ohw, p = k - n * ohw, oy = p / g.OW, ox = p - oy * g.OW;
        const int64_t iy = oy * g.stride + ky - g.pad, ix = ox * g.stride + kx - g.pad;
        if (iy < 0 || iy >= g.H || ix < 0 || ix >= g.W) return 0;
        return uint32_t(x[((n * g.C + c) * g.H + iy) * g.W + ix]);
    }
};

template <typename CodeT>
struct FetchWgradDy {  // X[r = f][k = (n,o)] = dy[n][f][o]
    const CodeT* dy;
    ConvGeom g;
    static constexpr bool kRowFastest = false;
    static constexpr bool kVecK = false, kVecR = false, kSep = true;
    __device__ const CodeT* ptr(int64_t, int64_t) const { return nullptr; }
    struct RI { int64_t base; int pad0, pad1; };
    struct KI { int64_t off; int pad0, pad1; };
    __device__ __forceinline__ RI row(int64_t r) const { return RI{r * g.OH * g.OW, 0, 0}; }
    __device__ __forceinline__ KI kin(int64_t k) const {
        const int64_t ohw = g.OH * g.OW;
        const int64_t n = k / ohw, p = k - n * ohw;
        return KI{n * g.F * ohw + p, 0, 0};
    }
    __device__ __forceinline__ uint32_t at(const RI& ri, const KI& ki) const {
        return uint32_t(dy[ri.base + ki.off]);
    }
    __device__ __forceinline__ uint32_t operator()(int64_t r, int64_t k) const {
        const int64_t ohw = g.OH * g.OW;
        const int64_t n = k / ohw, p = k - n * ohw;
        return uint32_t(dy[(n * g.F + r) * ohw + p]);
    }
};

// ---- bias grad / column sum -------------------------------------------------

// Exact quire sum of dy over (n, pixel) per channel: Q_f = 2^R * sum X (mod
// 2^W).  Stage 1: each block reduces a slice of (n) for one f into a 128-bit
// partial (|sum X| < 2^56 * 2^31 fits); stage 2 sums partials and rounds.
// P == 1 (Linear layers, column sums of dy [N][F]): a thread per channel,
// coalesced along F, a slice of rows per blockIdx.y; same partial layout.
template <typename CodeT>
__global__ void __launch_bounds__(256) bias_grad_cols_kernel(
    const CodeT* __restrict__ dy, int64_t N, int64_t F, PositFmt f, int slices,
    const int64_t* __restrict__ xlut, unsigned __int128* __restrict__ partial,
    uint8_t* __restrict__ nar_out) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const int64_t ch = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (ch >= F) return;
    const int64_t slice = blockIdx.y, per = (N + slices - 1) / slices;
    const int64_t n0 = slice * per, n1 = min(N, n0 + per);
    const uint32_t nar_code = 1u << (f.nbits - 1);
    // four independent load -> decode chains per step (the row loop is latency bound)
    __int128 acc = 0;
    bool nar = false;
    int64_t n = n0;
    auto term = [&](uint32_t code) -> int64_t {
        int64_t X;
        if (xlut != nullptr) {
            X = __ldg(xlut + code);
            nar |= code == nar_code;
        } else {
            nar |= decode_x(code, f, X);
        }
        return X;
    };
    for (; n + 4 <= n1; n += 4) {
        const uint32_t c0 = uint32_t(dy[n * F + ch]), c1 = uint32_t(dy[(n + 1) * F + ch]);
        const uint32_t c2 = uint32_t(dy[(n + 2) * F + ch]), c3 = uint32_t(dy[(n + 3) * F + ch]);
        const int64_t x0 = term(c0), x1 = term(c1), x2 = term(c2), x3 = term(c3);
        acc += (__int128)x0 + x1 + (__int128)x2 + x3;
    }
    for (; n < n1; ++n) acc += term(uint32_t(dy[n * F + ch]));
    partial[ch * slices + slice] = (unsigned __int128)acc;
    if (nar) nar_out[ch] = 1;
}

template <typename CodeT>
__global__ void __launch_bounds__(256) bias_grad_partial_kernel(
    const CodeT* __restrict__ dy, int64_t N, int64_t F, int64_t P, PositFmt f, int slices,
    const int64_t* __restrict__ xlut, unsigned __int128* __restrict__ partial,
    uint8_t* __restrict__ nar_out) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const int64_t ch = blockIdx.x, slice = blockIdx.y;
    const int64_t per = (N + slices - 1) / slices;
    const int64_t n0 = slice * per, n1 = min(N, n0 + per);
    const uint32_t nar_code = 1u << (f.nbits - 1);
    __int128 acc = 0;
    bool nar = false;
    auto term = [&](uint32_t code) {
        int64_t X;
        if (xlut != nullptr) {  // exact integer image from the per-call table
            X = __ldg(xlut + code);
            nar |= code == nar_code;
        } else {
            nar |= decode_x(code, f, X);
        }
        acc += X;
    };
    constexpr int VE = 16 / int(sizeof(CodeT));  // codes per 16-byte load
    const bool vec = P % VE == 0 && (reinterpret_cast<uintptr_t>(dy) & 15) == 0;
    if (vec) {
        // 16-byte loads over the flattened (image, vector) range of the slice, so
        // every thread works even when P / VE < blockDim (small feature maps)
        const int64_t vpr = P / VE, nv = (n1 - n0) * vpr;
        for (int64_t i = threadIdx.x; i < nv; i += blockDim.x) {
            const int64_t n = n0 + i / vpr, v = i - (n - n0) * vpr;
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(dy + (n * F + ch) * P) + v);
            const uint32_t* ww = reinterpret_cast<const uint32_t*>(&w);
#pragma unroll
            for (int j = 0; j < VE; ++j)
                term(sizeof(CodeT) == 1 ? (ww[j >> 2] >> (8 * (j & 3))) & 0xFFu
                                        : (ww[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
        }
    } else {
        for (int64_t n = n0; n < n1; ++n) {
            const CodeT* row = dy + (n * F + ch) * P;
            for (int o = threadIdx.x; o < int(P); o += blockDim.x) term(uint32_t(row[o]));
        }
    }
    // block reduction: 128-bit butterfly per warp, then one word per warp
    __shared__ unsigned __int128 warp_s[8];
    unsigned __int128 s = (unsigned __int128)acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t l2 = __shfl_xor_sync(0xFFFFFFFFu, uint64_t(s), o);
        const uint64_t h2 = __shfl_xor_sync(0xFFFFFFFFu, uint64_t(s >> 64), o);
        s += (unsigned __int128)l2 | ((unsigned __int128)h2 << 64);
    }
    nar = __syncthreads_or(nar) != 0;
    if ((threadIdx.x & 31) == 0) warp_s[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned __int128 t = 0;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) t += warp_s[i];
        partial[ch * slices + slice] = t;
        if (nar) nar_out[ch] = 1;
    }
}

// P > 1 bias gradient in one launch.  grid (slices, F): block (slice, f) sums
// X over its share of the (image, pixel) range of channel f -- 16-byte loads,
// X from a shared-memory table (LUTB = 1 << nbits entries, formats up to 12
// bits; LUTB = 0 decodes in registers) --, writes one 128-bit partial, and the
// last block of the channel (arrival counter) sums the partials in slice order
// and rounds once: Q = 2^R * sum X (mod 2^W), the reference's
// accumulate_value per term (tensor_ops.cpp:605-618, quire.hpp:62-67).
// GB > 0: dy gated by a ReLU's forward values (gate codes of GB bytes, nbits
// gnbits, same layout): the bias gradient of the ReLU's input gradient
// without materialising it.
template <typename CodeT, int LUTB, int GB = 0>
__global__ void __launch_bounds__(512) bias_grad_chan_kernel(
    const CodeT* __restrict__ dy, int64_t N, int64_t F, int64_t P, PositFmt f, int slices,
    FastDiv fd_vpr, const int64_t* __restrict__ xlut, unsigned __int128* __restrict__ partial,
    uint8_t* __restrict__ nar_flag, unsigned int* __restrict__ arrivals, CodeT* __restrict__ out,
    unsigned __int128* raw_words, uint8_t* raw_nar, const void* __restrict__ gate = nullptr,
    int gnbits = 0) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    __shared__ int64_t s_lut[LUTB];
    __shared__ unsigned __int128 warp_s[16];
    __shared__ bool s_last;
    // the per-call X table (x_lut_kernel) -> shared memory, 16-byte copies
    for (int i = threadIdx.x; i < LUTB / 2; i += blockDim.x)
        reinterpret_cast<int4*>(s_lut)[i] = __ldg(reinterpret_cast<const int4*>(xlut) + i);
    __syncthreads();
    const int64_t ch = blockIdx.y, slice = blockIdx.x;
    const int64_t per = (N + slices - 1) / slices;
    const int64_t n0 = min(N, slice * per), n1 = min(N, n0 + per);  // trailing slices may be empty
    const uint32_t nar_code = 1u << (f.nbits - 1);
    // two independent accumulators of <= 32 terms of |X| <= 2^56 each between
    // flushes into the 128-bit sum (no int64 wrap)
    __int128 acc = 0;
    bool nar = false;
    constexpr int VE = 16 / int(sizeof(CodeT));
    // gate codes of one 16-byte dy vector: VE * GB bytes
    using GV = typename std::conditional<(VE * GB > 8), uint4, uint2>::type;
    auto vsum = [&](const uint4& w, const GV& gv) {
        const uint32_t* ww = reinterpret_cast<const uint32_t*>(&w);
        const uint32_t* gw = reinterpret_cast<const uint32_t*>(&gv);
        int64_t t = 0;
#pragma unroll
        for (int j = 0; j < VE; ++j) {
            const uint32_t code = sizeof(CodeT) == 1 ? (ww[j >> 2] >> (8 * (j & 3))) & 0xFFu
                                                     : (ww[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
            bool open = true;
            if constexpr (GB > 0) {
                const uint32_t g = GB == 1 ? (gw[j >> 2] >> (8 * (j & 3))) & 0xFFu
                                           : (gw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
                open = g != 0 && ((g >> (gnbits - 1)) & 1u) == 0;
            }
            if (open) {
                t += s_lut[code];
                nar |= code == nar_code;
            }
        }
        return t;  // |t| <= 16 * 2^56
    };
    const uint32_t vpr = uint32_t(P / VE), nv = uint32_t((n1 - n0) * vpr);
    const CodeT* base = dy + (n0 * F + ch) * P;
    const int64_t img_stride = F * P;
    auto gload = [&](uint32_t q, uint32_t r) {
        GV g{};
        if constexpr (GB > 0)
            g = __ldg(reinterpret_cast<const GV*>(static_cast<const uint8_t*>(gate) +
                                                  ((n0 * F + ch) * P + q * img_stride) * GB) + r);
        return g;
    };
    uint32_t i = threadIdx.x;
    // four 16-byte loads in flight per thread (the loop is load-latency bound)
    for (; i + 3 * blockDim.x < nv; i += 4 * blockDim.x) {
        uint32_t q0, r0, q1, r1, q2, r2, q3, r3;
        fd_vpr.divmod(i, q0, r0);
        fd_vpr.divmod(i + blockDim.x, q1, r1);
        fd_vpr.divmod(i + 2 * blockDim.x, q2, r2);
        fd_vpr.divmod(i + 3 * blockDim.x, q3, r3);
        const uint4 w0 = __ldg(reinterpret_cast<const uint4*>(base + q0 * img_stride) + r0);
        const uint4 w1 = __ldg(reinterpret_cast<const uint4*>(base + q1 * img_stride) + r1);
        const uint4 w2 = __ldg(reinterpret_cast<const uint4*>(base + q2 * img_stride) + r2);
        const uint4 w3 = __ldg(reinterpret_cast<const uint4*>(base + q3 * img_stride) + r3);
        const GV g0 = gload(q0, r0), g1 = gload(q1, r1), g2 = gload(q2, r2), g3 = gload(q3, r3);
        acc += vsum(w0, g0) + vsum(w1, g1);  // 2 * 16 * 2^56 < 2^62
        acc += vsum(w2, g2) + vsum(w3, g3);
    }
    for (; i + blockDim.x < nv; i += 2 * blockDim.x) {
        uint32_t q0, r0, q1, r1;
        fd_vpr.divmod(i, q0, r0);
        fd_vpr.divmod(i + blockDim.x, q1, r1);
        const uint4 w0 = __ldg(reinterpret_cast<const uint4*>(base + q0 * img_stride) + r0);
        const uint4 w1 = __ldg(reinterpret_cast<const uint4*>(base + q1 * img_stride) + r1);
        const GV g0 = gload(q0, r0), g1 = gload(q1, r1);
        acc += vsum(w0, g0) + vsum(w1, g1);  // 2 * 16 * 2^56 < 2^62
    }
    if (i < nv) {
        uint32_t q0, r0;
        fd_vpr.divmod(i, q0, r0);
        acc += vsum(__ldg(reinterpret_cast<const uint4*>(base + q0 * img_stride) + r0), gload(q0, r0));
    }
    unsigned __int128 sum = (unsigned __int128)acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t l2 = __shfl_xor_sync(0xFFFFFFFFu, uint64_t(sum), o);
        const uint64_t h2 = __shfl_xor_sync(0xFFFFFFFFu, uint64_t(sum >> 64), o);
        sum += (unsigned __int128)l2 | ((unsigned __int128)h2 << 64);
    }
    nar = __syncthreads_or(nar) != 0;
    if ((threadIdx.x & 31) == 0) warp_s[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned __int128 t = 0;
        for (int k = 0; k < int(blockDim.x >> 5); ++k) t += warp_s[k];
        partial[ch * slices + slice] = t;
        if (nar) nar_flag[ch] = 1;
        __threadfence();
        s_last = atomicAdd(&arrivals[ch], 1u) == unsigned(slices - 1);
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    const volatile unsigned __int128* vp = partial + ch * slices;
    unsigned __int128 tot = 0;
    for (int k = 0; k < slices; ++k) tot += vp[k];
    const bool any_nar = *reinterpret_cast<volatile uint8_t*>(nar_flag + ch) != 0;
    const unsigned __int128 one = 1;
    const unsigned __int128 wmask = f.W >= 128 ? ~(unsigned __int128)0 : ((one << f.W) - 1);
    const unsigned __int128 q = (tot << f.R) & wmask;  // accumulate_value: X * 2^R
    if (raw_words) {
        raw_words[ch] = q;
        raw_nar[ch] = any_nar;
    }
    if (out) out[ch] = CodeT(any_nar ? nar_code : quire_word_to_posit(f, q));
    arrivals[ch] = 0;  // ready for the next call (graph replays)
}

// X (the exact integer image) of every code of a format, for table decode.
__global__ void x_lut_kernel(PositFmt f, int64_t* __restrict__ lut) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < (1 << f.nbits)) {
        int64_t X;
        decode_x(uint32_t(c), f, X);
        lut[c] = X;
    }
}

// the X table of a format for the life of the process (tables.h), else the
// per-call table in the workspace
inline int64_t* x_table(const PositFmt& f, int64_t* ws_lut, cudaStream_t st) {
    void* p = persistent_table(table_key(2, f.nbits, f.es, 0, 0, 0), (size_t(1) << f.nbits) * 8, st,
                               [&](void* q, cudaStream_t s) {
                                   x_lut_kernel<<<(1 << f.nbits) / 256 + 1, 256, 0, s>>>(f, static_cast<int64_t*>(q));
                               });
    if (p) return static_cast<int64_t*>(p);
    x_lut_kernel<<<(1 << f.nbits) / 256 + 1, 256, 0, st>>>(f, ws_lut);
    return ws_lut;
}

template <typename CodeT>
__global__ void bias_grad_final_kernel(const unsigned __int128* __restrict__ partial, int slices,
                                       const uint8_t* __restrict__ nar_in, int64_t F, PositFmt f,
                                       CodeT* __restrict__ out, unsigned __int128* raw_words,
                                       uint8_t* raw_nar) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    // a warp per channel: lanes sum interleaved partials (coalesced 16-byte
    // loads), then a shuffle tree; exact 128-bit integer sums in any order
    const unsigned __int128 one = 1;
    const unsigned __int128 wmask = f.W >= 128 ? ~(unsigned __int128)0 : ((one << f.W) - 1);
    const int lane = threadIdx.x & 31;
    for (int64_t ch = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; ch < F;
         ch += (int64_t(gridDim.x) * blockDim.x) >> 5) {
        unsigned __int128 s = 0;
        for (int i = lane; i < slices; i += 32) s += partial[ch * slices + i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t l2 = __shfl_xor_sync(0xFFFFFFFFu, uint64_t(s), o);
            const uint64_t h2 = __shfl_xor_sync(0xFFFFFFFFu, uint64_t(s >> 64), o);
            s += (unsigned __int128)l2 | ((unsigned __int128)h2 << 64);
        }
        if (lane != 0) continue;
        const unsigned __int128 q = (s << f.R) & wmask;  // accumulate_value: X * 2^R
        if (raw_words) {
            raw_words[ch] = q;
            raw_nar[ch] = nar_in[ch];
        }
        if (out) out[ch] = CodeT(nar_in[ch] ? (1u << (f.nbits - 1)) : quire_word_to_posit(f, q));
    }
}

}  // namespace pnn_b200

// =========================================================================
// C-ABI
// =========================================================================

using namespace pnn_b200;

namespace {

bool conv_fmt_ok(int nbits, int es) {
    if (nbits < 2 || nbits > 16 || es < 0 || es > 4) return false;
    return 2 * make_fmt(nbits, es).R <= 56;
}

int conv_geom(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int64_t KH, int64_t KW,
              int stride, int pad, ConvGeom* g) {
    if (N < 0 || C < 1 || H < 1 || W < 1 || F < 1 || KH < 1 || KW < 1 || stride < 1 || pad < 0)
        return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if (H + 2 * pad < KH || W + 2 * pad < KW) return set_status(PNN_EINVAL, "conv: invalid shape or argument");  // tensor_ops.cpp:215
    g->N = N; g->C = C; g->H = H; g->W = W; g->F = F; g->KH = KH; g->KW = KW;
    g->stride = stride;
    g->pad = pad;
    g->OH = (H + 2 * pad - KH) / stride + 1;
    g->OW = (W + 2 * pad - KW) / stride + 1;
    return PNN_OK;
}

// Logical GEMM sizes per pass.
void pass_dims(int pass, const ConvGeom& g, bool has_bias, int64_t* M, int64_t* Nn, int64_t* K) {
    const int64_t kconv = g.C * g.KH * g.KW;
    if (pass == 0) {
        *M = g.N * g.OH * g.OW; *Nn = g.F; *K = kconv + (has_bias ? 1 : 0);
    } else if (pass == 1) {
        *M = g.N * g.H * g.W; *Nn = g.C; *K = g.F * g.KH * g.KW;
    } else {
        *M = kconv; *Nn = g.F; *K = g.N * g.OH * g.OW;
    }
}

int status_of(int rc, const char* what) {
    if (rc == 0) return PNN_OK;
    set_last_error(std::string(what) + (rc == 2 ? ": format not supported"
                                        : rc == 3 ? ": workspace too small"
                                                  : ": CUDA launch failed"));
    return rc == 2 ? PNN_EUNSUPPORTED : rc == 3 ? PNN_EWORKSPACE : PNN_ECUDA;
}

uint32_t one_code(const PositFmt& f) { return 1u << (f.nbits - 2); }  // 0b01000.. = 1.0

// ---- Linear layers (1x1 kernels over 1x1 images: plain matrices) -----------
// x [N][C], w [F][C], y/dy [N][F]: the explicit path's operands are row- or
// column-major matrices, packed with 16-byte vector loads instead of the
// im2col gathers (same X[r][k] values, so the same results).

bool is_linear(const ConvGeom& g) {
    return g.H == 1 && g.W == 1 && g.KH == 1 && g.KW == 1 && g.stride == 1 && g.pad == 0;
}

// X[r][k] = p[r*C + k] for k < C; column C = the bias column (col[r] or cval)
template <typename CodeT>
struct FetchRowsBias {
    const CodeT* p;
    int64_t C;
    const CodeT* col;  // per-row bias codes (weights) or null
    uint32_t cval;     // constant bias column (activations: the code of 1.0)
    static constexpr bool kRowFastest = false;
    static constexpr bool kVecK = true, kVecR = false, kSep = false;
    __device__ __forceinline__ const CodeT* ptr(int64_t r, int64_t k) const {
        return k + int64_t(16 / sizeof(CodeT)) <= C ? p + r * C + k : nullptr;  // never spans the bias
    }
    __device__ __forceinline__ uint32_t operator()(int64_t r, int64_t k) const {
        return k < C ? uint32_t(p[r * C + k]) : (col ? uint32_t(col[r]) : cval);
    }
};

template <typename T>
int linear_fwd(GemmArgs& a, const ConvGeom& g, const void* x, const void* w, const void* bias, void* y,
               void* ws, size_t wsb, cudaStream_t st) {
    return run_quire_gemm<T>(a, FetchRowsBias<T>{(const T*)x, g.C, nullptr, one_code(a.f)},
                             FetchRowsBias<T>{(const T*)w, g.C, (const T*)bias, 0u},
                             out_nchw<T>(y, 1, g.F), ws, wsb, st, nullptr);
}

template <typename T>
int linear_dgrad(GemmArgs& a, const ConvGeom& g, const void* dy, const void* w, void* dx, void* ws,
                 size_t wsb, cudaStream_t st) {
    // dx[n][c] = sum_f dy[n][f] w[f][c]: A = dy row-major, B[r = c][k = f] = w[f][c]
    return run_quire_gemm<T>(a, FetchRowMajor<T>{(const T*)dy, g.F}, FetchColMajor<T>{(const T*)w, g.C},
                             out_nchw<T>(dx, 1, g.C), ws, wsb, st, nullptr);
}

template <typename T>
int linear_wgrad(GemmArgs& a, const ConvGeom& g, const void* dy, const void* x, void* dw, void* ws,
                 size_t wsb, cudaStream_t st) {
    // dw[f][c] = sum_n dy[n][f] x[n][c]: A[r = c][k = n] = x[n][c], B[r = f][k = n] = dy[n][f]
    return run_quire_gemm<T>(a, FetchColMajor<T>{(const T*)x, g.C}, FetchColMajor<T>{(const T*)dy, g.F},
                             out_nchw<T>(dw, a.M, g.F), ws, wsb, st, nullptr);
}

}  // namespace

extern "C" {

int pnn_conv2d_workspace(int pass, int nbits, int es, int64_t N, int64_t C, int64_t H, int64_t W,
                         int64_t F, int64_t KH, int64_t KW, int stride, int pad, int has_bias,
                         size_t* bytes) {
    if (!conv_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "conv: format not supported");
    ConvGeom g;
    if (!bytes || pass < 0 || pass > 2 || conv_geom(N, C, H, W, F, KH, KW, stride, pad, &g))
        return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    int64_t M, Nn, K;
    pass_dims(pass, g, has_bias != 0, &M, &Nn, &K);
    if (M == 0 || K == 0) {
        *bytes = 0;
        return PNN_OK;
    }
    if (igemm_eligible(pass, make_fmt(nbits, es), g, pass == 2, bytes)) return PNN_OK;
    if (conv_algo() == 2) return set_status(PNN_EUNSUPPORTED, "conv: implicit path not eligible");
    QuireGemmPlan p;
    if (plan_quire_gemm(make_fmt(nbits, es), M, Nn, K, 0, pass == 2, &p)) return PNN_EUNSUPPORTED;
    *bytes = p.workspace_bytes;
    return PNN_OK;
}

int pnn_conv2d_fwd(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H, int64_t W,
                   const void* w, int64_t F, int64_t KH, int64_t KW, const void* bias, int stride,
                   int pad, void* y, void* workspace, size_t workspace_bytes, void* stream) {
    if (!conv_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "conv: format not supported");
    ConvGeom g;
    if (conv_geom(N, C, H, W, F, KH, KW, stride, pad, &g) || !x || !w || !y) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if (N == 0) return PNN_OK;
    GemmArgs a;
    a.f = make_fmt(nbits, es);
    pass_dims(0, g, bias != nullptr, &a.M, &a.N, &a.K);
    a.max_kb_per_split = 0;
    a.row_nar = a.col_nar = true;
    const int64_t kconv = C * KH * KW;
    auto st = static_cast<cudaStream_t>(stream);
    int rc;
    if (igemm_eligible(0, a.f, g, false, nullptr))
        return status_of(igemm_conv_fwd(a.f, g, x, w, bias, y, workspace, workspace_bytes, st),
                         "conv2d_fwd");
    if (conv_algo() == 2) return set_status(PNN_EUNSUPPORTED, "conv2d_fwd: implicit path not eligible");
    if (is_linear(g))
        return status_of(nbits <= 8 ? linear_fwd<uint8_t>(a, g, x, w, bias, y, workspace, workspace_bytes, st)
                                    : linear_fwd<uint16_t>(a, g, x, w, bias, y, workspace, workspace_bytes, st),
                         "conv2d_fwd");
    if (nbits <= 8) {
        using T = uint8_t;
        rc = run_quire_gemm<T>(a, FetchIm2colFwd<T>{(const T*)x, g, kconv, one_code(a.f)},
                               FetchWeightFwd<T>{(const T*)w, (const T*)bias, kconv},
                               out_nchw<T>(y, g.OH * g.OW, F), workspace, workspace_bytes, st,
                               nullptr);
    } else {
        using T = uint16_t;
        rc = run_quire_gemm<T>(a, FetchIm2colFwd<T>{(const T*)x, g, kconv, one_code(a.f)},
                               FetchWeightFwd<T>{(const T*)w, (const T*)bias, kconv},
                               out_nchw<T>(y, g.OH * g.OW, F), workspace, workspace_bytes, st,
                               nullptr);
    }
    return status_of(rc, "conv2d_fwd");
}

int pnn_conv2d_dgrad(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t OH,
                     int64_t OW, const void* w, int64_t C, int64_t KH, int64_t KW, int64_t H,
                     int64_t W, int stride, int pad, void* dx, void* workspace,
                     size_t workspace_bytes, void* stream) {
    if (!conv_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "conv: format not supported");
    ConvGeom g;
    if (conv_geom(N, C, H, W, F, KH, KW, stride, pad, &g) || !dy || !w || !dx) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if (g.OH != OH || g.OW != OW) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if (N == 0) return PNN_OK;
    GemmArgs a;
    a.f = make_fmt(nbits, es);
    pass_dims(1, g, false, &a.M, &a.N, &a.K);
    a.max_kb_per_split = 0;
    a.row_nar = true;
    a.col_nar = false;  // weight NaR applied per valid tap below
    auto st = static_cast<cudaStream_t>(stream);
    if (igemm_eligible(1, a.f, g, false, nullptr))
        return status_of(igemm_conv_dgrad(a.f, g, dy, w, dx, workspace, workspace_bytes, st),
                         "conv2d_dgrad");
    if (conv_algo() == 2) return set_status(PNN_EUNSUPPORTED, "conv2d_dgrad: implicit path not eligible");
    if (is_linear(g)) {  // every tap valid: weight-column NaR is the B-column flag
        a.col_nar = true;
        return status_of(nbits <= 8 ? linear_dgrad<uint8_t>(a, g, dy, w, dx, workspace, workspace_bytes, st)
                                    : linear_dgrad<uint16_t>(a, g, dy, w, dx, workspace, workspace_bytes, st),
                         "conv2d_dgrad");
    }
    QuireGemmPlan p;
    if (plan_quire_gemm(a.f, a.M, a.N, a.K, 0, false, &p)) return PNN_EUNSUPPORTED;
    const uint8_t* flag_w = static_cast<const uint8_t*>(workspace) + p.off_flags + 1;
    int rc;
    const uint32_t nar = 1u << (nbits - 1);
    const int64_t total = N * C * H * W;
    if (nbits <= 8) {
        using T = uint8_t;
        rc = run_quire_gemm<T>(a, FetchDgradDy<T>{(const T*)dy, g}, FetchDgradW<T>{(const T*)w, g},
                               out_nchw<T>(dx, H * W, C), workspace, workspace_bytes, st, nullptr);
        if (rc == 0)
            launch_pdl(dgrad_weight_nar_kernel<T>, dim3(grid_fixup(total)), dim3(256), 0, st, (T*)dx, (const T*)w, g,
                                                                             flag_w, nar);
    } else {
        using T = uint16_t;
        rc = run_quire_gemm<T>(a, FetchDgradDy<T>{(const T*)dy, g}, FetchDgradW<T>{(const T*)w, g},
                               out_nchw<T>(dx, H * W, C), workspace, workspace_bytes, st, nullptr);
        if (rc == 0)
            launch_pdl(dgrad_weight_nar_kernel<T>, dim3(grid_fixup(total)), dim3(256), 0, st, (T*)dx, (const T*)w, g,
                                                                             flag_w, nar);
    }
    if (rc == 0 && cudaGetLastError() != cudaSuccess) rc = 4;
    return status_of(rc, "conv2d_dgrad");
}

int pnn_conv2d_wgrad(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t OH,
                     int64_t OW, const void* x, int64_t C, int64_t H, int64_t W, int64_t KH,
                     int64_t KW, int stride, int pad, void* dw, void* raw_words, void* raw_nar,
                     void* workspace, size_t workspace_bytes, void* stream) {
    if (!conv_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "conv: format not supported");
    ConvGeom g;
    if (conv_geom(N, C, H, W, F, KH, KW, stride, pad, &g) || !dy || !x) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if (g.OH != OH || g.OW != OW) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if (!dw && !raw_words) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if ((raw_words != nullptr) != (raw_nar != nullptr)) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    GemmArgs a;
    a.f = make_fmt(nbits, es);
    pass_dims(2, g, false, &a.M, &a.N, &a.K);
    auto st = static_cast<cudaStream_t>(stream);
    if (a.K == 0) {  // empty batch: all-zero gradient
        if (dw) cudaMemsetAsync(dw, 0, size_t(a.M * a.N) * (nbits <= 8 ? 1 : 2), st);
        if (raw_words) {
            cudaMemsetAsync(raw_words, 0, size_t(a.M * a.N) * 16, st);
            cudaMemsetAsync(raw_nar, 0, size_t(a.M * a.N), st);
        }
        return PNN_OK;
    }
    a.max_kb_per_split = 0;
    a.row_nar = a.col_nar = true;
    a.raw_words = static_cast<unsigned __int128*>(raw_words);
    a.raw_nar = static_cast<uint8_t*>(raw_nar);
    if (igemm_eligible(2, a.f, g, raw_words != nullptr, nullptr))
        return status_of(igemm_conv_wgrad(a.f, g, dy, x, dw, a.raw_words, a.raw_nar, workspace,
                                          workspace_bytes, st),
                         "conv2d_wgrad");
    if (conv_algo() == 2) return set_status(PNN_EUNSUPPORTED, "conv2d_wgrad: implicit path not eligible");
    if (is_linear(g))
        return status_of(nbits <= 8 ? linear_wgrad<uint8_t>(a, g, dy, x, dw, workspace, workspace_bytes, st)
                                    : linear_wgrad<uint16_t>(a, g, dy, x, dw, workspace, workspace_bytes, st),
                         "conv2d_wgrad");
    // dw[f][(c,ky,kx)]: output (m=(c,ky,kx), n=f) -> f*M + m  (NCHW map with one "image")
    int rc;
    if (nbits <= 8) {
        using T = uint8_t;
        rc = run_quire_gemm<T>(a, FetchWgradX<T>{(const T*)x, g}, FetchWgradDy<T>{(const T*)dy, g},
                               out_nchw<T>(dw, a.M, F), workspace, workspace_bytes, st, nullptr);
    } else {
        using T = uint16_t;
        rc = run_quire_gemm<T>(a, FetchWgradX<T>{(const T*)x, g}, FetchWgradDy<T>{(const T*)dy, g},
                               out_nchw<T>(dw, a.M, F), workspace, workspace_bytes, st, nullptr);
    }
    return status_of(rc, "conv2d_wgrad");
}

// ---- layer-level pair: forward keeping x's digits, fused backward ----------

int pnn_conv2d_saved_bytes(int nbits, int es, int64_t N, int64_t C, int64_t H, int64_t W, int64_t F,
                           int64_t KH, int64_t KW, int stride, int pad, size_t* bytes) {
    if (!conv_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "conv: format not supported");
    ConvGeom g;
    if (!bytes || conv_geom(N, C, H, W, F, KH, KW, stride, pad, &g))
        return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    *bytes = N > 0 ? igemm_saved_bytes(make_fmt(nbits, es), g) : 0;
    return PNN_OK;
}

int pnn_conv2d_fwd_save(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H, int64_t W,
                        const void* w, int64_t F, int64_t KH, int64_t KW, const void* bias, int stride,
                        int pad, void* y, void* saved, size_t saved_bytes, void* workspace,
                        size_t workspace_bytes, void* stream) {
    return pnn_conv2d_fwd_layer(nbits, es, x, N, C, H, W, w, F, KH, KW, bias, stride, pad, 0, y, nullptr,
                                saved, saved_bytes, workspace, workspace_bytes, stream);
}

int pnn_conv2d_fwd_layer(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H, int64_t W,
                         const void* w, int64_t F, int64_t KH, int64_t KW, const void* bias, int stride,
                         int pad, int relu, void* y, void* y_pre, void* saved, size_t saved_bytes,
                         void* workspace, size_t workspace_bytes, void* stream) {
    if (saved == nullptr && !relu)
        return pnn_conv2d_fwd(nbits, es, x, N, C, H, W, w, F, KH, KW, bias, stride, pad, y, workspace,
                              workspace_bytes, stream);
    if (!conv_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "conv: format not supported");
    ConvGeom g;
    if (conv_geom(N, C, H, W, F, KH, KW, stride, pad, &g) || !x || !w || !y)
        return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if (N == 0) return PNN_OK;
    const PositFmt f = make_fmt(nbits, es);
    if (saved != nullptr && igemm_saved_bytes(f, g) == 0)
        return set_status(PNN_EUNSUPPORTED, "conv2d_fwd_save: no implicit forward/weight-grad pair");
    if (!igemm_eligible(0, f, g, false, nullptr))
        return set_status(PNN_EUNSUPPORTED, "conv2d_fwd_layer: implicit forward not eligible");
    return status_of(igemm_conv_fwd(f, g, x, w, bias, y, workspace, workspace_bytes,
                                    static_cast<cudaStream_t>(stream), saved, saved_bytes, relu, y_pre),
                     "conv2d_fwd_layer");
}

int pnn_conv2d_backward_workspace(int f_nbits, int f_es, int b_nbits, int b_es, int g_nbits, int g_es,
                                  int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int64_t KH,
                                  int64_t KW, int stride, int pad, int raw, int has_dx, int has_saved,
                                  size_t* bytes) {
    if (!conv_fmt_ok(f_nbits, f_es) || !conv_fmt_ok(b_nbits, b_es) || !conv_fmt_ok(g_nbits, g_es))
        return set_status(PNN_EUNSUPPORTED, "conv: format not supported");
    ConvGeom g;
    if (!bytes || N < 1 || conv_geom(N, C, H, W, F, KH, KW, stride, pad, &g))
        return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if (!igemm_backward_eligible(make_fmt(f_nbits, f_es), make_fmt(b_nbits, b_es), make_fmt(g_nbits, g_es),
                                 g, raw != 0, has_dx != 0, has_saved != 0, bytes))
        return set_status(PNN_EUNSUPPORTED, "conv2d_backward: not eligible (use the per-pass calls)");
    return PNN_OK;
}

int pnn_conv2d_backward(int f_nbits, int f_es, int b_nbits, int b_es, int g_nbits, int g_es,
                        const void* dy, const void* x, const void* saved, size_t saved_bytes,
                        const void* w_bwd, int64_t N, int64_t C, int64_t H, int64_t W, int64_t F,
                        int64_t KH, int64_t KW, int stride, int pad, void* dx, void* dw,
                        void* raw_words, void* raw_nar, void* workspace, size_t workspace_bytes,
                        void* stream) {
    return pnn_conv2d_backward_gated(f_nbits, f_es, b_nbits, b_es, g_nbits, g_es, dy, nullptr, nullptr, x,
                                     saved, saved_bytes, w_bwd, N, C, H, W, F, KH, KW, stride, pad, dx, dw,
                                     raw_words, raw_nar, workspace, workspace_bytes, stream);
}

int pnn_conv2d_backward_gated(int f_nbits, int f_es, int b_nbits, int b_es, int g_nbits, int g_es,
                              const void* dy, const void* gate, void* dy_gated, const void* x,
                              const void* saved, size_t saved_bytes, const void* w_bwd, int64_t N,
                              int64_t C, int64_t H, int64_t W, int64_t F, int64_t KH, int64_t KW,
                              int stride, int pad, void* dx, void* dw, void* raw_words, void* raw_nar,
                              void* workspace, size_t workspace_bytes, void* stream) {
    if (!conv_fmt_ok(f_nbits, f_es) || !conv_fmt_ok(b_nbits, b_es) || !conv_fmt_ok(g_nbits, g_es))
        return set_status(PNN_EUNSUPPORTED, "conv: format not supported");
    ConvGeom g;
    if (N < 1 || conv_geom(N, C, H, W, F, KH, KW, stride, pad, &g) || !dy || (!x && !saved))
        return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if ((!dw && !raw_words) || ((raw_words != nullptr) != (raw_nar != nullptr)) || (dx && !w_bwd))
        return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    return status_of(igemm_conv_backward(make_fmt(f_nbits, f_es), make_fmt(b_nbits, b_es),
                                         make_fmt(g_nbits, g_es), g, dy, x, saved, saved_bytes, w_bwd, dx,
                                         dw, static_cast<unsigned __int128*>(raw_words),
                                         static_cast<uint8_t*>(raw_nar), workspace, workspace_bytes,
                                         static_cast<cudaStream_t>(stream), gate, f_nbits, dy_gated),
                     "conv2d_backward");
}

// workspace: [split partials F x 64 x 16 B][NaR flags F][X table of the format]
constexpr int kBiasLutBits = 12;
static size_t bias_lut_offset(int64_t F) {
    return (size_t(F) * 16 * 64 + size_t(F) + 255) & ~size_t(255);
}

static size_t bias_arrivals_offset(int64_t F) { return bias_lut_offset(F) + (size_t(8) << kBiasLutBits); }

int pnn_bias_grad_workspace(int64_t F, size_t* bytes) {
    if (F < 0 || !bytes) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    *bytes = bias_arrivals_offset(F) + size_t(F) * 4;
    return PNN_OK;
}

int pnn_bias_grad_gated(int nbits, int es, const void* dy, int gate_nbits, const void* gate, int64_t N,
                        int64_t F, int64_t P, void* db, void* raw_words, void* raw_nar, void* workspace,
                        size_t workspace_bytes, void* stream) {
    if (!conv_fmt_ok(nbits, es) || gate_nbits < 2 || gate_nbits > 16)
        return set_status(PNN_EUNSUPPORTED, "conv: format not supported");
    if (N < 1 || F < 1 || P < 1 || !dy || !gate || (!db && !raw_words))
        return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if ((raw_words != nullptr) != (raw_nar != nullptr)) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    const int VE = nbits <= 8 ? 16 : 8, GB = gate_nbits <= 8 ? 1 : 2;
    if (nbits > kBiasLutBits || P % VE || (reinterpret_cast<uintptr_t>(dy) & 15) ||
        (reinterpret_cast<uintptr_t>(gate) & 15) || (nbits <= 8 && GB == 2))
        return set_status(PNN_EUNSUPPORTED, "bias_grad_gated: table formats, 16-byte rows");
    size_t need;
    pnn_bias_grad_workspace(F, &need);
    if (workspace_bytes < need) return PNN_EWORKSPACE;
    const PositFmt f = make_fmt(nbits, es);
    auto* partial = static_cast<unsigned __int128*>(workspace);
    auto* nar = static_cast<uint8_t*>(workspace) + size_t(F) * 16 * 64;
    auto* arrivals = reinterpret_cast<unsigned int*>(static_cast<uint8_t*>(workspace) + bias_arrivals_offset(F));
    auto* lut = reinterpret_cast<int64_t*>(static_cast<uint8_t*>(workspace) + bias_lut_offset(F));
    auto st = static_cast<cudaStream_t>(stream);
    cudaMemsetAsync(nar, 0, size_t(F), st);
    cudaMemsetAsync(arrivals, 0, size_t(F) * 4, st);
    lut = x_table(f, lut, st);
    int64_t want = (int64_t(2) * 148 + F - 1) / F;  // ~2 blocks of 512 per SM: the X table loads once per block
    int sl = int(want > 64 ? 64 : want);
    if (sl > N) sl = int(N);
    const int64_t per = (N + sl - 1) / sl;
    if (per * P / VE >= (int64_t(1) << 31)) return set_status(PNN_EUNSUPPORTED, "bias_grad_gated: size");
    const FastDiv fd{uint32_t(P / VE)};
    const dim3 g2{unsigned(sl), unsigned(F), 1u};
#define PNN_BGG(T, B, G)                                                                              \
    launch_pdl(bias_grad_chan_kernel<T, B, G>, dim3(g2), dim3(512), 0, st, (const T*)dy, N, F, P, f, sl, fd, lut, partial,  \
                                                       nar, arrivals, (T*)db,                          \
                                                       (unsigned __int128*)raw_words, (uint8_t*)raw_nar, \
                                                       gate, gate_nbits)
    if (nbits <= 8) PNN_BGG(uint8_t, 256, 1);
    else if (nbits <= 10 && GB == 1) PNN_BGG(uint16_t, 1024, 1);
    else if (nbits <= 10) PNN_BGG(uint16_t, 1024, 2);
    else if (GB == 1) PNN_BGG(uint16_t, 4096, 1);
    else PNN_BGG(uint16_t, 4096, 2);
#undef PNN_BGG
    return cudaGetLastError() == cudaSuccess ? PNN_OK : PNN_ECUDA;
}

int pnn_bias_grad(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t P, void* db,
                  void* raw_words, void* raw_nar, void* workspace, size_t workspace_bytes,
                  void* stream) {
    if (!conv_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "conv: format not supported");
    if (N < 0 || F < 1 || P < 1 || !dy || (!db && !raw_words)) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    if ((raw_words != nullptr) != (raw_nar != nullptr)) return set_status(PNN_EINVAL, "conv: invalid shape or argument");
    size_t need;
    pnn_bias_grad_workspace(F, &need);
    if (workspace_bytes < need) return PNN_EWORKSPACE;
    const PositFmt f = make_fmt(nbits, es);
    int slices = int(N < 64 ? (N < 1 ? 1 : N) : 64);
    auto* partial = static_cast<unsigned __int128*>(workspace);
    auto* nar = static_cast<uint8_t*>(workspace) + size_t(F) * 16 * 64;
    auto st = static_cast<cudaStream_t>(stream);
    cudaMemsetAsync(nar, 0, size_t(F), st);
    // single-launch path below: table-decoded formats, 16-byte rows
    const bool chan = P > 1 && nbits <= kBiasLutBits && P % (nbits <= 8 ? 16 : 8) == 0 &&
                      (reinterpret_cast<uintptr_t>(dy) & 15) == 0;
    if (!chan) cudaMemsetAsync(partial, 0, size_t(F) * 16 * slices, st);
    const dim3 grid{unsigned(F), unsigned(slices), 1u};
    int64_t* xlut = nullptr;
    if (!chan && nbits <= kBiasLutBits && N * P >= 4096) {  // table pays for itself
        xlut = x_table(f, reinterpret_cast<int64_t*>(static_cast<uint8_t*>(workspace) + bias_lut_offset(F)), st);
    }
    const dim3 cgrid{unsigned((F + 255) / 256), unsigned(slices), 1u};
    if (P == 1 && nbits <= 8) {
        launch_pdl(bias_grad_cols_kernel<uint8_t>, dim3(cgrid), dim3(256), 0, st, (const uint8_t*)dy, N, F, f, slices,
                                                              xlut, partial, nar);
        launch_pdl(bias_grad_final_kernel<uint8_t>, dim3(grid_for(F * 32, 256)), dim3(256), 0, st, 
            partial, slices, nar, F, f, (uint8_t*)db, (unsigned __int128*)raw_words,
            (uint8_t*)raw_nar);
    } else if (P == 1) {
        launch_pdl(bias_grad_cols_kernel<uint16_t>, dim3(cgrid), dim3(256), 0, st, (const uint16_t*)dy, N, F, f,
                                                               slices, xlut, partial, nar);
        launch_pdl(bias_grad_final_kernel<uint16_t>, dim3(grid_for(F * 32, 256)), dim3(256), 0, st, 
            partial, slices, nar, F, f, (uint16_t*)db, (unsigned __int128*)raw_words,
            (uint8_t*)raw_nar);
    } else if (chan) {
        // channel-uniform blocks, X table in shared memory, last-block rounding;
        // >= 8 blocks per SM, each at least one image
        auto* arrivals = reinterpret_cast<unsigned int*>(static_cast<uint8_t*>(workspace) +
                                                         bias_arrivals_offset(F));
        auto* lut = reinterpret_cast<int64_t*>(static_cast<uint8_t*>(workspace) + bias_lut_offset(F));
        cudaMemsetAsync(arrivals, 0, size_t(F) * 4, st);
        lut = x_table(f, lut, st);
        int64_t want = (int64_t(2) * 148 + F - 1) / F;  // ~2 blocks of 512 per SM: the X table loads once per block
        int sl = int(want > 64 ? 64 : want);
        if (sl > N) sl = int(N < 1 ? 1 : N);
        const int VE = nbits <= 8 ? 16 : 8;
        const int64_t per = (N + sl - 1) / sl;
        if (P % VE || per * P / VE >= (int64_t(1) << 31) || (reinterpret_cast<uintptr_t>(dy) & 15))
            return set_status(PNN_EUNSUPPORTED, "bias_grad: unaligned rows");
        const FastDiv fd{uint32_t(P / VE)};
        const dim3 g2{unsigned(sl), unsigned(F), 1u};
#define PNN_BGC(T, B)                                                                             \
    launch_pdl(bias_grad_chan_kernel<T, B>, dim3(g2), dim3(512), 0, st, (const T*)dy, N, F, P, f, sl, fd, lut, partial, \
                                                    nar, arrivals, (T*)db,                        \
                                                    (unsigned __int128*)raw_words, (uint8_t*)raw_nar, \
                                                    static_cast<const void*>(nullptr), 0)
        if (nbits <= 8) PNN_BGC(uint8_t, 256);
        else if (nbits <= 10) PNN_BGC(uint16_t, 1024);
        else PNN_BGC(uint16_t, 4096);
#undef PNN_BGC
    } else if (nbits <= 8) {
        launch_pdl(bias_grad_partial_kernel<uint8_t>, dim3(grid), dim3(256), 0, st, (const uint8_t*)dy, N, F, P, f,
                                                                 slices, xlut, partial, nar);
        launch_pdl(bias_grad_final_kernel<uint8_t>, dim3(grid_for(F * 32, 256)), dim3(256), 0, st, 
            partial, slices, nar, F, f, (uint8_t*)db, (unsigned __int128*)raw_words,
            (uint8_t*)raw_nar);
    } else {
        launch_pdl(bias_grad_partial_kernel<uint16_t>, dim3(grid), dim3(256), 0, st, (const uint16_t*)dy, N, F, P, f,
                                                                  slices, xlut, partial, nar);
        launch_pdl(bias_grad_final_kernel<uint16_t>, dim3(grid_for(F * 32, 256)), dim3(256), 0, st, 
            partial, slices, nar, F, f, (uint16_t*)db, (unsigned __int128*)raw_words,
            (uint8_t*)raw_nar);
    }
    return cudaGetLastError() == cudaSuccess ? PNN_OK : PNN_ECUDA;
}

}  // extern "C"
