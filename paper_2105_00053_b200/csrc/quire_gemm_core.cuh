// Exact posit-quire GEMM core on the 5th-gen tensor cores (tcgen05 kind::i8).
// Templated on operand-fetch functors and an output map, so the matmul, the
// Conv2d forward / input-grad / weight-grad and the Linear passes all run
// through the same pack -> tcgen05 -> epilogue pipeline (implicit GEMM with
// the im2col gather done once per element in the pack stage).
//
// Replaces matmul_quire (proj/src/tensor_ops.cpp:166-185, via matmul :461-487):
//   C[i,j] = round( sum_k A[i,k] * B[k,j] )  with one exact quire per output.
//
// Method.  Each operand is decoded to its exact
// integer image X (posit_device.cuh) and split into D balanced int8 digits,
// X = sum_d x_d 256^d.  Then
//     Q[i,j] = sum_k X_A[i,k] X_B[k,j] = sum_g 256^g * S_g[i,j],
//     S_g    = sum_{p+q=g} A_p . B_q           (int8 x int8 -> int32 GEMMs)
// and Q mod 2^W is exactly the reference quire (quire.cpp:26-53).  Every S_g
// is computed exactly by tcgen05.mma.kind::i8 as long as it stays inside
// int32: |S_g| <= D * 128^2 * K, so K is processed in chunks of at most
// 131071/D (split-K with raw quire partials) whenever W > 32.
//
// Tensor-core mapping.  One CTA owns a 128 x NT output tile.  B's D digit
// planes for the tile are concatenated along N (N_mma = D*NT <= 256); the MMA
// for A-plane p writes TMEM columns [p*NT, p*NT + D*NT), so the product
// A_p . B_q lands in columns (p+q)*NT -- group S_{p+q} -- without any
// data movement.  TMEM holds (2D-1)*NT int32 columns.
//
// Data path.  pack_a / pack_b write the digit planes in HBM already in the
// canonical no-swizzle K-major UMMA shared-memory image, chunked per
// (tile, k-block), so the producer warp moves each stage with one
// cp.async.bulk per operand (TMA engine) into a STAGES-deep mbarrier ring.
// Warp roles: warp 0 producer, warp 1 MMA issuer (+TMEM owner), warps 2-5
// epilogue (TMEM -> registers -> 128-bit quire -> posit code).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "epilogue.cuh"
#include "fastdiv.cuh"
#include "posit_device.cuh"
#include "quire_gemm.h"
#include "pdl.cuh"
#include "sm100_ptx.cuh"
#include "tables.h"

namespace pnn_b200 {

template <int D>
struct TileCfg;
// ~190 KB of stages per CTA.  (D=2 measured: 3 x 64 KB stages beat 6 x 32 KB,
// 182 vs 193 us on the 4096^3 GEMM -- the kernel is shared-memory-bandwidth
// bound, not refill-latency bound; profiles/README.md.)
template <> struct TileCfg<2> { static constexpr int NT = 128, KB = 128, STAGES = 3; };
template <> struct TileCfg<3> { static constexpr int NT = 64, KB = 64, STAGES = 5; };
template <> struct TileCfg<4> { static constexpr int NT = 64, KB = 64, STAGES = 4; };
template <> struct TileCfg<5> { static constexpr int NT = 32, KB = 32, STAGES = 6; };
template <> struct TileCfg<6> { static constexpr int NT = 32, KB = 32, STAGES = 6; };
template <> struct TileCfg<7> { static constexpr int NT = 32, KB = 32, STAGES = 5; };
template <> struct TileCfg<8> { static constexpr int NT = 32, KB = 32, STAGES = 5; };

constexpr int kBM = 128;          // output rows per CTA (UMMA M)
constexpr int kEpiWarps = 8;      // epilogue warps (2 per TMEM lane quarter)
constexpr int kThreads = 64 + 32 * kEpiWarps;  // producer + MMA + epilogue
constexpr int kZeroBytes = kBM * 32;

// DR < D: the reduced-digit variant -- operands use only their first DR digit
// planes (every value within DR balanced digits, flags from the pack kernels);
// the packed images keep D planes per chunk (IMG_*), stages hold DR.
// CPS = 2: two CTAs per SM (reduced-digit variants whose groups fit 256 TMEM
// columns): half the stages and half the TMEM each, so one CTA's TMEM drain and
// rounding overlap the other's MMAs -- the short-K GEMMs of the Linear layers
// are bound by that per-tile serial chain, not by the tensor pipe.
template <int D, int DR = D, int CPS = 1>
struct Geometry {
    static constexpr int NT = TileCfg<D>::NT;
    static constexpr int KB = TileCfg<D>::KB;
    static constexpr int STAGES1 = TileCfg<D>::STAGES * D / DR > 12 ? 12 : TileCfg<D>::STAGES * D / DR;
    static constexpr int STAGES = CPS == 2 ? STAGES1 / 2 : STAGES1;
    static constexpr int G = 2 * DR - 1;
    static constexpr int NMMA = DR * NT;
    static constexpr int A_BYTES = DR * kBM * KB;
    static constexpr int B_BYTES = DR * NT * KB;
    static constexpr int IMG_A = D * kBM * KB;  // packed chunk strides in the workspace
    static constexpr int IMG_B = D * NT * KB;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int SMEM = STAGES * STAGE_BYTES + kZeroBytes + 256;
    static_assert((NT / 2) % 8 == 0, "epilogue column split");
    static constexpr uint32_t TMEM_COLS = CPS == 2 ? 256 : 512;
    static_assert(G * NT <= int(TMEM_COLS), "TMEM overflow");
    static_assert(STAGES >= 2, "pipeline depth");
    static_assert(NMMA % 16 == 0 && NMMA <= 256, "bad UMMA N");
    static_assert(KB % 32 == 0, "KB must hold whole i8 MMA k-steps");
};

// ---------------------------------------------------------------- packing

template <int D>
__device__ __forceinline__ void digit_words(uint32_t code, const PositFmt& f, uint32_t& lo,
                                            uint32_t& hi, bool& nar) {
    int64_t X;
    nar = decode_x_bf(code, f, X);
    // Balanced digits in two instructions: with bias = sum_{i<D} 128*256^i,
    // Y = X + bias has plain bytes (d_i + 128) in [0, 255] (|X| is within the
    // D-digit balanced capacity, so Y < 256^D), and d_i = byte_i(Y) ^ 0x80.
    constexpr uint64_t bias = 0x8080808080808080ull >> (8 * (8 - D));
    const uint64_t y = (uint64_t(X) + bias) ^ bias;
    lo = uint32_t(y);
    hi = uint32_t(y >> 32);
}

constexpr int kLutMaxBits = 10;  // shared-memory decode LUT up to 1024 codes (8 KB)

// Digit words of every code of a format (wider formats: a global table),
// built once per call into the workspace and read through L1 by the digitiser.
template <int D>
__global__ void digit_lut_kernel(PositFmt f, uint32_t* __restrict__ lut) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < (1 << f.nbits);
         c += gridDim.x * blockDim.x) {
        uint32_t lo, hi;
        bool nar;
        digit_words<D>(uint32_t(c), f, lo, hi, nar);
        lut[2 * c] = lo;
        lut[2 * c + 1] = hi;
    }
}



// Operand fetch functors: X[r][k] for r < rows, k < K (bounds checked by the
// caller).  kRowFastest picks the coalesced load order of the pack kernel.
template <typename CodeT>
struct FetchRowMajor {  // X[r][k] = p[r*ld + k]
    const CodeT* p;
    int64_t ld;
    static constexpr bool kRowFastest = false;
    static constexpr bool kVecK = true, kVecR = false, kSep = false;
    __device__ __forceinline__ const CodeT* ptr(int64_t r, int64_t k) const { return p + r * ld + k; }
    __device__ __forceinline__ uint32_t operator()(int64_t r, int64_t k) const {
        return uint32_t(p[r * ld + k]);
    }
};
template <typename CodeT>
struct FetchColMajor {  // X[r][k] = p[k*ld + r]
    const CodeT* p;
    int64_t ld;
    static constexpr bool kRowFastest = true;
    static constexpr bool kVecK = false, kVecR = true, kSep = false;
    __device__ __forceinline__ const CodeT* ptr(int64_t r, int64_t k) const { return p + k * ld + r; }
    __device__ __forceinline__ uint32_t operator()(int64_t r, int64_t k) const {
        return uint32_t(p[k * ld + r]);
    }
};

// One CTA packs (tile, k-block) chunks of the logical operand X[r][k] (A: rows
// are output rows m; B: rows are output columns n) into the canonical K-major
// no-swizzle UMMA image [D][ROWS/8][KB/16][8][16], and flags X rows that
// contain a NaR.  Loads go through a shared-memory tile (coalesced for either
// fetch order), decode is a shared-memory LUT for nbits <= 10.
// FMT: the format as a compile-time constant (BASELINE formats; fixed_fmt):
// the in-register decode of the 16-bit formats folds its shifts and masks.
template <int D, int ROWS, typename CodeT, class Fetch, int FMT = 0>
__global__ void __launch_bounds__(256) pack_kernel(Fetch fetch, int64_t rows_total, int64_t K,
                                                   PositFmt f_arg,
                                                   int8_t* __restrict__ img,
                                                   uint8_t* __restrict__ nar_flags,
                                                   uint8_t* __restrict__ any_nar_flag, int64_t tiles,
                                                   int64_t kbt, const uint2* __restrict__ glut,
                                                   uint8_t* __restrict__ wide_flag = nullptr,
                                                   int wide_planes = 0) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const PositFmt f = fixed_fmt<FMT>(f_arg);
    constexpr int KB = Geometry<D>::KB;
    constexpr int KC = KB / 16;
    // k-blocks per pass, so that every thread owns at least one 16-code unit
    constexpr int KBS = ROWS * KC >= 256 ? 1 : 256 / (ROWS * KC);
    constexpr int KW = KB * KBS;             // codes per tile row per pass
    constexpr int PADC = 4 / sizeof(CodeT);  // row stride = odd multiple of 4 bytes
    constexpr int LD = KW + PADC;
    __shared__ __align__(16) CodeT tile[ROWS * LD];
    __shared__ __align__(8) uint32_t lut[2 << kLutMaxBits];
    const bool use_lut = f.nbits <= kLutMaxBits;
    if (use_lut) {
        for (int c = threadIdx.x; c < (1 << f.nbits); c += blockDim.x) {
            uint32_t lo, hi;
            bool nar;
            digit_words<D>(uint32_t(c), f, lo, hi, nar);
            lut[2 * c] = lo;
            lut[2 * c + 1] = hi;
        }
    }
    const uint32_t nar_code = 1u << (f.nbits - 1);
    const int64_t groups_per_tile = (kbt + KBS - 1) / KBS;
    const int64_t work = tiles * groups_per_tile;
    for (int64_t wi = blockIdx.x; wi < work; wi += gridDim.x) {
        const int64_t t = wi / groups_per_tile;
        const int64_t kb0 = (wi - t * groups_per_tile) * KBS;
        const int nkb = int(kbt - kb0 < KBS ? kbt - kb0 : KBS);
        const int64_t r0 = t * ROWS, k0 = kb0 * KB;
        __syncthreads();  // previous pass's readers are done with `tile` (and LUT is built)
        constexpr int VE = 16 / int(sizeof(CodeT));  // codes per 16-byte vector
        if constexpr (Fetch::kVecK) {
            // X rows contiguous in memory: 16-byte loads along k
            constexpr int VPR = KW / VE;
            for (int i = threadIdx.x; i < ROWS * VPR; i += blockDim.x) {
                const int r = i / VPR, v = i % VPR;
                const int64_t gr = r0 + r, gk = k0 + int64_t(v) * VE;
                alignas(16) CodeT vals[VE];
                const CodeT* src = (gr < rows_total) ? fetch.ptr(gr, gk) : nullptr;
                if (src && gk + VE <= K && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                    *reinterpret_cast<uint4*>(vals) = __ldg(reinterpret_cast<const uint4*>(src));
                } else {
#pragma unroll
                    for (int j = 0; j < VE; ++j)
                        vals[j] = (gr < rows_total && gk + j < K) ? CodeT(fetch(gr, gk + j)) : CodeT(0);
                }
                uint32_t* dst = reinterpret_cast<uint32_t*>(tile + r * LD + v * VE);
#pragma unroll
                for (int w = 0; w < 4; ++w) dst[w] = reinterpret_cast<const uint32_t*>(vals)[w];
            }
        } else if constexpr (Fetch::kVecR) {
            // X columns contiguous in memory (B row-major): 16-byte loads along r
            constexpr int VPC = ROWS / VE;
            for (int i = threadIdx.x; i < KW * VPC; i += blockDim.x) {
                const int k = i / VPC, v = i % VPC;
                const int64_t gr = r0 + int64_t(v) * VE, gk = k0 + k;
                alignas(16) CodeT vals[VE];
                const CodeT* src = (gk < K) ? fetch.ptr(gr, gk) : nullptr;
                if (src && gr + VE <= rows_total && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                    *reinterpret_cast<uint4*>(vals) = __ldg(reinterpret_cast<const uint4*>(src));
                } else {
#pragma unroll
                    for (int j = 0; j < VE; ++j)
                        vals[j] = (gr + j < rows_total && gk < K) ? CodeT(fetch(gr + j, gk)) : CodeT(0);
                }
#pragma unroll
                for (int j = 0; j < VE; ++j) tile[(v * VE + j) * LD + k] = vals[j];
            }
        } else if constexpr (Fetch::kSep) {
            // Separable gathers (im2col & co): the index decomposition of a row
            // and of a k is computed once per pass into shared memory; each
            // element is then a few adds, two range tests and one load.
            __shared__ typename Fetch::RI rinfo[ROWS];
            __shared__ typename Fetch::KI kinfo[KW];
            for (int r = threadIdx.x; r < ROWS; r += blockDim.x)
                rinfo[r] = fetch.row(r0 + r < rows_total ? r0 + r : 0);
            for (int k = threadIdx.x; k < KW; k += blockDim.x)
                kinfo[k] = fetch.kin(k0 + k < K ? k0 + k : 0);
            __syncthreads();
            for (int i = threadIdx.x; i < ROWS * KW; i += blockDim.x) {
                int r, k;
                if constexpr (Fetch::kRowFastest) {
                    k = i / ROWS;
                    r = i % ROWS;
                } else {
                    r = i / KW;
                    k = i % KW;
                }
                const bool in = (r0 + r < rows_total) && (k0 + k < K);
                tile[r * LD + k] = in ? CodeT(fetch.at(rinfo[r], kinfo[k])) : CodeT(0);
            }
        } else if constexpr (!Fetch::kRowFastest) {
            for (int i = threadIdx.x; i < ROWS * KW; i += blockDim.x) {
                const int r = i / KW, k = i % KW;  // k fastest: coalesced along a row of X
                const int64_t gr = r0 + r, gk = k0 + k;
                tile[r * LD + k] = (gr < rows_total && gk < K) ? CodeT(fetch(gr, gk)) : CodeT(0);
            }
        } else {
            for (int i = threadIdx.x; i < ROWS * KW; i += blockDim.x) {
                const int k = i / ROWS, r = i % ROWS;  // r fastest: coalesced along X's column
                const int64_t gr = r0 + r, gk = k0 + k;
                tile[r * LD + k] = (gr < rows_total && gk < K) ? CodeT(fetch(gr, gk)) : CodeT(0);
            }
        }
        __syncthreads();
        for (int u = threadIdx.x; u < ROWS * KC * nkb; u += blockDim.x) {
            const int r8 = u & 7;
            const int rest = u >> 3;
            const int kc = rest % KC;
            const int rg = (rest / KC) % (ROWS / 8);
            const int kbl = rest / (KC * (ROWS / 8));
            const int r = rg * 8 + r8;
            uint32_t lo[16], hi[16];
            const CodeT* tr = tile + r * LD + kbl * KB + kc * 16;
            constexpr int NW = int(16 * sizeof(CodeT) / 4);
            uint32_t wv[NW];
#pragma unroll
            for (int w = 0; w < NW; ++w) wv[w] = reinterpret_cast<const uint32_t*>(tr)[w];
            // NaR codes, word-wise: a zero byte / halfword of (codes ^ NaR pattern)
            // (exact zero-lane test: (x - 1s) & ~x & msbs != 0 iff some lane of x is 0)
            uint32_t narm = 0;
            {
                constexpr uint32_t ones = sizeof(CodeT) == 1 ? 0x01010101u : 0x00010001u;
                constexpr uint32_t msbs = sizeof(CodeT) == 1 ? 0x80808080u : 0x80008000u;
                const uint32_t cmask = ((1u << f.nbits) - 1u) * ones;
                const uint32_t narw = nar_code * ones;
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    const uint32_t x = (wv[w] & cmask) ^ narw;
                    narm |= (x - ones) & ~x & msbs;
                }
            }
            const bool any_nar = narm != 0;
            auto code_of = [&](int j) -> uint32_t {
                return sizeof(CodeT) == 1 ? (wv[j >> 2] >> (8 * (j & 3))) & 0xFFu
                                          : (wv[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
            };
            // (one straight-line loop per decode source: no per-code branches)
            if (use_lut) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t code = code_of(j);
                    if constexpr (D > 4) {
                        const uint2 v = reinterpret_cast<const uint2*>(lut)[code];
                        lo[j] = v.x;
                        hi[j] = v.y;
                    } else {
                        lo[j] = lut[2 * code];
                        hi[j] = 0u;
                    }
                }
            } else if (glut != nullptr) {  // 11-16-bit formats: L2-resident table
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint2 v = __ldg(glut + code_of(j));
                    lo[j] = v.x;
                    hi[j] = v.y;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    bool nar;
                    digit_words<D>(code_of(j), f, lo[j], hi[j], nar);
                }
            }
            if (any_nar && r0 + r < rows_total) {
                nar_flags[r0 + r] = 1;
                *any_nar_flag = 1;
            }
            if (wide_flag != nullptr) {  // a digit plane >= wide_planes in use (digit bytes != 0)
                const uint32_t mlo = wide_planes >= 4 ? 0u : ~0u << (8 * wide_planes);
                const uint32_t mhi = wide_planes >= 4 ? ~0u << (8 * (wide_planes - 4)) : ~0u;
                uint32_t o = 0;
#pragma unroll
                for (int j = 0; j < 16; ++j) o |= (lo[j] & mlo) | (hi[j] & mhi);
                if (o && *reinterpret_cast<volatile uint8_t*>(wide_flag) == 0) *wide_flag = 1;  // read first: no same-address store storm
            }
            int8_t* chunk = img + (t * kbt + kb0 + kbl) * int64_t(D * ROWS * KB);
#pragma unroll
            for (int p = 0; p < D; ++p) {
                const uint32_t* w = p < 4 ? lo : hi;
                const uint32_t q = p & 3;
                const uint32_t sel = q | ((q + 4) << 4);
                uint4 v;
                uint32_t* vv = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const uint32_t a = __byte_perm(w[4 * jj], w[4 * jj + 1], sel);
                    const uint32_t b = __byte_perm(w[4 * jj + 2], w[4 * jj + 3], sel);
                    vv[jj] = __byte_perm(a, b, 0x5410);
                }
                *reinterpret_cast<uint4*>(chunk + p * (ROWS * KB) + rg * (8 * KB) + kc * 128 +
                                          r8 * 16) = v;
            }
        }
    }
}

// The pack for operands that are plain matrices (FetchRowMajor / FetchColMajor
// / the Linear layers' FetchRowsBias): no shared-memory tile and no block
// barriers.  A thread owns 16-code units (one row x 16 consecutive k) of the
// image, fetched straight from global memory --
//   k contiguous (kVecK): 16-byte loads of the row; lanes (r8, kc, rg), so a
//     warp reads whole 32-byte sectors and writes 512 contiguous image bytes;
//   r contiguous (kVecR): one 4-byte load per k holding the codes of RPT = 2
//     (16-bit) or 4 (8-bit) consecutive rows, i.e. RPT units per thread; lanes
//     = consecutive row groups, so every request is full sectors (RPT = 1:
//     scalar loads, for operands whose rows are not 4-byte aligned) --
// and the NEXT step's codes are loaded before this step is digitised, so the
// load latency hides under the (ALU-bound) digit arithmetic.  Same image,
// NaR flags and wide flags as pack_kernel (tests: every GEMM / Linear test).
template <int D, int ROWS, typename CodeT, class Fetch, int FMT = 0, int RPT = 1>
__global__ void __launch_bounds__(256) pack_direct_kernel(Fetch fetch, int64_t rows_total, int64_t K,
                                                          PositFmt f_arg, int8_t* __restrict__ img,
                                                          uint8_t* __restrict__ nar_flags,
                                                          uint8_t* __restrict__ any_nar_flag,
                                                          uint32_t chunks, FastDiv fd_kbt,
                                                          const uint2* __restrict__ glut,
                                                          uint8_t* __restrict__ wide_flag = nullptr,
                                                          int wide_planes = 0) {
    static_assert(Fetch::kVecK || Fetch::kVecR, "plain-matrix operands only");
    static_assert(RPT == 1 || (Fetch::kVecR && RPT * sizeof(CodeT) == 4), "row groups: 4-byte loads");
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const PositFmt f = fixed_fmt<FMT>(f_arg);
    constexpr int KB = Geometry<D>::KB;
    constexpr int KC = KB / 16;
    constexpr int UPC = ROWS * KC / RPT;  // steps (units or row groups) per (tile, k-block) chunk
    constexpr int CB = 8 * int(sizeof(CodeT));  // code bits in a word lane
    // words per step: a unit's 16 codes packed, or one word per k (RPT rows each)
    constexpr int NW = RPT == 1 ? int(16 * sizeof(CodeT) / 4) : 16;
    constexpr int VE = 16 / int(sizeof(CodeT));
    // Shared-memory digit table (formats up to 10 bits).  8-bit codes with
    // D <= 4 (one digit word per code): 32 copies, entry (code, lane) at word
    // code * 32 + lane, so a warp's 32 lookups of arbitrary codes hit 32
    // different banks; otherwise {lo, hi} pairs per code.
    constexpr bool kLaneLut = D <= 4 && sizeof(CodeT) == 1;
    __shared__ __align__(8) uint32_t lut[kLaneLut ? 256 * 32 : (2 << kLutMaxBits)];
    const bool use_lut = f.nbits <= kLutMaxBits;
    if (use_lut) {
        for (int c = threadIdx.x; c < (1 << f.nbits); c += blockDim.x) {
            uint32_t lo, hi;
            bool nar;
            digit_words<D>(uint32_t(c), f, lo, hi, nar);
            if constexpr (kLaneLut) {
#pragma unroll
                for (int l = 0; l < 32; ++l) lut[c * 32 + ((l + c) & 31)] = lo;  // (rotated: conflict-free stores)
            } else {
                lut[2 * c] = lo;
                lut[2 * c + 1] = hi;
            }
        }
        __syncthreads();
    }
    const uint32_t* lut_lane = lut + (threadIdx.x & 31);
    const uint32_t nar_code = 1u << (f.nbits - 1);
    const uint32_t total = chunks * uint32_t(UPC);  // < 2^31 (launcher)
    const uint32_t stride = gridDim.x * blockDim.x;

    // step g -> (chunk, first row in the tile, 16-code column)
    auto locate = [&](uint32_t g, uint32_t& chunk, int& r, int& kc) {
        chunk = g / uint32_t(UPC);
        const int u = int(g % uint32_t(UPC));
        if constexpr (Fetch::kVecK) {
            kc = (u >> 3) % KC;
            r = ((u >> 3) / KC) * 8 + (u & 7);
        } else {
            r = (u % (ROWS / RPT)) * RPT;
            kc = u / (ROWS / RPT);
        }
    };
    auto load = [&](uint32_t g, uint32_t (&wv)[NW]) {
        uint32_t chunk, t, kb;
        int r, kc;
        locate(g, chunk, r, kc);
        fd_kbt.divmod(chunk, t, kb);
        const int64_t gr = int64_t(t) * ROWS + r, gk = int64_t(kb) * KB + kc * 16;
        if constexpr (Fetch::kVecK) {
#pragma unroll
            for (int v = 0; v < NW / 4; ++v) {
                const int64_t k0 = gk + v * VE;
                const CodeT* src = gr < rows_total ? fetch.ptr(gr, k0) : nullptr;
                if (src != nullptr && k0 + VE <= K && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                    const uint4 q = __ldg(reinterpret_cast<const uint4*>(src));
                    wv[4 * v] = q.x, wv[4 * v + 1] = q.y, wv[4 * v + 2] = q.z, wv[4 * v + 3] = q.w;
                } else {
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        uint32_t acc = 0;
#pragma unroll
                        for (int j = 0; j < VE / 4; ++j) {
                            const int64_t k = k0 + w * (VE / 4) + j;
                            const uint32_t c = (gr < rows_total && k < K) ? fetch(gr, k) : 0u;
                            acc |= c << (CB * j);
                        }
                        wv[4 * v + w] = acc;
                    }
                }
            }
        } else if constexpr (RPT > 1) {
            // one aligned word per k: the codes of rows gr .. gr + RPT - 1
            if (gr + RPT <= rows_total && gk + 16 <= K) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    wv[j] = __ldg(reinterpret_cast<const uint32_t*>(fetch.ptr(gr, gk + j)));
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    uint32_t acc = 0;
#pragma unroll
                    for (int i = 0; i < RPT; ++i) {
                        const uint32_t c = (gr + i < rows_total && gk + j < K) ? fetch(gr + i, gk + j) : 0u;
                        acc |= c << (CB * i);
                    }
                    wv[j] = acc;
                }
            }
        } else {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                uint32_t acc = 0;
#pragma unroll
                for (int j = 0; j < 16 / NW; ++j) {
                    const int64_t k = gk + w * (16 / NW) + j;
                    const uint32_t c = (gr < rows_total && k < K) ? fetch(gr, k) : 0u;
                    acc |= c << (CB * j);
                }
                wv[w] = acc;
            }
        }
    };

    uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t cur[NW], nxt[NW];
    if (g < total) load(g, cur);
    for (; g < total; g += stride) {
        const bool more = g + stride < total;  // (total + stride < 2^32)
        if (more) load(g + stride, nxt);
        uint32_t chunk;
        int r0, kc;
        locate(g, chunk, r0, kc);
        // NaR codes, word-wise: the exactly-zero lanes of (codes ^ NaR pattern)
        uint32_t narm = 0;
        {
            constexpr uint32_t ones = sizeof(CodeT) == 1 ? 0x01010101u : 0x00010001u;
            constexpr uint32_t low = sizeof(CodeT) == 1 ? 0x7F7F7F7Fu : 0x7FFF7FFFu;
            const uint32_t cmask = ((1u << f.nbits) - 1u) * ones;
            const uint32_t narw = nar_code * ones;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const uint32_t x = (cur[w] & cmask) ^ narw;
                narm |= ~(((x & low) + low) | x | low);
            }
        }
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = r0 + i;
            auto code_of = [&](int j) -> uint32_t {
                if constexpr (RPT > 1) return (cur[j] >> (CB * i)) & ((1u << CB) - 1u);
                else
                    return sizeof(CodeT) == 1 ? (cur[j >> 2] >> (8 * (j & 3))) & 0xFFu
                                              : (cur[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
            };
            uint32_t lo[16], hi[16];
            if (use_lut) {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint32_t code = code_of(j);
                    if constexpr (kLaneLut) {
                        lo[j] = lut_lane[code * 32];
                        hi[j] = 0u;
                    } else if constexpr (D > 4) {
                        const uint2 v = reinterpret_cast<const uint2*>(lut)[code];
                        lo[j] = v.x;
                        hi[j] = v.y;
                    } else {
                        lo[j] = lut[2 * code];
                        hi[j] = 0u;
                    }
                }
            } else if (glut != nullptr) {  // 11-12-bit formats: process-lifetime table, L1-resident
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const uint2 v = __ldg(glut + code_of(j));
                    lo[j] = v.x;
                    hi[j] = v.y;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    bool nar;
                    digit_words<D>(code_of(j), f, lo[j], hi[j], nar);
                }
            }
            const uint32_t rowm = RPT == 1 ? narm : narm & (((1u << CB) - 1u) << (CB * i));
            if (rowm != 0) {
                uint32_t t, kb;
                fd_kbt.divmod(chunk, t, kb);
                const int64_t gr = int64_t(t) * ROWS + r;
                if (gr < rows_total) {
                    nar_flags[gr] = 1;
                    *any_nar_flag = 1;
                }
            }
            if (wide_flag != nullptr) {  // a digit plane >= wide_planes in use (digit bytes != 0)
                const uint32_t mlo = wide_planes >= 4 ? 0u : ~0u << (8 * wide_planes);
                const uint32_t mhi = wide_planes >= 4 ? ~0u << (8 * (wide_planes - 4)) : ~0u;
                uint32_t o = 0;
#pragma unroll
                for (int j = 0; j < 16; ++j) o |= (lo[j] & mlo) | (hi[j] & mhi);
                if (o && *reinterpret_cast<volatile uint8_t*>(wide_flag) == 0) *wide_flag = 1;  // read first: no same-address store storm
            }
            int8_t* dst = img + int64_t(chunk) * int64_t(D * ROWS * KB) + (r >> 3) * (8 * KB) + kc * 128 +
                          (r & 7) * 16;
#pragma unroll
            for (int p = 0; p < D; ++p) {
                const uint32_t* w = p < 4 ? lo : hi;
                const uint32_t q = p & 3;
                const uint32_t sel = q | ((q + 4) << 4);
                uint4 v;
                uint32_t* vv = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const uint32_t a = __byte_perm(w[4 * jj], w[4 * jj + 1], sel);
                    const uint32_t b = __byte_perm(w[4 * jj + 2], w[4 * jj + 3], sel);
                    vv[jj] = __byte_perm(a, b, 0x5410);
                }
                *reinterpret_cast<uint4*>(dst + p * (ROWS * KB)) = v;
            }
        }
#pragma unroll
        for (int w = 0; w < NW; ++w) cur[w] = nxt[w];
    }
}

// ------------------------------------------------------------- main kernel

// Where output element (m, n) lives: mode 0 row-major (m*ldc + n); mode 1
// NCHW scatter for convolutions (m = img*inner + pixel, n = channel); mode 2
// tap-major weight-gradient rows (m = tap*inner + c -> n*ldc + c*ncols + tap).
template <typename CodeT>
struct OutMap {
    CodeT* base;
    int64_t ldc;
    int64_t inner;
    int64_t ncols;
    int mode;
    // mode 3 (implicit weight grad): 128-row tiles (ky, kx group, 32-channel group),
    // row within a tile = (slice j, kx k, channel c16) -> dw[n][c][ky][kx]
    int kh, kw, kgroups, cgroups, cvalid;
    FastDiv fd_inner;  // mode 1: division by inner (set when inner < 2^31)
    __device__ __forceinline__ int64_t row_base(int64_t m) const {
        if (mode == 0) return m * ldc;
        if (mode == 3) {
            const int mt = int(m >> 7), ml = int(m & 127);
            const int kc = kgroups * cgroups;
            const int ky = mt / kc, kx = ((mt % kc) / cgroups) * 4 + ((ml >> 4) & 3);
            const int c = (mt % cgroups) * 32 + (ml >> 6) * 16 + (ml & 15);
            if (ky >= kh || kx >= kw || c >= cvalid) return -1;  // padding rows
            return int64_t(c) * (kh * kw) + ky * kw + kx;
        }
        int64_t hi, lo;
        if (mode == 1 && fd_inner.d == uint64_t(inner) && m < (int64_t(1) << 31)) {
            uint32_t q, r;
            fd_inner.divmod(uint32_t(m), q, r);
            hi = q;
            lo = r;
        } else if (m < (int64_t(1) << 31) && inner < (int64_t(1) << 31)) {  // 32-bit division
            const uint32_t h32 = uint32_t(m) / uint32_t(inner);
            hi = h32;
            lo = m - int64_t(h32) * inner;
        } else {
            hi = m / inner;
            lo = m - hi * inner;
        }
        if (mode == 2) return lo * ncols + hi;
        return hi * ncols * inner + lo;
    }
    // index(m, n) == row_base(m) + n * col_stride(); -1: no output for row m
    __device__ __forceinline__ int64_t index(int64_t m, int64_t n) const {
        const int64_t b = row_base(m);
        return b < 0 ? -1 : b + n * col_stride();
    }
    __device__ __forceinline__ int64_t col_stride() const {
        return mode == 0 ? 1 : (mode == 2 || mode == 3) ? ldc : inner;
    }
};

template <typename CodeT>
__device__ __forceinline__ void store_codes8(CodeT* dst, const uint32_t (&c)[8], int valid,
                                             bool vec_ok) {
    if (vec_ok && valid == 8) {
        if constexpr (sizeof(CodeT) == 1) {
            uint2 v;
            v.x = (c[0] & 0xFF) | ((c[1] & 0xFF) << 8) | ((c[2] & 0xFF) << 16) | (c[3] << 24);
            v.y = (c[4] & 0xFF) | ((c[5] & 0xFF) << 8) | ((c[6] & 0xFF) << 16) | (c[7] << 24);
            *reinterpret_cast<uint2*>(dst) = v;
        } else {
            uint4 v;
            v.x = (c[0] & 0xFFFF) | (c[1] << 16);
            v.y = (c[2] & 0xFFFF) | (c[3] << 16);
            v.z = (c[4] & 0xFFFF) | (c[5] << 16);
            v.w = (c[6] & 0xFFFF) | (c[7] << 16);
            *reinterpret_cast<uint4*>(dst) = v;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j)  // unrolled: c[] stays in registers
            if (j < valid) dst[j] = CodeT(c[j]);
    }
}

template <int QW>
struct QuireWord;
template <> struct QuireWord<1> { using T = uint32_t; };
template <> struct QuireWord<2> { using T = uint64_t; };
template <> struct QuireWord<4> { using T = unsigned __int128; };

// Sign-extend an int32 group sum and weight it by 256^g, modulo the word size
// (the quire itself is only defined mod 2^W <= word bits).
template <typename T>
__device__ __forceinline__ T group_term(uint32_t acc, int sh) {
    if constexpr (sizeof(T) == 4) return T(acc) << sh;
    else if constexpr (sizeof(T) == 8) return T(int64_t(int32_t(acc))) << sh;
    else return T(__int128(int32_t(acc))) << sh;
}

// Quire word of one output from its int32 group sums, Q = sum_g S_g 256^g
// (mod the word size).  Groups are accumulated per 32-bit word position in
// int64 (one IMAD.WIDE each: |S_g * 2^(8g mod 32)| < 2^55, <= 4 terms per
// word) and the words are combined once -- instead of a wide shift-add per
// group.  `gg` is a compile-time constant after unrolling.
template <typename T>
struct QAcc;
template <>
struct QAcc<uint32_t> {  // W <= 32
    uint32_t v = 0;
    __device__ __forceinline__ void add(int gg, uint32_t s) {
        if (8 * gg < 32) v += s << (8 * gg);
    }
    __device__ __forceinline__ uint32_t get() const { return v; }
};
template <>
struct QAcc<uint64_t> {  // W <= 64
    int64_t w0 = 0, w1 = 0;
    __device__ __forceinline__ void add(int gg, uint32_t s) {
        const int64_t x = int64_t(int32_t(s));
        if (8 * gg < 32) w0 += x * int64_t(1 << (8 * gg));
        else if (8 * gg < 64) w1 += x * int64_t(1 << (8 * gg - 32));
    }
    __device__ __forceinline__ uint64_t get() const { return uint64_t(w0) + (uint64_t(w1) << 32); }
};
template <>
struct QAcc<unsigned __int128> {  // W <= 128
    int64_t w[4] = {0, 0, 0, 0};
    __device__ __forceinline__ void add(int gg, uint32_t s) {
        const int64_t x = int64_t(int32_t(s));
        const int wi = (8 * gg) >> 5;
        if (wi < 4) w[wi] += x * int64_t(1 << ((8 * gg) & 31));
    }
    __device__ __forceinline__ unsigned __int128 get() const {
        return (unsigned __int128)(__int128(w[0]) + (__int128(w[1]) << 32) + (__int128(w[2]) << 64) +
                                   (__int128(w[3]) << 96));
    }
};

// Raster: tiles grouped by kGroupM m-tiles so the ~148 tiles in flight share
// A and B digit planes in L2.
constexpr int kGroupM = 8;

// 32-bit arithmetic (the planners keep tile counts below 2^31): 64-bit integer
// division is a ~100-instruction call, and every role of every tile runs this.
__device__ __forceinline__ void tile_coords(int64_t t64, int64_t mtiles64, int64_t ntiles64,
                                            int64_t& split, int64_t& mt, int64_t& nt) {
    const uint32_t t = uint32_t(t64), mtiles = uint32_t(mtiles64), ntiles = uint32_t(ntiles64);
    const uint32_t per_split = mtiles * ntiles;
    const uint32_t sp = t / per_split;
    const uint32_t r = t - sp * per_split;
    const uint32_t group = r / (kGroupM * ntiles);
    const uint32_t within = r - group * (kGroupM * ntiles);
    const uint32_t left = mtiles - group * kGroupM;
    const uint32_t gm = left < uint32_t(kGroupM) ? left : uint32_t(kGroupM);
    split = sp;
    mt = group * kGroupM + within % gm;
    nt = within / gm;
}

// Persistent, warp-specialized: warp 0 = bulk-copy producer, warp 1 = MMA
// issuer, warps 2..9 = epilogue (2 warps per TMEM lane quarter, each owning
// half of the tile's columns).  The epilogue drains TMEM into registers,
// releases it (tmem_empty), and rounds/stores while the next tile's MMAs run.
template <int D, int QW, typename CodeT, bool kPair, int FMT = 0, int DR = D, int CPS = 1>
__global__ void __launch_bounds__(kThreads, CPS)
    quire_gemm_tc_kernel(const int8_t* __restrict__ a_img, const int8_t* __restrict__ b_img,
                         int64_t kbt, int64_t kb_per_split, const uint8_t* __restrict__ row_nar,
                         const uint8_t* __restrict__ col_nar, OutMap<CodeT> out, int64_t M,
                         int64_t N, PositFmt f_arg,
                         unsigned __int128* __restrict__ partial, int64_t mtiles, int64_t ntiles,
                         int64_t splits, const uint8_t* __restrict__ vflags, int vmode,
                         const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB) {
    pdl_trigger();  // the next kernel's CTAs may start their prologue in this grid's tail
    // kPair: clusters of 2 CTAs run one M=256 tcgen05.mma.cta_group::2 per
    // digit plane; each CTA stages its own 128-row A tile and HALF of the
    // concatenated B rows, halving each SM's shared-memory operand traffic.
    const PositFmt f = fixed_fmt<FMT>(f_arg);  // compile-time for the BASELINE formats
    using Geo = Geometry<D, DR, CPS>;
    using QT = typename QuireWord<QW>::T;
    constexpr int NT = Geo::NT, KB = Geo::KB, STAGES = Geo::STAGES, G = Geo::G;
    constexpr int COLS = NT / 2;                 // columns per epilogue thread
    constexpr int GB = G < 8 ? G : 8;            // TMEM loads batched per wait
    constexpr int B_LOCAL = kPair ? Geo::B_BYTES / 2 : Geo::B_BYTES;
    constexpr int STAGE_TX = Geo::A_BYTES + B_LOCAL;
    extern __shared__ __align__(1024) uint8_t smem[];
    // 64-bit quire words round through the FP64 converter + rounding table
    // (epilogue.cuh q_to_posit_lut_f64: the word is the exact value, any W)
    __shared__ uint4 s_lut[QW == 2 ? kPackLutEntries : 1];
    if constexpr (QW == 2) build_pack_lut(f, s_lut, threadIdx.x, kThreads);
    // 8-bit outputs: the rounding as one table lookup (epilogue.cuh)
    constexpr bool kTab8 = sizeof(CodeT) == 1 && QW == 2;
    __shared__ uint8_t s_tab8[kTab8 ? kTab8Bytes : 1];
    if constexpr (kTab8) {
        __syncthreads();
        build_pack_tab8(f, s_lut, s_tab8, threadIdx.x, kThreads);
    }
    uint8_t* zero_tile = smem + STAGES * Geo::STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(zero_tile + kZeroBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = kPair ? ptx::cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    // work units: pair-tiles (2 m-tiles x 1 n-tile) in pair mode
    const int64_t unit_m = kPair ? (mtiles + 1) / 2 : mtiles;
    const int64_t tiles = unit_m * ntiles * splits;
    const int64_t unit0 = kPair ? blockIdx.x / 2 : blockIdx.x;
    const int64_t ustride = kPair ? gridDim.x / 2 : gridDim.x;

    for (int i = threadIdx.x; i < kZeroBytes / 16; i += kThreads)
        reinterpret_cast<int4*>(zero_tile)[i] = make_int4(0, 0, 0, 0);
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            // (pair: both CTAs' tensor loads complete_tx on the leader's barrier;
            // its one arrival is the leader's expect_tx)
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(tmem_full, 1);
        ptx::mbar_init(tmem_empty, kPair ? 2 * kEpiWarps : kEpiWarps);
        ptx::fence_barrier_init();
    }
    // everything above touched only shared memory and parameters (PDL prologue)
    pdl_wait();
    // device-selected variant (vflags = {A wide, B wide} from the pack kernels):
    // vmode 1 runs iff neither operand is wide, 2 iff either is; exit at once otherwise
    if ((vmode & 0xFF) != 0) {
        const bool wide = vflags[0] != 0 || vflags[1] != 0;
        if (wide != ((vmode & 0xFF) == 2)) return;
    }
    if (warp == 1) {
        if constexpr (kPair) ptx::tmem_alloc2<Geo::TMEM_COLS>(tmem_slot);
        else ptx::tmem_alloc<Geo::TMEM_COLS>(tmem_slot);
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    if constexpr (kPair) ptx::cluster_sync();
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ===== producer: one bulk copy per operand per stage =====
            uint32_t it = 0;
            for (int64_t t = unit0; t < tiles; t += ustride) {
                int64_t split, um, nt;
                tile_coords(t, unit_m, ntiles, split, um, nt);
                const int64_t mt = kPair ? 2 * um + rank : um;
                const int64_t kb0 = split * kb_per_split;
                const int nkb = int(min(kbt, kb0 + kb_per_split) - kb0);
                const int8_t* a_src = a_img + (mt * kbt + kb0) * int64_t(Geo::IMG_A);
                const int8_t* b_src = b_img + (nt * kbt + kb0) * int64_t(Geo::IMG_B) +
                                      (kPair ? rank * B_LOCAL : 0);
                for (int i = 0; i < nkb; ++i, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    ptx::mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* sa = smem + s * Geo::STAGE_BYTES;
                    if constexpr (kPair) {
                        // 2-D tensor boxes of the packed images (rows of 256 bytes), each CTA
                        // its own A tile and half of B, both signalling the leader's barrier
                        if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * STAGE_TX);
                        const int64_t ra = ((mt * kbt + kb0 + i) * int64_t(Geo::IMG_A)) >> 8;
                        const int64_t rb = ((nt * kbt + kb0 + i) * int64_t(Geo::IMG_B) + rank * B_LOCAL) >> 8;
                        ptx::tma_load_2d_pair(sa, &tmA, 0, int(ra), &full[s]);
                        ptx::tma_load_2d_pair(sa + Geo::A_BYTES, &tmB, 0, int(rb), &full[s]);
                    } else {
                        ptx::mbar_arrive_expect_tx(&full[s], STAGE_TX);
                        ptx::bulk_g2s(sa, a_src + int64_t(i) * Geo::IMG_A, Geo::A_BYTES, &full[s]);
                        ptx::bulk_g2s(sa + Geo::A_BYTES, b_src + int64_t(i) * Geo::IMG_B, B_LOCAL,
                                      &full[s]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {
            // ===== MMA issuer =====
            constexpr uint32_t idesc = ptx::idesc_i8(kPair ? 2 * kBM : kBM, Geo::NMMA);
            constexpr uint32_t SBO = 8 * KB, LBO = 128;
            const uint64_t zdesc = ptx::smem_desc_kmajor(ptx::smem_u32(zero_tile), LBO, 8 * 32);
            uint32_t it = 0, j = 0;
            for (int64_t t = unit0; t < tiles; t += ustride, ++j) {
                int64_t split, um, nt;
                tile_coords(t, unit_m, ntiles, split, um, nt);
                const int64_t kb0 = split * kb_per_split;
                const int nkb = int(min(kbt, kb0 + kb_per_split) - kb0);
                ptx::mbar_wait(tmem_empty, (j & 1) ^ 1);  // epilogue(s) drained the previous tile
                ptx::tc_fence_after();
                for (int i = 0; i < nkb; ++i, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    ptx::mbar_wait(&full[s], ph);
                    ptx::tc_fence_after();
                    const uint32_t a_base = ptx::smem_u32(smem + s * Geo::STAGE_BYTES);
                    const uint32_t b_base = a_base + Geo::A_BYTES;
#pragma unroll
                    for (int ks = 0; ks < KB / 32; ++ks) {
                        const uint64_t bdesc = ptx::smem_desc_kmajor(b_base + ks * 256, LBO, SBO);
                        const bool first = (i == 0 && ks == 0);
                        if (first) {  // zero groups DR-1 .. 2DR-2 (plane 0 initialises 0 .. DR-1)
                            if constexpr (kPair) ptx::mma_i8_pair(tmem + (DR - 1) * NT, zdesc, bdesc, idesc, 0);
                            else ptx::mma_i8(tmem + (DR - 1) * NT, zdesc, bdesc, idesc, 0);
                        }
#pragma unroll
                        for (int p = 0; p < DR; ++p) {
                            const uint64_t adesc = ptx::smem_desc_kmajor(
                                a_base + p * (kBM * KB) + ks * 256, LBO, SBO);
                            if constexpr (kPair)
                                ptx::mma_i8_pair(tmem + p * NT, adesc, bdesc, idesc,
                                                 (first && p == 0) ? 0u : 1u);
                            else
                                ptx::mma_i8(tmem + p * NT, adesc, bdesc, idesc,
                                            (first && p == 0) ? 0u : 1u);
                        }
                    }
                    if constexpr (kPair) ptx::mma_commit_pair(&empty[s]);
                    else ptx::mma_commit(&empty[s]);
                }
                if constexpr (kPair) ptx::mma_commit_pair(tmem_full);
                else ptx::mma_commit(tmem_full);
            }
        }
    } else {
        // ===== epilogue: TMEM -> quire words (registers) -> posit codes =====
        const int quarter = warp & 3;
        const int half = (warp - 2) >> 2;
        // the two warps of a lane quarter take alternate 8-column chunks, so both
        // stay busy when the valid columns (N) fill only part of the tile
        const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16) + half * 8;
        const bool vec_ok = out.mode == 0 && (out.ldc % 8) == 0;
        uint32_t j = 0;
        const uint32_t tmem_empty_leader = kPair ? ptx::mapa(ptx::smem_u32(tmem_empty), 0) : 0u;
        for (int64_t t = unit0; t < tiles; t += ustride, ++j) {
            int64_t split, um, nt;
            tile_coords(t, unit_m, ntiles, split, um, nt);
            const int64_t mt = kPair ? 2 * um + rank : um;
            ptx::mbar_wait(tmem_full, j & 1);
            ptx::tc_fence_after();
            QT q[COLS];
#pragma unroll
            for (int c0 = 0; c0 < COLS; c0 += 8) {
                QAcc<QT> acc[8];
#pragma unroll
                for (int g0 = 0; g0 < G; g0 += GB) {
                    uint32_t r[GB][8];
#pragma unroll
                    for (int g = 0; g < GB; ++g)
                        if (g0 + g < G) {
#ifdef PNN_GEMM_DEBUG_HOOKS  // profiling (tools/probes/gemm_drain.sh): no TMEM loads
                            if (vmode & 0x100) {
                                for (int x = 0; x < 8; ++x) r[g][x] = 0;
                                continue;
                            }
#endif
                            ptx::tmem_ld8(trow + (g0 + g) * NT + 2 * c0, r[g]);
                        }
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int g = 0; g < GB; ++g)
                        if (g0 + g < G)
#pragma unroll
                            for (int x = 0; x < 8; ++x) acc[x].add(g0 + g, r[g][x]);
                }
#pragma unroll
                for (int x = 0; x < 8; ++x) q[c0 + x] = acc[x].get();
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (kPair && !leader) ptx::mbar_arrive_remote(tmem_empty_leader);
                else ptx::mbar_arrive(tmem_empty);
            }

            const int64_t row = mt * kBM + quarter * 32 + lane;
            if (row >= M) continue;
#ifdef PNN_GEMM_DEBUG_HOOKS  // profiling: no rounding, no stores
            if (vmode & 0x200) continue;
#endif
            const bool rnar = row_nar != nullptr && row_nar[row] != 0;
            const int64_t colbase = nt * NT + half * 8;  // + 2 * c0 for chunk c0 / 8
#pragma unroll
            for (int c0 = 0; c0 < COLS; c0 += 8) {
                const int64_t col0 = colbase + 2 * c0;
                if (col0 >= N) break;
                const int valid = int(N - col0 < 8 ? N - col0 : 8);
                if (partial != nullptr) {
                    unsigned __int128* dst = partial + (split * M + row) * N + col0;
#pragma unroll
                    for (int x = 0; x < 8; ++x)
                        if (x < valid) {
                            if constexpr (QW == 2)  // sign-extended: the exact value for any W
                                dst[x] = (unsigned __int128)(__int128)int64_t(q[c0 + x]);
                            else
                                dst[x] = (unsigned __int128)q[c0 + x];
                        }
                    continue;
                }
                // column NaR flags as one 8-byte load (flag buffer padded to whole tiles)
                const uint64_t cn =
                    col_nar != nullptr ? *reinterpret_cast<const uint64_t*>(col_nar + col0) : 0ull;
                uint32_t codes[8];
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    const bool nar = rnar || ((cn >> (8 * x)) & 0xFF) != 0;
                    uint32_t c;
                    if constexpr (kTab8) c = q_to_posit_tab8<false, false>(f, uint64_t(q[c0 + x]), s_tab8);
                    else if constexpr (QW == 2) c = q_to_posit_lut_f64x<false, false>(f, uint64_t(q[c0 + x]), s_lut);
                    else c = quire_word_to_posit_bf(f, q[c0 + x]);
                    codes[x] = nar ? (1u << (f.nbits - 1)) : c;
                }
                if (vec_ok) {
                    store_codes8(out.base + row * out.ldc + col0, codes, valid, true);
                } else {
                    const int64_t cs = out.col_stride();
                    CodeT* dst = out.base + out.row_base(row) + col0 * cs;
                    if (cs == 1) {  // contiguous columns (Linear layers): one vector store
                        store_codes8(dst, codes, valid,
                                     (reinterpret_cast<uintptr_t>(dst) & (8 * sizeof(CodeT) - 1)) == 0);
                    } else {
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            if (x < valid) dst[x * cs] = CodeT(codes[x]);
                    }
                }
            }
        }
    }
    __syncwarp();
    ptx::tc_fence_before();
    if constexpr (kPair) ptx::cluster_sync();
    else __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        if constexpr (kPair) ptx::tmem_dealloc2<Geo::TMEM_COLS>(tmem);
        else ptx::tmem_dealloc<Geo::TMEM_COLS>(tmem);
    }
}

// Sum split-K quire partials (mod 2^W), apply NaR, round once -- or, in raw
// mode, emit the exact W-bit quire words and NaR mask (data-parallel
// gradient reduction input).
template <typename CodeT>
__global__ void quire_finalize_kernel(const unsigned __int128* __restrict__ partial, int splits,
                                      const uint8_t* __restrict__ row_nar,
                                      const uint8_t* __restrict__ col_nar, OutMap<CodeT> out,
                                      int64_t M, int64_t N, PositFmt f,
                                      unsigned __int128* __restrict__ raw_words,
                                      uint8_t* __restrict__ raw_nar) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const int64_t total = M * N;
    const unsigned __int128 one = 1;
    const unsigned __int128 wmask = f.W >= 128 ? ~(unsigned __int128)0 : ((one << f.W) - 1);
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = idx / N, j = idx % N;
        const bool nar = (row_nar != nullptr && row_nar[i]) || (col_nar != nullptr && col_nar[j]);
        // four independent chains: the split partials' loads overlap
        unsigned __int128 q = 0, q1 = 0, q2 = 0, q3 = 0;
        int s = 0;
        for (; s + 4 <= splits; s += 4) {
            q += partial[s * total + idx];
            q1 += partial[(s + 1) * total + idx];
            q2 += partial[(s + 2) * total + idx];
            q3 += partial[(s + 3) * total + idx];
        }
        for (; s < splits; ++s) q += partial[s * total + idx];
        q += q1 + q2 + q3;
        const int64_t o = out.index(i, j);
        if (o < 0) continue;  // padding row of the implicit weight gradient
        if (raw_words != nullptr) {  // raw words/NaR mask land in the output's layout
            raw_words[o] = q & wmask;
            raw_nar[o] = nar ? 1 : 0;
        }
        if (out.base != nullptr)
            out.base[o] = CodeT(nar ? (1u << (f.nbits - 1)) : quire_word_to_posit(f, q));
    }
}

// Few outputs, many splits (weight gradients of small layers: thousands of
// outputs, ~100 splits): a warp per output, lanes over the splits, 128-bit
// butterfly -- the thread-per-output loop above would be a long serial chain
// of dependent loads on a handful of blocks.
template <typename CodeT>
__global__ void __launch_bounds__(256) quire_finalize_warp_kernel(
    const unsigned __int128* __restrict__ partial, int splits, const uint8_t* __restrict__ row_nar,
    const uint8_t* __restrict__ col_nar, OutMap<CodeT> out, int64_t M, int64_t N, PositFmt f,
    unsigned __int128* __restrict__ raw_words, uint8_t* __restrict__ raw_nar) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const int64_t total = M * N;
    const unsigned __int128 one = 1;
    const unsigned __int128 wmask = f.W >= 128 ? ~(unsigned __int128)0 : ((one << f.W) - 1);
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t idx = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; idx < total; idx += nw) {
        unsigned __int128 q = 0;
        for (int sp = lane; sp < splits; sp += 32) q += partial[sp * total + idx];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t l2 = __shfl_xor_sync(0xFFFFFFFFu, uint64_t(q), o);
            const uint64_t h2 = __shfl_xor_sync(0xFFFFFFFFu, uint64_t(q >> 64), o);
            q += (unsigned __int128)l2 | ((unsigned __int128)h2 << 64);
        }
        if (lane != 0) continue;
        const int64_t i = idx / N, j = idx - (idx / N) * N;
        const bool nar = (row_nar != nullptr && row_nar[i]) || (col_nar != nullptr && col_nar[j]);
        const int64_t o = out.index(i, j);
        if (o < 0) continue;
        if (raw_words != nullptr) {
            raw_words[o] = q & wmask;
            raw_nar[o] = nar ? 1 : 0;
        }
        if (out.base != nullptr)
            out.base[o] = CodeT(nar ? (1u << (f.nbits - 1)) : quire_word_to_posit(f, q));
    }
}

// Many splits: a block = 32 consecutive outputs x 8 split groups.  Loads are
// coalesced along the outputs (32 x 16 bytes per warp instruction), every
// thread runs two independent chains over its splits, and the 8 group sums
// meet in shared memory -- exact 128-bit integer sums, any order.
template <typename CodeT>
__global__ void __launch_bounds__(256) quire_finalize_2d_kernel(
    const unsigned __int128* __restrict__ partial, int splits, const uint8_t* __restrict__ row_nar,
    const uint8_t* __restrict__ col_nar, OutMap<CodeT> out, int64_t M, int64_t N, PositFmt f,
    unsigned __int128* __restrict__ raw_words, uint8_t* __restrict__ raw_nar) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    __shared__ unsigned __int128 s_q[8][32];
    const int64_t total = M * N;
    const int x = threadIdx.x & 31, y = threadIdx.x >> 5;
    const int64_t idx = blockIdx.x * int64_t(32) + x;
    unsigned __int128 q0 = 0, q1 = 0;
    if (idx < total) {
        int sp = y;
        for (; sp + 8 < splits; sp += 16) {
            q0 += partial[sp * total + idx];
            q1 += partial[(sp + 8) * total + idx];
        }
        if (sp < splits) q0 += partial[sp * total + idx];
    }
    s_q[y][x] = q0 + q1;
    __syncthreads();
    if (y != 0 || idx >= total) return;
    unsigned __int128 q = s_q[0][x];
#pragma unroll
    for (int g = 1; g < 8; ++g) q += s_q[g][x];
    const unsigned __int128 one = 1;
    const unsigned __int128 wmask = f.W >= 128 ? ~(unsigned __int128)0 : ((one << f.W) - 1);
    const int64_t i = idx / N, j = idx - (idx / N) * N;
    const bool nar = (row_nar != nullptr && row_nar[i]) || (col_nar != nullptr && col_nar[j]);
    const int64_t o = out.index(i, j);
    if (o < 0) return;
    if (raw_words != nullptr) {
        raw_words[o] = q & wmask;
        raw_nar[o] = nar ? 1 : 0;
    }
    if (out.base != nullptr) out.base[o] = CodeT(nar ? (1u << (f.nbits - 1)) : quire_word_to_posit(f, q));
}

inline int grid_for(int64_t items, int threads);
int64_t variant_min_work();  // igemm.cu: work (MACs) below which no reduced-digit variant launches

// split-K finalize: the variant by shape
template <typename CodeT>
inline void launch_finalize(const unsigned __int128* partial, int splits, const uint8_t* row_nar,
                            const uint8_t* col_nar, const OutMap<CodeT>& out, int64_t M, int64_t N,
                            const PositFmt& f, unsigned __int128* raw_words, uint8_t* raw_nar,
                            cudaStream_t st) {
    const int64_t total = M * N;
    if (splits >= 8)
        launch_pdl(quire_finalize_2d_kernel<CodeT>, dim3(unsigned((total + 31) / 32)), dim3(256), 0, st, 
            partial, splits, row_nar, col_nar, out, M, N, f, raw_words, raw_nar);
    else
        launch_pdl(quire_finalize_kernel<CodeT>, dim3(grid_for(total, 256)), dim3(256), 0, st, 
            partial, splits, row_nar, col_nar, out, M, N, f, raw_words, raw_nar);
}

// ------------------------------------------------------------------ host

inline int digits_for(const PositFmt& f) {
    // smallest D with balanced capacity 127*(256^D-1)/255 >= 2^(2R)
    for (int D = 1; D <= 8; ++D) {
        const long double cap = 127.0L * (powl(256.0L, D) - 1.0L) / 255.0L;
        if (cap >= powl(2.0L, 2 * f.R)) return D < 2 ? 2 : D;
    }
    return -1;
}


inline int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// K-blocks per split: at most `cap` (int32 exactness of the group sums), and,
// when the output tiles alone cannot fill the SMs, a split count that makes
// whole waves of sms / tiles units (a partial last wave doubles the time).
inline int64_t split_kblocks(int64_t kbt, int64_t cap, int64_t tiles, int sms) {
    int64_t splits = (kbt + cap - 1) / cap;  // minimum for exactness
    if (tiles < sms && kbt >= 8) {
        const int64_t per_wave = sms / tiles;
        int64_t s = (splits + per_wave - 1) / per_wave * per_wave;
        const int64_t most = kbt / 4 > splits ? kbt / 4 : splits;  // >= 4 k-blocks each
        splits = s < most ? s : most;
    }
    const int64_t kbps = (kbt + splits - 1) / splits;
    return kbps < 1 ? 1 : kbps;
}

inline int grid_for(int64_t items, int threads) {
    int64_t b = (items + threads - 1) / threads;
    if (b > 148 * 64) b = 148 * 64;
    if (b < 1) b = 1;
    return int(b);
}

// Grid of the NaR fix-up kernels: they exit at once unless a NaR was seen
// (device flag), so launch few blocks (grid-stride loops cover the rest).
inline int grid_fixup(int64_t items) {
    const int g = grid_for(items, 256);
    return g < 2 * 148 ? g : 2 * 148;
}

// Arguments of one logical quire GEMM  C[m][n] = round(sum_k A[m][k] B[k][n]).
struct GemmArgs {
    PositFmt f;
    int64_t M, N, K;
    int64_t max_kb_per_split;  // 0: automatic (int32 exactness + SM fill)
    bool row_nar, col_nar;     // apply operand NaR flags in the epilogue
    unsigned __int128* raw_words = nullptr;  // raw mode: exact W-bit quire words out
    uint8_t* raw_nar = nullptr;              //           and the NaR mask
    bool pack_b = true;  // false: B's digit image, column NaR flags and B flags are already in
                         // the workspace (an earlier launch with the same plan layout and B)
};

template <int D>
inline QuireGemmPlan plan_for(const PositFmt& f, int64_t M, int64_t N, int64_t K,
                              int64_t max_kb_per_split, bool raw) {
    using Geo = Geometry<D>;
    QuireGemmPlan p{};
    p.D = D;
    p.NT = Geo::NT;
    p.KB = Geo::KB;
    p.mtiles = (M + kBM - 1) / kBM;
    p.ntiles = (N + Geo::NT - 1) / Geo::NT;
    p.kbt = (K + Geo::KB - 1) / Geo::KB;
    // int32 group sums stay exact for K <= 131071 / D (|digit| <= 128); a
    // quire of W <= 32 bits is itself mod 2^32, so wrapping is exact there.
    int64_t kbps = f.W <= 32 ? p.kbt : (131071 / D) / Geo::KB;
    if (max_kb_per_split > 0)
        kbps = kbps < max_kb_per_split ? kbps : max_kb_per_split;
    else
        kbps = split_kblocks(p.kbt, kbps < 1 ? 1 : kbps, p.mtiles * p.ntiles, num_sms());
    if (kbps < 1) kbps = 1;
    p.kb_per_split = p.kbt < kbps ? p.kbt : kbps;
    p.splits = (p.kbt + p.kb_per_split - 1) / p.kb_per_split;
    // CTA pairs (cta_group::2) are opt-in (PNN_B200_PAIR=1): measured on B200
    // they cost more in cross-CTA stage hand-off bubbles (tensor pipe 79% vs
    // 92% active, profiles/README.md) than they save in shared-memory traffic.
    static const bool want_pair = getenv("PNN_B200_PAIR") != nullptr;
    p.pair = (p.mtiles >= 2 && want_pair) ? 1 : 0;
    p.mtiles_alloc = p.pair ? (p.mtiles + 1) / 2 * 2 : p.mtiles;
    p.a_img_bytes = size_t(p.mtiles_alloc) * p.kbt * Geo::A_BYTES;
    p.b_img_bytes = size_t(p.ntiles) * p.kbt * Geo::B_BYTES;
    p.row_nar_bytes = size_t(p.mtiles_alloc) * kBM;
    p.col_nar_bytes = size_t(p.ntiles) * Geo::NT;
    p.partial_bytes = (p.splits > 1 || raw) ? size_t(p.splits) * M * N * 16 : 0;
    p.smem_bytes = Geo::SMEM;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    p.off_a = take(p.a_img_bytes);
    p.off_b = take(p.b_img_bytes);
    p.off_row_nar = take(p.row_nar_bytes);
    p.off_col_nar = take(p.col_nar_bytes);
    p.off_flags = take(16);
    p.off_glut = take(0);
    p.off_partial = take(p.partial_bytes);
    p.workspace_bytes = off;
    return p;
}

inline int plan_quire_gemm(const PositFmt& f, int64_t M, int64_t N, int64_t K,
                           int64_t max_kb_per_split, bool raw, QuireGemmPlan* plan) {
    if (f.nbits < 2 || f.nbits > 16 || f.es < 0 || 2 * f.R > 56) return 2;
    switch (digits_for(f)) {
        case 2: *plan = plan_for<2>(f, M, N, K, max_kb_per_split, raw); break;
        case 3: *plan = plan_for<3>(f, M, N, K, max_kb_per_split, raw); break;
        case 4: *plan = plan_for<4>(f, M, N, K, max_kb_per_split, raw); break;
        case 5: *plan = plan_for<5>(f, M, N, K, max_kb_per_split, raw); break;
        case 6: *plan = plan_for<6>(f, M, N, K, max_kb_per_split, raw); break;
        case 7: *plan = plan_for<7>(f, M, N, K, max_kb_per_split, raw); break;
        case 8: *plan = plan_for<8>(f, M, N, K, max_kb_per_split, raw); break;
        default: return 2;
    }
    // the kernels index tiles in 32 bits
    if (plan->mtiles_alloc * plan->ntiles * plan->splits >= (int64_t(1) << 31)) return 2;
    return 0;
}

// A packed operand image as a 2-D uint8 tensor of 256-byte rows, box = one
// stage's bytes (rows of the box = bytes / 256): the CTA-pair producer's
// cp.async.bulk.tensor boxes.  (Driver entry point, resolved once.)
inline bool encode_rows256(CUtensorMap* m, const void* base, size_t bytes, int box_bytes) {
    using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Enc enc = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return Enc(nullptr);
        return reinterpret_cast<Enc>(fn);
    }();
    if (enc == nullptr || bytes % 256 || box_bytes % 256 || box_bytes / 256 > 256) return false;
    const cuuint64_t dims[2] = {256, cuuint64_t(bytes / 256)};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t box[2] = {256, cuuint32_t(box_bytes / 256)};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Digit words of every code of f, for the life of the process (tables.h; the
// key and contents of igemm.cu's table for the same (D, f -> f)).
template <int D>
inline const uint32_t* pack_digit_table(const PositFmt& f, cudaStream_t st) {
    return static_cast<const uint32_t*>(persistent_table(
        table_key(1, D, f.nbits, f.es, f.nbits, f.es), (size_t(2) << f.nbits) * 4, st,
        [&](void* p, cudaStream_t s) { digit_lut_kernel<D><<<16, 256, 0, s>>>(f, static_cast<uint32_t*>(p)); }));
}

// PNN_GEMM_DEBUG (profiling builds with -DPNN_GEMM_DEBUG_HOOKS): 1 = no TMEM
// loads in the epilogue, 2 = no rounding / stores; results are then garbage
inline int gemm_debug_bits() {
#ifdef PNN_GEMM_DEBUG_HOOKS
    const char* v = getenv("PNN_GEMM_DEBUG");
    return v ? (atoi(v) & 3) << 8 : 0;
#else
    return 0;
#endif
}

// PNN_DIRECT_PACK=0: the shared-memory-tile pack for plain matrices too (A/B experiments)
inline bool direct_pack_enabled() {
    static const bool on = [] {
        const char* v = getenv("PNN_DIRECT_PACK");
        return v == nullptr || v[0] != '0';
    }();
    return on;
}

template <int D, typename CodeT, class FA, class FB>
cudaError_t launch_generic(const QuireGemmPlan& p, const GemmArgs& g, FA fa, FB fb,
                           OutMap<CodeT> out, uint8_t* ws, cudaStream_t st,
                           QuireGemmStats* stats) {
    using Geo = Geometry<D>;
    const PositFmt& f = g.f;
    int8_t* a_img = reinterpret_cast<int8_t*>(ws + p.off_a);
    int8_t* b_img = reinterpret_cast<int8_t*>(ws + p.off_b);
    uint8_t* rnar = ws + p.off_row_nar;
    uint8_t* cnar = ws + p.off_col_nar;
    uint8_t* flags = ws + p.off_flags;  // [0] any NaR in A, [1] any NaR in B
    const bool use_partial = p.splits > 1 || g.raw_words != nullptr;
    auto* partial = use_partial ? reinterpret_cast<unsigned __int128*>(ws + p.off_partial) : nullptr;
    cudaError_t e;
    if (g.pack_b) {
        if ((e = cudaMemsetAsync(rnar, 0, p.off_flags + 16 - p.off_row_nar, st)) != cudaSuccess) return e;
    } else {  // keep B's column NaR flags and flags[1], flags[3]
        if ((e = cudaMemsetAsync(rnar, 0, p.off_col_nar - p.off_row_nar, st)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(flags, 0, 1, st)) != cudaSuccess) return e;
        if ((e = cudaMemsetAsync(flags + 2, 0, 1, st)) != cudaSuccess) return e;
    }
    if (stats) cudaEventRecord(stats->ev[0], st);
    const int64_t a_work = p.mtiles_alloc * p.kbt, b_work = p.ntiles * p.kbt;  // upper bounds
    // Formats wider than the shared-memory LUT decode arithmetically: a global
    // 2^16-entry digit table (glut) measured slower for posit(16,1) (L2-latency
    // bound lookups: 176 vs 133 us for the 4096^2 pair of packs).
    const uint2* glut = nullptr;
    // reduced-digit variant (posit(12,1)-class D = 6 operands within 3 digits):
    // the packs flag wide operands in flags[2], flags[3]
    constexpr int kRed = D == 8 ? 4 : 3;
    // (D = 4: posit(8,1)-class operands within 3 digits, 9 instead of 16 digit MMAs)
    const bool reduced = ((D == 6 || D == 8) && sizeof(CodeT) == 2 || D == 4 && sizeof(CodeT) == 1) &&
                         !p.pair && g.M * g.N * g.K >= variant_min_work();  // the extra launch pays off
    const int ga = int(a_work < 148 * 8 ? a_work : 148 * 8), gb = int(b_work < 148 * 8 ? b_work : 148 * 8);
    // plain-matrix operands (GEMM entry, Linear layers): barrier-free direct pack
    const int64_t a_units = a_work * int64_t(kBM) * (Geo::KB / 16), b_units = b_work * int64_t(Geo::NT) * (Geo::KB / 16);
    constexpr bool kDirectA = FA::kVecK || FA::kVecR, kDirectB = FB::kVecK || FB::kVecR;
    const bool direct = direct_pack_enabled() && a_units < (int64_t(1) << 31) - 148 * 8 * 256 &&
                        b_units < (int64_t(1) << 31) - 148 * 8 * 256;
    // one resident wave: whole multiples of the kernel's blocks per SM
    auto dgrid = [](int64_t units, auto kern) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0) != cudaSuccess || per_sm < 1)
            per_sm = 4;
        const int64_t b = (units + 255) / 256, cap = int64_t(num_sms()) * per_sm;
        return int(b < cap ? b : cap);
    };
    const bool f161 = D == 8 && sizeof(CodeT) == 2 && fixed_fmt_id(f) == 4;  // posit(16,1): compile-time decode
    // 11-12-bit formats: the process-lifetime digit table (32 KB: L1-resident
    // lookups instead of ~30 ALU instructions per code); null while capturing
    // before it exists -> the in-register decode, same digits
    const uint2* dlut = (direct && f.nbits > kLutMaxBits && f.nbits <= 12)
                            ? reinterpret_cast<const uint2*>(pack_digit_table<D>(f, st))
                            : nullptr;
    bool a_done = false, b_done = !g.pack_b;
    constexpr int kRows4 = 4 / int(sizeof(CodeT));  // rows per 4-byte load (r-contiguous operands)
    auto launch_direct = [&](auto fx, auto rows_c, int64_t rows, int8_t* dimg, uint8_t* dnar, uint8_t* dany,
                             int64_t work, int64_t units, uint8_t* wflag) {
        using FX = decltype(fx);
        constexpr int RW = decltype(rows_c)::value;
        constexpr int kF = D == 8 ? 4 : 0;
        void (*k)(FX, int64_t, int64_t, PositFmt, int8_t*, uint8_t*, uint8_t*, uint32_t, FastDiv, const uint2*,
                  uint8_t*, int) = f161 ? pack_direct_kernel<D, RW, CodeT, FX, kF, 1> : pack_direct_kernel<D, RW, CodeT, FX, 0, 1>;
        int64_t steps = units;
        if constexpr (FX::kVecR) {
            // rows of 4-byte-aligned length from a 4-byte-aligned base: row groups per load
            if (fx.ld % kRows4 == 0 && (reinterpret_cast<uintptr_t>(fx.p) & 3) == 0) {
                k = f161 ? pack_direct_kernel<D, RW, CodeT, FX, kF, kRows4> : pack_direct_kernel<D, RW, CodeT, FX, 0, kRows4>;
                steps = units / kRows4;
            }
        }
        launch_pdl(k, dim3(dgrid(steps, k)), dim3(256), 0, st, fx, rows, g.K, f, dimg, dnar, dany, uint32_t(work),
                   FastDiv(uint32_t(p.kbt)), dlut, wflag, kRed);
    };
    if constexpr (kDirectA) {
        if (direct) {
            launch_direct(fa, std::integral_constant<int, kBM>{}, g.M, a_img, rnar, flags, a_work, a_units,
                          reduced ? flags + 2 : nullptr);
            a_done = true;
        }
    }
    if constexpr (kDirectB) {
        if (direct && !b_done) {
            launch_direct(fb, std::integral_constant<int, Geo::NT>{}, g.N, b_img, cnar, flags + 1, b_work, b_units,
                          reduced ? flags + 3 : nullptr);
            b_done = true;
        }
    }
    if (f161) {
        if (!a_done)
            launch_pdl(pack_kernel<D, kBM, CodeT, FA, 4>, dim3(ga), dim3(256), 0, st, fa, g.M, g.K, f, a_img, rnar, flags,
                       p.mtiles_alloc, p.kbt, glut, reduced ? flags + 2 : nullptr, kRed);
        if (!b_done)
            launch_pdl(pack_kernel<D, Geo::NT, CodeT, FB, 4>, dim3(gb), dim3(256), 0, st, fb, g.N, g.K, f, b_img, cnar,
                       flags + 1, p.ntiles, p.kbt, glut, reduced ? flags + 3 : nullptr, kRed);
    } else {
        if (!a_done)
            launch_pdl(pack_kernel<D, kBM, CodeT, FA>, dim3(ga), dim3(256), 0, st, fa, g.M, g.K, f, a_img, rnar, flags,
                       p.mtiles_alloc, p.kbt, glut, reduced ? flags + 2 : nullptr, kRed);
        if (!b_done)
            launch_pdl(pack_kernel<D, Geo::NT, CodeT, FB>, dim3(gb), dim3(256), 0, st, fb, g.N, g.K, f, b_img, cnar,
                       flags + 1, p.ntiles, p.kbt, glut, reduced ? flags + 3 : nullptr, kRed);
    }
    if (stats) cudaEventRecord(stats->ev[1], st);
    // D <= 3 implies R <= 11, hence W <= 64: no 128-bit instantiation needed.
    using KernFn = void (*)(const int8_t*, const int8_t*, int64_t, int64_t, const uint8_t*,
                            const uint8_t*, OutMap<CodeT>, int64_t, int64_t, PositFmt,
                            unsigned __int128*, int64_t, int64_t, int64_t, const uint8_t*, int, CUtensorMap,
                            CUtensorMap);
    KernFn kern;
    // CTA pairs: 2-D tensor maps over the packed images (256-byte rows; boxes
    // = one CTA's A tile / half B tile per stage); unused otherwise
    CUtensorMap tmA{}, tmB{};
    if (p.pair) {
        if (!encode_rows256(&tmA, a_img, p.a_img_bytes, Geo::A_BYTES) ||
            !encode_rows256(&tmB, b_img, p.b_img_bytes, Geo::B_BYTES / 2))
            return cudaErrorInvalidValue;
    }
    if (p.pair) {
        if constexpr (D <= 3)
            kern = f.W <= 32 ? quire_gemm_tc_kernel<D, 1, CodeT, true>
                             : quire_gemm_tc_kernel<D, 2, CodeT, true>;
        else
            kern = f.W <= 64 ? quire_gemm_tc_kernel<D, 2, CodeT, true>
                             : quire_gemm_tc_kernel<D, 4, CodeT, true>;
    } else {
        if constexpr (D <= 3)
            kern = f.W <= 32 ? quire_gemm_tc_kernel<D, 1, CodeT, false>
                             : quire_gemm_tc_kernel<D, 2, CodeT, false>;
        else
            kern = f.W <= 64 ? quire_gemm_tc_kernel<D, 2, CodeT, false>
                             : quire_gemm_tc_kernel<D, 4, CodeT, false>;
        // BASELINE formats: epilogue specialised on the compile-time format
        const int fid = fixed_fmt_id(f);
        if constexpr (D == 2 && sizeof(CodeT) == 1)
            if (fid == 1) kern = quire_gemm_tc_kernel<2, 1, CodeT, false, 1>;
        if constexpr (D == 4 && sizeof(CodeT) == 1)
            if (fid == 2) kern = quire_gemm_tc_kernel<4, 2, CodeT, false, 2>;
        if constexpr (D == 6 && sizeof(CodeT) == 2)
            if (fid == 3) kern = quire_gemm_tc_kernel<6, 4, CodeT, false, 3>;
        if constexpr (D == 8 && sizeof(CodeT) == 2)
            if (fid == 4) kern = quire_gemm_tc_kernel<8, 4, CodeT, false, 4>;
    }
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM)) !=
        cudaSuccess)
        return e;
    const uint8_t* rn = g.row_nar ? rnar : nullptr;
    const uint8_t* cn = g.col_nar ? cnar : nullptr;
    if (p.pair) {
        const int64_t units = (p.mtiles + 1) / 2 * p.ntiles * p.splits;
        const int64_t pairs = units < num_sms() / 2 ? units : num_sms() / 2;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(2 * pairs), 1, 1);
        cfg.blockDim = dim3(kThreads, 1, 1);
        cfg.dynamicSmemBytes = Geo::SMEM;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if ((e = cudaLaunchKernelEx(&cfg, kern, (const int8_t*)a_img, (const int8_t*)b_img, p.kbt,
                                    p.kb_per_split, rn, cn, out, g.M, g.N, f, partial, p.mtiles,
                                    p.ntiles, p.splits, (const uint8_t*)nullptr, 0, tmA, tmB)) != cudaSuccess)
            return e;
    } else {
        const int64_t tiles = p.mtiles * p.ntiles * p.splits;
        const int grid = int(tiles < num_sms() ? tiles : num_sms());
        if constexpr ((D == 6 || D == 8) && sizeof(CodeT) == 2 || D == 4 && sizeof(CodeT) == 1) {
            if (reduced) {  // both launched; the pack flags let exactly one run
                // 64-bit-word variants whose 2 kRed - 1 groups fit 256 TMEM columns: two CTAs per SM
                constexpr int kCps = (D == 6 && (2 * kRed - 1) * Geo::NT <= 256) ? 2 : 1;
                using GR = Geometry<D, kRed, kCps>;
                // (128-bit word: this epilogue's quire_word_to_posit_bf takes W <= word bits)
                constexpr int kFmt = D == 4 ? 2 : D == 6 ? 3 : 4;
                // 64-bit words: posit(8,1)-class (W <= 64) and the 3-digit posit(12,1)-class
                // variant (|X| < 2^23: |sum| < 2^46 * K <= 2^61 per split, exact as int64)
                constexpr int kQW = D == 8 ? 4 : 2;
                KernFn kr = fixed_fmt_id(f) == kFmt ? quire_gemm_tc_kernel<D, kQW, CodeT, false, kFmt, kRed, kCps>
                                                    : quire_gemm_tc_kernel<D, kQW, CodeT, false, 0, kRed, kCps>;
                const int64_t slots = int64_t(kCps) * num_sms();
                const int rgrid = int(tiles < slots ? tiles : slots);
                if ((e = cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, GR::SMEM)) !=
                    cudaSuccess)
                    return e;
                launch_pdl(kr, dim3(rgrid), dim3(kThreads), GR::SMEM, st, a_img, b_img, p.kbt, p.kb_per_split, rn, cn, out, g.M,
                                                     g.N, f, partial, p.mtiles, p.ntiles, p.splits, flags + 2, 1,
                                                     tmA, tmB);
            }
        }
        launch_pdl(kern, dim3(grid), dim3(kThreads), Geo::SMEM, st, a_img, b_img, p.kbt, p.kb_per_split, rn, cn, out,
                                                g.M, g.N, f, partial, p.mtiles, p.ntiles, p.splits,
                                                reduced ? flags + 2 : nullptr, (reduced ? 2 : 0) | gemm_debug_bits(), tmA, tmB);
    }
    if (stats) cudaEventRecord(stats->ev[2], st);
    if (use_partial) {
        launch_finalize<CodeT>(partial, int(p.splits), g.row_nar ? rnar : nullptr,
                               g.col_nar ? cnar : nullptr, out, g.M, g.N, f, g.raw_words, g.raw_nar, st);
    }
    if (stats) cudaEventRecord(stats->ev[3], st);
    return cudaGetLastError();
}

// 0 ok, 2 unsupported format, 3 workspace too small, 4 CUDA error.
template <typename CodeT, class FA, class FB>
int run_quire_gemm(const GemmArgs& g, FA fa, FB fb, OutMap<CodeT> out, void* workspace,
                   size_t workspace_bytes, cudaStream_t st, QuireGemmStats* stats) {
    QuireGemmPlan p;
    if (plan_quire_gemm(g.f, g.M, g.N, g.K, g.max_kb_per_split, g.raw_words != nullptr, &p))
        return 2;
    if (workspace_bytes < p.workspace_bytes) return 3;
    auto* ws = static_cast<uint8_t*>(workspace);
    cudaError_t e = cudaSuccess;
    switch (p.D) {
        case 2: e = launch_generic<2, CodeT>(p, g, fa, fb, out, ws, st, stats); break;
        case 3: e = launch_generic<3, CodeT>(p, g, fa, fb, out, ws, st, stats); break;
        case 4: e = launch_generic<4, CodeT>(p, g, fa, fb, out, ws, st, stats); break;
        case 5: e = launch_generic<5, CodeT>(p, g, fa, fb, out, ws, st, stats); break;
        case 6: e = launch_generic<6, CodeT>(p, g, fa, fb, out, ws, st, stats); break;
        case 7: e = launch_generic<7, CodeT>(p, g, fa, fb, out, ws, st, stats); break;
        case 8: e = launch_generic<8, CodeT>(p, g, fa, fb, out, ws, st, stats); break;
        default: return 2;
    }
    return e == cudaSuccess ? 0 : 4;
}

template <typename CodeT>
inline OutMap<CodeT> out_rowmajor(void* base, int64_t ldc) {
    OutMap<CodeT> o{};
    o.base = static_cast<CodeT*>(base);
    o.ldc = ldc;
    o.inner = 1;
    o.ncols = 0;
    o.mode = 0;
    return o;
}

template <typename CodeT>
inline OutMap<CodeT> out_nchw(void* base, int64_t pixels, int64_t channels) {
    OutMap<CodeT> o{};
    o.base = static_cast<CodeT*>(base);
    o.ldc = 0;
    o.inner = pixels;
    o.ncols = channels;
    o.mode = 1;
    if (pixels < (int64_t(1) << 31)) o.fd_inner = FastDiv(uint32_t(pixels));
    return o;
}

}  // namespace pnn_b200
