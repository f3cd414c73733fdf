// Implicit-GEMM convolution on the tcgen05 quire core: the im2col gather is
// done by the TMA engine, not by a pack pass.
//
// Activations (and output gradients) are digitised ONCE per call into a
// position-major digit tensor  dig[D][N][H][W][Cp]  (Cp = channels rounded up
// to 32; one byte per balanced int8 digit, same digits as the pack path).  A
// convolution tap is then a shifted box of that tensor: a 5-D TMA tile load
// {32 channels, W, Hb, Nb, D planes} at signed coordinates, whose out-of-range
// elements the TMA unit zero-fills -- exactly the convolution's zero padding
// (tensor_ops.cpp:274-279, 546-554, 590-596).  HBM traffic per stage is the
// digit bytes of the box, not KH*KW copies of every element.
//
//   mode 0  forward      M = output pixels (n,oy,ox)   N = F   K = (tap, c)   both K-major
//   mode 1  input grad   M = input pixels (n,iy,ix)    N = C   K = (tap, f)   both K-major
//   mode 2  weight grad  M = (tap, c)                  N = F   K = (n,oy,ox)  both MN-major
//
// K-major modes use the 32-byte-swizzled UMMA layout (one 32-channel chunk of
// one tap per pipeline stage = one i8 MMA K-step); mode 2 reads the same
// position-major tensors as MN-major operands (swizzle = channel bytes).
// Accumulation, TMEM grouping, split-K and the quire epilogue are those of
// quire_gemm_core.cuh.  The forward bias enters the quire in the epilogue as
// X_bias * 2^R (= bias * 1.0, tensor_ops.cpp:292).
#pragma once

#include <cuda.h>

#include "epilogue.cuh"
#include "fastdiv.cuh"
#include "pdl.cuh"
#include "igemm.h"
#include "posit_scalar.cuh"
#include "quire_gemm_core.cuh"

// PNN_IGEMM_DEBUG_HOOKS: compile the epilogue's profiling switches (a.debug
// bits 1, 8, 16; tools/igemm_bottleneck.sh).  Off in the product build: they
// cost branches in the per-output loop.
#ifdef PNN_IGEMM_DEBUG_HOOKS
#define PNN_EPI_DEBUG(bit) (a.debug & (bit))
#else
#define PNN_EPI_DEBUG(bit) false
#endif

namespace pnn_b200 {

constexpr int kIKB = 32;         // K bytes (channels or pixels) per pipeline stage
constexpr int kActLutBits = 12;  // digitiser LUT up to 4096 codes (32 KB, L1-resident)

// Tile geometry.  CPS = CTAs per SM.  CPS 2 (the forward / input-grad passes):
// each CTA owns 256 TMEM columns and ~100 KB of stages, so two tiles are in
// flight per SM -- one CTA's TMEM drain and rounding overlap the other's MMAs
// (a single CTA cannot double-buffer G*NT > 256 columns).  CPS 1 (weight grad,
// whose few output tiles run long split-K loops): 512 columns, ~200 KB.
// DA: digit planes of the A operand (== D except in the weight gradient fed by
// the forward pass's saved activation digits of a narrower, exactly widening
// format: DA planes whose groups land OFF digit positions up, igemm_kernel).
// DB: digit planes of the B operand (== D except for an input gradient whose
// weights all fit DB < D digits, run_dgrad's device-selected variant).
template <int D, int NT_, int CPS, int ACC = 1, int DA = D, int DB = D>
struct ImplGeo {
    static constexpr int NT = NT_;
    static constexpr int G = DA + DB - 1;
    static constexpr int NMMA = DB * NT;
    static constexpr int A_BYTES = DA * kBM * kIKB;
    static constexpr int B_BYTES = DB * NT * kIKB;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int BUDGET = CPS == 2 ? 104 * 1024 : 200 * 1024;
    static constexpr int STAGES_FIT = BUDGET / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT > 12 ? 12 : STAGES_FIT;
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + kZeroBytes + 256;
    static constexpr uint32_t TMEM_COLS = CPS == 2 ? 256 : 512;
    // ACC = 2: two accumulator buffers (at columns 0 and 256): tile t+1's MMAs
    // run while the epilogue drains and rounds tile t.
    static constexpr int ACC_STRIDE = 256;
    static constexpr int EPI = CPS == 2 ? 8 : 16;  // epilogue warps
    static constexpr int THREADS = 64 + 32 * EPI;
    static_assert(G * NT <= (ACC == 2 ? ACC_STRIDE : int(TMEM_COLS)), "TMEM overflow");
    static_assert(ACC == 1 || CPS == 1, "double buffering needs the whole TMEM");
    static_assert(DA >= 1 && DB >= 1 && DB <= D, "digit planes");
    static_assert(NMMA % 16 == 0 && NMMA <= 256, "bad UMMA N");
    static_assert(STAGES >= 2, "pipeline depth");
    static_assert(A_BYTES % 1024 == 0 && B_BYTES % 512 == 0, "stage alignment");
};

// N tile of the two-CTAs-per-SM passes: G * NT <= 256 TMEM columns
__host__ __device__ constexpr int small_nt(int D) { return D == 2 ? 64 : D <= 4 ? 32 : 16; }

struct IgemmArgs {
    int64_t M, N;
    int64_t mtiles, ntiles, kbt, kb_per_split, splits;
    // modes 0/1: m-tile -> (n0, y0) of the output-pixel raster
    int tiles_per_img;  // > 0: an image spans tiles_per_img tiles of Hb rows
    int imgs_per_tile;  // tiles_per_img == 0: a tile holds imgs_per_tile images
    int Hb;
    int KW, pad, cch;   // taps' width, padding, 32-wide chunks per tap
    // mode 2: K blocks of OWb x OHb output pixels; m-tile = one ky, 4 kx, 32 channels
    int taps, C, OWb, OHb, kpr, kpi;  // k-blocks per row-block set / per image
    int KH, kgroups, cgroups, Hp;     // kx groups of 4, 32-channel groups, padded height
    int apad;  // mode 0: zero ring stored around the A digits (box coordinates shift by it)
    const uint8_t* vflag;  // variant selection (see igemm_kernel): run iff (*vflag != 0) == vexpect
    int vexpect;           // and (*vflag2 != 0) == vexpect2 (null flags: no condition)
    const uint8_t* vflag2;
    int vexpect2;
    int vor;               // 1: run iff (*vflag | *vflag2 != 0) == vexpect
    int nowrap;     // 64-bit quire words: |sum| < 2^(W-1) for this pass, q is the exact value
    int relu;       // mode 0: output relu(y) (ReLU layer fused) ...
    void* pre_out;  // ... and, if non-null, the pre-activation y here (same layout)
    // tile raster (tile_coords) with launch-constant divisions: by mtiles * ntiles,
    // by kGroupM * ntiles, and by the group height (kGroupM, or the last group's)
    FastDiv fd_split, fd_group, fd_g8, fd_glast;
    const int64_t* col_add;  // mode 0: X(bias) per column (added as X * 2^R)
    const uint8_t* col_nar;
    PositFmt f;
    unsigned __int128* partial;
    int debug;  // profiling only (PNN_IGEMM_DEBUG): 1 skip conversion, 2 skip MMA, 4 skip TMA waits
};

// tile_coords (quire_gemm_core.cuh) with the divisions precomputed per launch.
__device__ __forceinline__ void itile_coords(int64_t t64, const IgemmArgs& a, int64_t& split,
                                             int64_t& mt, int64_t& nt) {
    uint32_t sp, r, group, within, q, rem;
    a.fd_split.divmod(uint32_t(t64), sp, r);
    a.fd_group.divmod(r, group, within);
    const uint32_t left = uint32_t(a.mtiles) - group * kGroupM;
    (left < uint32_t(kGroupM) ? a.fd_glast : a.fd_g8).divmod(within, q, rem);
    split = sp;
    mt = group * kGroupM + rem;
    nt = q;
}

// quire word -> posit code in the epilogue: 64-bit words through the FP64
// converter (PNN_EPI_INT_ROUND: the integer leading-one search), the other
// widths through the integer paths
#ifndef PNN_EPI_INT_ROUND
__device__ __forceinline__ uint32_t epi_round(const PositFmt& f, uint64_t q, const uint4* lut) {
    return q_to_posit_lut_f64x<false, false>(f, q, lut);
}
#else
__device__ __forceinline__ uint32_t epi_round(const PositFmt& f, uint64_t q, const uint4* lut) {
    return q_to_posit_lut(f, q, lut);
}
#endif
__device__ __forceinline__ uint32_t epi_round(const PositFmt& f, uint32_t q, const uint4* lut) {
    return q_to_posit_lut(f, q, lut);
}
__device__ __forceinline__ uint32_t epi_round(const PositFmt& f, unsigned __int128 q, const uint4* lut) {
    return q_to_posit_lut(f, q, lut);
}

// Epilogue warps: 8 (two CTAs per SM) or 16 (one): the epilogue (TMEM drain,
// quire accumulation, quire -> posit) is latency-bound, so it gets the warps.
//
// DA / OFF (mode 2 only): the A operand has DA digit planes of X_A * 256^-OFF
// (the saved forward digits of an exactly widening format, X_g = X_f *
// 2^(R_g - R_f), R_g - R_f = 8 * OFF); MMA group g is digit position g + OFF.
template <int D, int NT_, int CPS, int ACC, int QW, typename CodeT, int MODE, int FMT = 0,
          int DA = D, int OFF = 0, int DB = D>
__global__ void __launch_bounds__(ImplGeo<D, NT_, CPS, ACC, DA, DB>::THREADS, CPS)
    igemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const IgemmArgs a, const OutMap<CodeT> out) {
    static_assert(MODE == 2 || OFF == 0, "digit offset: weight gradient only");
    using Geo = ImplGeo<D, NT_, CPS, ACC, DA, DB>;
    pdl_trigger();  // the next kernel's CTAs may start their prologue in this grid's tail
    constexpr int kIEpiWarps = Geo::EPI;
    constexpr int kIThreads = Geo::THREADS;
    using QT = typename QuireWord<QW>::T;
    constexpr int NT = Geo::NT, STAGES = Geo::STAGES, G = Geo::G;
    constexpr int SUB = kIEpiWarps / 4;  // warps per lane quarter
    constexpr int COLS = NT / SUB;       // columns per epilogue thread
    static_assert(COLS % 8 == 0, "epilogue chunks");
    constexpr int GB = G < 4 ? G : 4;  // TMEM loads per wait (registers)
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint4 s_lut[kPackLutEntries];  // per-scale rounding table (epilogue)
    uint8_t* smem = smem_raw + ((1024 - (ptx::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t* zero_tile = smem + STAGES * Geo::STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(zero_tile + kZeroBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;      // [ACC]
    uint64_t* tmem_empty = tmem_full + ACC;    // [ACC]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + ACC);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t tiles = a.mtiles * a.ntiles * a.splits;

    for (int i = threadIdx.x; i < kZeroBytes / 16; i += kIThreads)
        reinterpret_cast<int4*>(zero_tile)[i] = make_int4(0, 0, 0, 0);
    build_pack_lut(fixed_fmt<FMT>(a.f), s_lut, threadIdx.x, kIThreads);
    // 8-bit outputs from 64-bit words: the rounding as one table (epilogue.cuh)
    constexpr bool kTab8 = sizeof(CodeT) == 1 && QW <= 2;
    __shared__ uint8_t s_tab8[kTab8 ? kTab8Bytes : 1];
    if constexpr (kTab8) {
        __syncthreads();
        build_pack_tab8(fixed_fmt<FMT>(a.f), s_lut, s_tab8, threadIdx.x, kIThreads);
    }
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < ACC; ++b) {
            ptx::mbar_init(&tmem_full[b], 1);
            ptx::mbar_init(&tmem_empty[b], kIEpiWarps);
        }
        ptx::fence_barrier_init();
    }
    // everything above touched only shared memory and parameters (PDL prologue)
    pdl_wait();
    // device-selected variant: exit at once unless the flag (written by the
    // weight digitiser on this stream) matches
    if (a.vor) {  // run iff (either flag set) == vexpect
        if (int(*a.vflag != 0 || *a.vflag2 != 0) != a.vexpect) return;
    } else {
        if (a.vflag != nullptr && int(*a.vflag != 0) != a.vexpect) return;
        if (a.vflag2 != nullptr && int(*a.vflag2 != 0) != a.vexpect2) return;
    }
    if (warp == 1) ptx::tmem_alloc<Geo::TMEM_COLS>(tmem_slot);
    // forward bias: X(bias) * 2^R per column, once per CTA in shared memory
    // (zero past N: the epilogue adds without bounds tests)
    constexpr int kColSmem = MODE == 0 ? 256 : 1;
    __shared__ int64_t s_colx[kColSmem];
    const bool col_smem = MODE == 0 && a.col_add != nullptr && a.N <= kColSmem;
    if (col_smem)
        for (int i = threadIdx.x; i < kColSmem; i += kIThreads) {
            const int64_t xb = i < a.N ? a.col_add[i] : 0;
            s_colx[i] = QW <= 2 ? int64_t(uint64_t(xb) << fixed_fmt<FMT>(a.f).R) : xb;
        }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ===== producer: TMA tile boxes (the im2col gather) =====
            // Slice layout: every box row is a run of pixels x 16 channel bytes,
            // contiguous in HBM (up to 2 KB), so a stage is a few dozen requests.
            // The stage index / phase and the k-block's tap / chunk / pixel-block
            // coordinates are running counters (one division set per tile, none
            // per k-block): this single thread's instruction chain, not the TMA
            // unit, paced the short K loops of the convolution tiles.
            int s = 0;
            uint32_t ph = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                int64_t split, mt, nt;
                itile_coords(t, a, split, mt, nt);
                const int64_t kb0 = split * a.kb_per_split;
                const int nkb = int(min(a.kbt, kb0 + a.kb_per_split) - kb0);
                int n0 = 0, y0 = 0;
                if (MODE != 2) {
                    if (a.tiles_per_img > 0) {
                        n0 = int(mt) / a.tiles_per_img;
                        y0 = (int(mt) % a.tiles_per_img) * a.Hb;
                    } else {
                        n0 = int(mt) * a.imgs_per_tile;
                    }
                }
                // modes 0/1: k-block = (tap (ky, kx), 32-channel chunk cc)
                int cc = 0, kx = 0, ky = 0;
                // mode 2: k-block = (image n, pixel-row block yb, pixel-column block xb);
                // the m-tile's (ky, kx group, channel group) is fixed per tile
                int wn = 0, wy = 0, wx = 0, mky = 0, mkg = 0, mcg = 0;
                if constexpr (MODE != 2) {
                    const int tap = int(kb0) / a.cch;
                    cc = int(kb0) - tap * a.cch;
                    ky = tap / a.KW;
                    kx = tap - ky * a.KW;
                } else {
                    wn = int(kb0) / a.kpi;
                    const int r = int(kb0) - wn * a.kpi;
                    wy = r / a.kpr;
                    wx = r - wy * a.kpr;
                    const int kc = a.kgroups * a.cgroups;
                    mky = int(mt) / kc;
                    mkg = (int(mt) % kc) / a.cgroups;
                    mcg = int(mt) % a.cgroups;
                }
                const int kpc = MODE == 2 ? a.kpi / a.kpr : 0;  // pixel-row blocks per image
                for (int i = 0; i < nkb; ++i) {
                    ptx::mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* sa = smem + s * Geo::STAGE_BYTES;
                    uint8_t* sb = sa + Geo::A_BYTES;
                    uint64_t* fb = &full[s];
                    if (++s == STAGES) s = 0, ph ^= 1;
                    if (a.debug & 4) {  // profiling: no operand traffic
                        ptx::mbar_arrive(fb);
                        continue;
                    }
                    ptx::mbar_arrive_expect_tx(fb, Geo::STAGE_BYTES);
                    if constexpr (MODE != 2) {
                        // A box {w, h, n, 2 slices, D} -> [D][2][pixels][16 B]
                        if constexpr (MODE == 0)  // apad: zero ring stored around the digits
                            ptx::tma_load_5d(sa, &tmA, 2 * (kx - a.pad + a.apad), y0 + ky - a.pad + a.apad,
                                             n0, 2 * cc, 0, fb);
                        else
                            ptx::tma_load_5d(sa, &tmA, 2 * (a.pad - kx), y0 + a.pad - ky, n0, 2 * cc, 0, fb);
                        // B box {NT rows, D, 2 slices} -> [2][D][NT][16 B]
                        ptx::tma_load_3d(sb, &tmB, 2 * int(nt) * NT, 0, 2 * int(kb0 + i), fb);
                        if (++cc == a.cch) {
                            cc = 0;
                            if (++kx == a.KW) kx = 0, ++ky;
                        }
                    } else {
                        const int yb = wy * a.OHb, xb = wx * a.OWb;
                        // A: ONE box {pixels, rows, 4 kx taps, 2 slices, D} of the
                        // zero-padded x digits; the kx dimension is an overlapping view
                        // (stride = one 16-byte pixel) -> [D][2][4][OHb][OWb][16 B]
                        ptx::tma_load_5d(sa, &tmA, 2 * (xb + 4 * mkg), wn * a.Hp + yb + mky, 0, 2 * mcg, 0, fb);
                        // B box {pixels, rows, 1, NT/16 slices, D} -> [D][NT/16][32][16 B]
                        ptx::tma_load_5d(sb, &tmB, 2 * xb, yb, wn, int(nt) * (NT / 16), 0, fb);
                        if (++wx == a.kpr) {
                            wx = 0;
                            if (++wy == kpc) wy = 0, ++wn;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer (no-swizzle canonical layouts, 16-byte core rows) =====
            constexpr uint32_t idesc = ptx::idesc_i8(kBM, Geo::NMMA, MODE == 2, MODE == 2);
            // all-zero A operand for initialising groups D-1 .. 2D-2; footprint <= 4 KB
            const uint64_t zdesc = MODE == 2 ? ptx::smem_desc_kmajor(ptx::smem_u32(zero_tile), 128, 512)
                                             : ptx::smem_desc_kmajor(ptx::smem_u32(zero_tile), 128, 256);
            uint32_t j = 0, ph = 0;
            int s = 0;
            const uint32_t smem0 = ptx::smem_u32(smem);
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
                int64_t split, mt, nt;
                itile_coords(t, a, split, mt, nt);
                const int64_t kb0 = split * a.kb_per_split;
                const int nkb = int(min(a.kbt, kb0 + a.kb_per_split) - kb0);
                const int buf = ACC == 2 ? int(j & 1) : 0;
                const uint32_t jb = ACC == 2 ? (j >> 1) : j;  // uses of this buffer so far
                ptx::mbar_wait(&tmem_empty[buf], (jb & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t tacc = tmem + buf * Geo::ACC_STRIDE;
                for (int i = 0; i < nkb; ++i) {
                    ptx::mbar_wait(&full[s], ph);
                    ptx::tc_fence_after();
                    const uint32_t a_base = smem0 + s * Geo::STAGE_BYTES;
                    uint64_t* eb = &empty[s];
                    if (++s == STAGES) s = 0, ph ^= 1;
                    const uint32_t b_base = a_base + Geo::A_BYTES;
                    // K-major: LBO = next 16 K bytes (next slice), SBO = next 8 rows (128 B).
                    // MN-major: LBO = next 8 K rows (128 B), SBO = next 16-wide MN atom.
                    const uint64_t bdesc = MODE == 2
                                               ? ptx::smem_desc_kmajor(b_base, 128, kIKB * 16)
                                               : ptx::smem_desc_kmajor(b_base, DB * NT * 16, 128);
                    const bool first = i == 0;
                    if (first) {  // zero groups DB .. G-1 (plane 0's MMA initialises 0 .. DB-1)
#pragma unroll
                        for (int z = DB; z < Geo::G; z += DB) {
                            const int off = z < Geo::G - DB ? z : Geo::G - DB;
                            ptx::mma_i8(tacc + off * NT, zdesc, bdesc, idesc, 0);
                        }
                    }
#pragma unroll
                    for (int p = 0; p < DA; ++p) {
                        const uint32_t ap = a_base + p * (kBM * kIKB);
                        const uint64_t adesc = MODE == 2 ? ptx::smem_desc_kmajor(ap, 128, kIKB * 16)
                                                         : ptx::smem_desc_kmajor(ap, kBM * 16, 128);
                        if (!(a.debug & 2))
                            ptx::mma_i8(tacc + p * NT, adesc, bdesc, idesc, (first && p == 0) ? 0u : 1u);
                    }
                    ptx::mma_commit(eb);
                }
                ptx::mma_commit(&tmem_full[buf]);
            }
        }
    } else {
        // ===== epilogue: TMEM -> quire words -> posit codes / split-K partials =====
        const int quarter = warp & 3;
        const PositFmt f = fixed_fmt<FMT>(a.f);  // compile-time for the BASELINE formats
        const int sub = (warp - 2) >> 2;
        // the SUB warps of a lane quarter take interleaved 8-column chunks
        // (chunk i of warp sub = tile columns (sub + SUB * i) * 8: balanced when N < NT)
        const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16) + sub * 8;
        uint32_t j = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
            int64_t split, mt, nt;
            itile_coords(t, a, split, mt, nt);
            const int buf = ACC == 2 ? int(j & 1) : 0;
            ptx::mbar_wait(&tmem_full[buf], ((ACC == 2 ? (j >> 1) : j)) & 1);
            ptx::tc_fence_after();
            const uint32_t trow_b = trow + buf * Geo::ACC_STRIDE;
            QT q[COLS];
#pragma unroll
            for (int c0 = 0; c0 < COLS; c0 += 8) {
                QAcc2<QW> acc[8];
#pragma unroll
                for (int g0 = 0; g0 < G; g0 += GB) {
                    uint32_t r[GB][8];
#pragma unroll
                    for (int g = 0; g < GB; ++g)
                        if (g0 + g < G) {
                            if (PNN_EPI_DEBUG(8)) {
                                for (int x = 0; x < 8; ++x) r[g][x] = 0;
                            } else {
                                ptx::tmem_ld8(trow_b + (g0 + g) * NT + SUB * c0, r[g]);
                            }
                        }
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int g = 0; g < GB; ++g)
                        if (g0 + g < G)
#pragma unroll
                            for (int x = 0; x < 8; ++x) acc[x].add(g0 + g + OFF, r[g][x]);
                }
#pragma unroll
                for (int x = 0; x < 8; ++x) q[c0 + x] = acc[x].get();
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tmem_empty[buf]);
            if (PNN_EPI_DEBUG(16)) continue;  // profiling: no output

            const int64_t row = mt * kBM + quarter * 32 + lane;
            if (row >= a.M) continue;
            const int64_t colbase = nt * NT + sub * 8;  // chunk c0 / 8 at colbase + SUB * c0
            const int64_t obase = out.row_base(row), ostride = out.col_stride();
            if (obase < 0 && a.partial == nullptr) continue;  // padding row (weight grad)
            if constexpr (MODE == 0) if (a.col_add != nullptr && split == 0) {
                const int cb = int(colbase), nn = int(a.N);
                if (col_smem) {  // (columns past N read zeros)
#pragma unroll
                    for (int c = 0; c < COLS; ++c) {
                        const int64_t xs = s_colx[cb + SUB * (c & ~7) + (c & 7)];
                        if constexpr (QW == 4) q[c] += QT(__int128(xs)) << f.R;
                        else q[c] += QT(xs);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < COLS; ++c)
                        if (cb + SUB * (c & ~7) + (c & 7) < nn) {
                            const int64_t xb = a.col_add[cb + SUB * (c & ~7) + (c & 7)];
                            if constexpr (QW == 4) q[c] += QT(__int128(xb)) << f.R;
                            else q[c] += QT(xb) << f.R;
                        }
                }
            }
#pragma unroll
            for (int c0 = 0; c0 < COLS; c0 += 8) {
                const int64_t col0 = colbase + SUB * c0;
                if (col0 >= a.N) break;
                const int valid = int(a.N - col0 < 8 ? a.N - col0 : 8);
                if (a.partial != nullptr) {
                    unsigned __int128* dst = a.partial + (split * a.M + row) * a.N + col0;
#pragma unroll
                    for (int x = 0; x < 8; ++x)
                        if (x < valid) dst[x] = (unsigned __int128)q[c0 + x];
                    continue;
                }
                // 8 independent branch-free conversions, then predicated stores;
                // column NaR flags as one 8-byte load (buffers are 256-byte padded)
                const uint64_t cn = a.col_nar != nullptr
                                        ? *reinterpret_cast<const uint64_t*>(a.col_nar + col0)
                                        : 0ull;
                uint32_t codes[8];
#ifndef PNN_EPI_INT_ROUND
                // relu(y) is the only output: magnitude-only rounding, NaR -> 0
                const bool relu_only = MODE == 0 && (QW == 2 || kTab8) && a.relu && a.pre_out == nullptr;
                if (QW == 1 && kTab8 && relu_only && !PNN_EPI_DEBUG(1)) {
#pragma unroll
                    for (int x = 0; x < 8; ++x) codes[x] = q32_to_posit_tab8<true>(f, uint32_t(q[c0 + x]), s_tab8);
                    if (cn != 0) {  // (warp-uniform: the flags are per column)
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            if ((cn >> (8 * x)) & 0xFF) codes[x] = 0u;
                    }
                } else if (QW == 2 && relu_only && !PNN_EPI_DEBUG(1)) {
                    if (a.nowrap) {
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            codes[x] = kTab8 ? q_to_posit_tab8<true, true>(f, uint64_t(q[c0 + x]), s_tab8)
                                             : q_to_posit_lut_f64x<true, true>(f, uint64_t(q[c0 + x]), s_lut);
                    } else {
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            codes[x] = kTab8 ? q_to_posit_tab8<true, false>(f, uint64_t(q[c0 + x]), s_tab8)
                                             : q_to_posit_lut_f64x<true, false>(f, uint64_t(q[c0 + x]), s_lut);
                    }
                    if (cn != 0) {  // (warp-uniform: the flags are per column)
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            if ((cn >> (8 * x)) & 0xFF) codes[x] = 0u;
                    }
                } else
#endif
                {
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        if constexpr (kTab8 && QW == 1)
                            codes[x] = PNN_EPI_DEBUG(1) ? uint32_t(q[c0 + x])
                                                        : q32_to_posit_tab8<false>(f, uint32_t(q[c0 + x]), s_tab8);
                        else if constexpr (kTab8)
                            codes[x] = PNN_EPI_DEBUG(1) ? uint32_t(q[c0 + x])
                                                        : q_to_posit_tab8<false, false>(f, uint64_t(q[c0 + x]), s_tab8);
                        else
                            codes[x] = PNN_EPI_DEBUG(1) ? uint32_t(q[c0 + x]) : epi_round(f, q[c0 + x], s_lut);
                    }
                    if (cn != 0) {  // (warp-uniform: the flags are per column)
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            if ((cn >> (8 * x)) & 0xFF) codes[x] = 1u << (f.nbits - 1);
                    }
                }
                if constexpr (MODE == 0) if (a.relu && !relu_only) {
                    // fused ReLU (the layer after the convolution):
                    // the pre-activation to pre_out when asked, relu(y) to the output
                    if (a.pre_out != nullptr) {
                        CodeT* pd = static_cast<CodeT*>(a.pre_out) + obase + col0 * ostride;
#pragma unroll
                        for (int x = 0; x < 8; ++x)
                            if (x < valid) pd[x * ostride] = CodeT(codes[x]);
                    }
#pragma unroll
                    for (int x = 0; x < 8; ++x)
                        codes[x] = (codes[x] != 0 && ((codes[x] >> (f.nbits - 1)) & 1u) == 0) ? codes[x] : 0u;
                }
                CodeT* dst = out.base + obase + col0 * ostride;
                if (ostride == 1) {  // contiguous columns (Linear: [N][features]): one vector store
                    store_codes8(dst, codes, valid,
                                 (reinterpret_cast<uintptr_t>(dst) & (8 * sizeof(CodeT) - 1)) == 0);
                } else {
#pragma unroll
                    for (int x = 0; x < 8; ++x)
                        if (x < valid) dst[x * ostride] = CodeT(codes[x]);
                }
            }
        }
    }
    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<Geo::TMEM_COLS>(tmem);
    }
}

// ------------------------------------------------------------- digitising

// Digit words of convert(c, fs -> f) for every code c of the source format
// fs (== digit_lut_kernel when fs == f): the digitisers then read codes of
// one stage format and emit the digits of another (SURVEY.md Appendix A.6 stage
// conversions) without a separate convert pass.
template <int D>
__global__ void digit_lut_conv_kernel(PositFmt fs, PositFmt f, uint32_t* __restrict__ lut) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const bool same = fs.nbits == f.nbits && fs.es == f.es;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < (1 << fs.nbits);
         c += gridDim.x * blockDim.x) {
        uint32_t lo, hi;
        bool nar;
        digit_words<D>(same ? uint32_t(c) : p_convert(fs, f, uint32_t(c)), f, lo, hi, nar);
        lut[2 * c] = lo;
        lut[2 * c + 1] = hi;
    }
}

// Digits of 4 consecutive channels (codes c[0..3]) as one 4-byte word per
// plane in registers: words[p][q] for 4-channel group q (the caller stores
// whole 32-byte rows per plane); returns a mask of NaR codes.
template <int D, bool kSmemLut = false>
__device__ __forceinline__ uint32_t digits4_words(const uint32_t (&c)[4], const PositFmt& f,
                                                  uint32_t nar_code, const uint32_t* __restrict__ lut,
                                                  uint32_t (&words)[D][8], int q) {
    uint32_t lo[4], hi[4], nm = 0;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
        bool nar;
        if (lut != nullptr) {
            const uint2 v = kSmemLut ? reinterpret_cast<const uint2*>(lut)[c[jj]]  // shared-memory table
                                     : __ldg(reinterpret_cast<const uint2*>(lut) + c[jj]);
            lo[jj] = v.x;
            hi[jj] = v.y;
            nar = c[jj] == nar_code;
        } else {
            digit_words<D>(c[jj], f, lo[jj], hi[jj], nar);
        }
        nm |= nar ? 1u << jj : 0u;
    }
#pragma unroll
    for (int p = 0; p < D; ++p) {
        const uint32_t* w = p < 4 ? lo : hi;
        const uint32_t sel = (p & 3) | (((p & 3) + 4) << 4);
        const uint32_t a = __byte_perm(w[0], w[1], sel);
        const uint32_t b = __byte_perm(w[2], w[3], sel);
        words[p][q] = __byte_perm(a, b, 0x5410);
    }
    return nm;
}

// ReLU gate fused into a digitiser (the Conv2d backward after a ReLU layer,
// SURVEY.md Appendix A.2): code -> positive(gate) ? code : 0 with gate codes
// of the same [N][C][H][W] layout (gb bytes each, nbits gnbits).
struct DigitGate {
    const void* gate = nullptr;
    int gb = 0, gnbits = 0;
    __device__ __forceinline__ bool open(int64_t i) const {
        const uint32_t c = gb == 1 ? uint32_t(static_cast<const uint8_t*>(gate)[i])
                                   : uint32_t(static_cast<const uint16_t*>(gate)[i]);
        return c != 0 && ((c >> (gnbits - 1)) & 1u) == 0;
    }
};

// out = gated codes (the ReLU backward, when its result itself is wanted)
template <typename CodeT>
__global__ void gate_codes_kernel(const CodeT* __restrict__ dy, DigitGate gt, CodeT* __restrict__ out,
                                  int64_t n) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = gt.open(i) ? dy[i] : CodeT(0);
}

// codes [N][C][H][W] -> dig[D][N][Hp][Cp/16][Wp][16] (slice layout, balanced
// int8 digits; channels >= C are zero; Hp = H + 2 pad, Wp = W + 2 pad with the
// pad ring written as zeros by the border pixels' threads), plus NaR summaries
// written only where a NaR is found: pos_nar[n][h][w] (any channel),
// chw_nar[c][h][w] (any image), chan_nar[c], *any.  A thread owns one pixel x
// one 32-channel chunk: its 32 loads are coalesced across the warp
// (consecutive pixels of one channel plane), and it writes 32 contiguous digit
// bytes per plane (two 16-byte stores), so the warp's stores are 1 KB
// contiguous per plane.  lut: digit words per SOURCE code (digit_lut_kernel:
// the digits of convert(code, fs -> f), formats up to 12 bits) or null
// (in-register decode; then fs == f).  fs: the codes' format (NaR pattern).
// Grid: (pixel blocks, 32-channel chunks); 32-bit indices (pixels < 2^31,
// checked by the launcher) with launch-constant divisions by multiplication.
// One pixel x one 32-channel chunk: digits of code[0..31] -> the slice-layout
// cells of pixel (n, h, w) (+ the zero ring cells a border pixel owns), NaR
// summaries.  plane = bytes per digit plane.  Shared by the digitisers below.
template <int D, bool kSmemLut = false>
__device__ __forceinline__ void emit_pixel_digits(const uint32_t (&code)[32], uint32_t r, uint32_t n,
                                                  uint32_t pix, uint32_t h, uint32_t w, int cc, int C,
                                                  int H, int W, int Cp, int pad, int64_t plane,
                                                  uint32_t HW, const PositFmt& f, uint32_t nar_code,
                                                  const uint32_t* __restrict__ lut,
                                                  int8_t* __restrict__ dig, uint8_t* __restrict__ pos_nar,
                                                  uint8_t* __restrict__ chw_nar,
                                                  uint8_t* __restrict__ chan_nar, uint8_t* __restrict__ any,
                                                  bool ring = true, uint8_t* __restrict__ wide = nullptr,
                                                  int wide_planes = 0, int store_planes = D) {
    const int Hp = H + 2 * pad, Wp = W + 2 * pad;
    const int CS = Cp / 16;
    const int c0 = cc * 32;
    uint32_t words[D][8];
    uint32_t nm = 0;
    if (lut != nullptr) {  // (branch hoisted out of the per-code loop)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t c4[4] = {code[4 * q], code[4 * q + 1], code[4 * q + 2], code[4 * q + 3]};
            nm |= digits4_words<D, kSmemLut>(c4, f, nar_code, lut, words, q) << (4 * q);
        }
    } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t c4[4] = {code[4 * q], code[4 * q + 1], code[4 * q + 2], code[4 * q + 3]};
            nm |= digits4_words<D>(c4, f, nar_code, nullptr, words, q) << (4 * q);
        }
    }
    if (wide != nullptr) {  // digit planes >= wide_planes in use (reduced-digit variants)
        uint32_t o = 0;
#pragma unroll
        for (int p = 0; p < D; ++p)
#pragma unroll
            for (int q = 0; q < 8; ++q) o |= p >= wide_planes ? words[p][q] : 0u;
        if (o && *reinterpret_cast<volatile uint8_t*>(wide) == 0) *wide = 1;  // read first: no same-address store storm
    }
    // this chunk = slices 2cc, 2cc + 1 of pixel (h + pad, w + pad)
    auto cell = [&](int hh, int ww) {
        return dig + (((int64_t(n) * Hp + hh) * CS + 2 * cc) * Wp + ww) * 16;
    };
    int8_t* dst = cell(int(h) + pad, int(w) + pad);
#pragma unroll
    for (int p = 0; p < D; ++p) {
        if (p >= store_planes) break;  // high planes: written by the completion pass if used
        *reinterpret_cast<uint4*>(dst + p * plane) =
            make_uint4(words[p][0], words[p][1], words[p][2], words[p][3]);
        *reinterpret_cast<uint4*>(dst + p * plane + int64_t(Wp) * 16) =
            make_uint4(words[p][4], words[p][5], words[p][6], words[p][7]);
    }
    if (ring && pad > 0 && (h == 0 || w == 0 || int(h) == H - 1 || int(w) == W - 1)) {
        // border pixel: zero the ring cells of its row / column (corners by
        // the corner pixels)
        const int ylo = h == 0 ? 0 : int(h) + pad, yhi = int(h) == H - 1 ? Hp - 1 : int(h) + pad;
        const int xlo = w == 0 ? 0 : int(w) + pad, xhi = int(w) == W - 1 ? Wp - 1 : int(w) + pad;
        for (int hh = ylo; hh <= yhi; ++hh)
            for (int ww = xlo; ww <= xhi; ++ww) {
                if (hh == int(h) + pad && ww == int(w) + pad) continue;
                int8_t* z = cell(hh, ww);
                for (int p = 0; p < store_planes; ++p) {
                    *reinterpret_cast<uint4*>(z + p * plane) = make_uint4(0, 0, 0, 0);
                    *reinterpret_cast<uint4*>(z + p * plane + int64_t(Wp) * 16) = make_uint4(0, 0, 0, 0);
                }
            }
    }
    if (nm) {
        for (int j = 0; j < 32; ++j)
            if (((nm >> j) & 1) && c0 + j < C) {
                if (pos_nar) pos_nar[r] = 1;
                if (chw_nar) chw_nar[int64_t(c0 + j) * HW + pix] = 1;
                if (chan_nar) chan_nar[c0 + j] = 1;
                *any = 1;
            }
    }
}

// codes [N][C][H][W] -> dig[D][N][Hp][Cp/16][Wp][16] (slice layout, balanced
// int8 digits; channels >= C are zero; Hp = H + 2 pad, Wp = W + 2 pad with the
// pad ring written as zeros by the border pixels' threads), plus NaR summaries
// written only where a NaR is found: pos_nar[n][h][w] (any channel),
// chw_nar[c][h][w] (any image), chan_nar[c], *any.  A thread owns one pixel x
// one 32-channel chunk: its 32 loads are coalesced across the warp
// (consecutive pixels of one channel plane), and it writes 32 contiguous digit
// bytes per plane (two 16-byte stores), so the warp's stores are 1 KB
// contiguous per plane.  lut: digit words per SOURCE code (digit_lut_kernel:
// the digits of convert(code, fs -> f), formats up to 12 bits) or null
// (in-register decode; then fs == f).  fs: the codes' format (NaR pattern).
// Grid: (pixel blocks, 32-channel chunks); 32-bit indices (pixels < 2^31,
// checked by the launcher) with launch-constant divisions by multiplication.
template <int D, typename CodeT>
__global__ void __launch_bounds__(256) act_digits_kernel(
    const CodeT* __restrict__ x, int N, int C, int H, int W, int Cp, int pad, FastDiv fd_hw,
    FastDiv fd_w, PositFmt f, PositFmt fs, const uint32_t* __restrict__ lut,
    int8_t* __restrict__ dig, uint8_t* __restrict__ pos_nar, uint8_t* __restrict__ chw_nar,
    uint8_t* __restrict__ chan_nar, uint8_t* __restrict__ any, DigitGate gt = DigitGate{},
    uint8_t* __restrict__ wide = nullptr, int wide_planes = 0, int store_planes = D,
    const uint8_t* __restrict__ only_if = nullptr, const uint8_t* __restrict__ only_if2 = nullptr) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    // completion pass: runs iff a consumer reads the high planes
    if (only_if != nullptr && *only_if == 0 && (only_if2 == nullptr || *only_if2 == 0)) return;
    const uint32_t HW = uint32_t(H) * uint32_t(W);
    const uint32_t pixels = uint32_t(N) * HW;
    const int64_t plane = int64_t(N) * (H + 2 * pad) * (W + 2 * pad) * Cp;
    const int cc = blockIdx.y;
    const uint32_t nar_code = 1u << (fs.nbits - 1);
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < pixels; r += gridDim.x * blockDim.x) {
        uint32_t n, pix;  // pixel raster index r = (n, h, w)
        fd_hw.divmod(r, n, pix);
        const int c0 = cc * 32;
        const int64_t base = (int64_t(n) * C + c0) * HW + pix;
        const CodeT* src = x + base;
        uint32_t code[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) code[j] = c0 + j < C ? uint32_t(src[j * HW]) : 0u;
        if (gt.gate != nullptr) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (c0 + j < C && !gt.open(base + int64_t(j) * HW)) code[j] = 0u;
        }
        uint32_t h, w;
        fd_w.divmod(pix, h, w);
        emit_pixel_digits<D>(code, r, n, pix, h, w, cc, C, H, W, Cp, pad, plane, HW, f, nar_code, lut,
                             dig, pos_nar, chw_nar, chan_nar, any, true, wide, wide_planes, store_planes);
    }
}

// As act_digits_kernel for images of HW % 256 == 0 pixels (16-byte aligned
// channel planes): a block digitises tiles of 256 pixels x 32 channels; the
// tile's codes arrive by 16-byte loads of whole channel rows into shared
// memory (the per-thread strided loads of the generic kernel move 32 or 64
// bytes per warp instruction), then each thread reads its pixel's 32 codes
// across the rows.
template <int D, typename CodeT, int GB = 0>
__global__ void __launch_bounds__(256) act_digits_tiled_kernel(
    const CodeT* __restrict__ x, int N, int C, int H, int W, int Cp, int pad, FastDiv fd_hw,
    FastDiv fd_w, PositFmt f, PositFmt fs, const uint32_t* __restrict__ lut,
    int8_t* __restrict__ dig, uint8_t* __restrict__ pos_nar, uint8_t* __restrict__ chw_nar,
    uint8_t* __restrict__ chan_nar, uint8_t* __restrict__ any, DigitGate gt = DigitGate{},
    uint8_t* __restrict__ wide = nullptr, int wide_planes = 0, int store_planes = D,
    const uint8_t* __restrict__ only_if = nullptr, const uint8_t* __restrict__ only_if2 = nullptr) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    // completion pass: runs iff a consumer reads the high planes
    if (only_if != nullptr && *only_if == 0 && (only_if2 == nullptr || *only_if2 == 0)) return;
    constexpr int TP = 256;                                   // pixels per tile
    constexpr int VPR = TP * int(sizeof(CodeT)) / 16;         // 16-byte vectors per channel row
    // ungated: two tile buffers, the next tile's rows in flight (cp.async)
    // while this tile is digitised
    constexpr int NB = GB == 0 ? 2 : 1;
    __shared__ uint4 s_tile[NB][32 * VPR];
    __shared__ uint4 s_gate[GB > 0 ? 32 * TP * GB / 16 : 1];  // gate codes (GB bytes each)
    const uint32_t HW = uint32_t(H) * uint32_t(W);
    const uint32_t tiles = uint32_t(N) * (HW / TP);
    const int64_t plane = int64_t(N) * (H + 2 * pad) * (W + 2 * pad) * Cp;
    const int cc = blockIdx.y, c0 = cc * 32;
    const uint32_t nar_code = 1u << (fs.nbits - 1);
    // 8-bit source codes: the digit table (<= 256 x 8 bytes) in shared memory
    constexpr bool kSL = sizeof(CodeT) == 1;
    __shared__ uint2 s_dlut[kSL ? 256 : 1];
    if constexpr (kSL)
        if (lut != nullptr)
            for (int i = threadIdx.x; i < (1 << fs.nbits); i += blockDim.x)
                s_dlut[i] = __ldg(reinterpret_cast<const uint2*>(lut) + i);
    const uint32_t* lut_use = kSL && lut != nullptr ? reinterpret_cast<const uint32_t*>(s_dlut) : lut;
    auto load_async = [&](uint32_t t, int b) {
        uint32_t n, pix0;
        fd_hw.divmod(t * TP, n, pix0);
        for (int i = threadIdx.x; i < 32 * VPR; i += blockDim.x) {
            const int c = i / VPR, v = i - c * VPR;
            if (c0 + c < C)
                ptx::cp_async16(&s_tile[b][i],
                                reinterpret_cast<const uint4*>(x + (int64_t(n) * C + c0 + c) * HW + pix0) + v);
            else
                s_tile[b][i] = make_uint4(0, 0, 0, 0);
        }
        ptx::cp_async_commit();
    };
    if constexpr (GB == 0)
        if (blockIdx.x < tiles) load_async(blockIdx.x, 0);
    int buf = 0;
    for (uint32_t t = blockIdx.x; t < tiles; t += gridDim.x, buf ^= NB - 1) {
        const uint32_t r0 = t * TP;
        uint32_t n, pix0;
        fd_hw.divmod(r0, n, pix0);
        __syncthreads();  // previous tile's readers are done
        if constexpr (GB == 0) {
            if (t + gridDim.x < tiles) {
                load_async(t + gridDim.x, buf ^ 1);
                ptx::cp_async_wait<1>();  // this tile's group has landed
            } else {
                ptx::cp_async_wait<0>();
            }
            __syncthreads();
        } else {
            for (int i = threadIdx.x; i < 32 * VPR; i += blockDim.x) {
                const int c = i / VPR, v = i - c * VPR;
                s_tile[0][i] = c0 + c < C ? __ldg(reinterpret_cast<const uint4*>(
                                                x + (int64_t(n) * C + c0 + c) * HW + pix0) + v)
                                          : make_uint4(0, 0, 0, 0);
            }
        }
        if constexpr (GB > 0) {
            constexpr int GVPR = TP * GB / 16;
            for (int i = threadIdx.x; i < 32 * GVPR; i += blockDim.x) {
                const int c = i / GVPR, v = i - c * GVPR;
                s_gate[i] = c0 + c < C
                                ? __ldg(reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(gt.gate) +
                                                                       ((int64_t(n) * C + c0 + c) * HW + pix0) *
                                                                           GB) + v)
                                : make_uint4(0, 0, 0, 0);
            }
        }
        if constexpr (GB > 0) __syncthreads();
        const CodeT* st = reinterpret_cast<const CodeT*>(s_tile[buf]);
        uint32_t code[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) code[j] = uint32_t(st[j * TP + threadIdx.x]);
        if constexpr (GB > 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int k = j * TP + threadIdx.x;
                const uint32_t g = GB == 1 ? uint32_t(reinterpret_cast<const uint8_t*>(s_gate)[k])
                                           : uint32_t(reinterpret_cast<const uint16_t*>(s_gate)[k]);
                if (!(g != 0 && ((g >> (gt.gnbits - 1)) & 1u) == 0)) code[j] = 0u;
            }
        }
        const uint32_t pix = pix0 + threadIdx.x;
        uint32_t h, w;
        fd_w.divmod(pix, h, w);
        // pixel cells only (pad 0 below); the zero ring of this tile's rows is
        // written cooperatively afterwards (per-thread ring loops diverge in
        // every warp: each image row has a first and a last pixel)
        emit_pixel_digits<D, kSL>(code, r0 + threadIdx.x, n, pix, h, w, cc, C, H, W, Cp, pad, plane, HW, f,
                                  nar_code, lut_use, dig, pos_nar, chw_nar, chan_nar, any, /*ring=*/false, wide,
                             wide_planes, store_planes);
        if (pad > 0) {
            const int Hp = H + 2 * pad, Wp = W + 2 * pad, CS = Cp / 16;
            uint32_t hh0, ww0;
            fd_w.divmod(pix0, hh0, ww0);  // a tile = whole rows (W | 256) or part of one row (256 | W)
            const int rows = TP / W > 0 ? TP / W : 1;  // (part-row tiles rewrite both side cells: zeros)
            const int y0 = int(hh0), y1 = y0 + rows - 1;
            // ring cells: left/right pad cells of rows y0..y1, plus the top pad rows
            // (tile holds row 0) and the bottom pad rows (tile holds row H-1)
            const int side = rows * 2 * pad;
            const int top = y0 == 0 ? pad * Wp : 0, bot = y1 == H - 1 ? pad * Wp : 0;
            const int cells = side + top + bot;
            const int SP = store_planes;
            for (int i = threadIdx.x; i < cells * SP * 2; i += blockDim.x) {
                const int cell = i / (SP * 2), rest = i - cell * (SP * 2), p = rest >> 1, sl = rest & 1;
                int hh, ww;
                if (cell < side) {
                    const int r = cell / (2 * pad), k = cell - r * (2 * pad);
                    hh = y0 + r + pad;
                    ww = k < pad ? k : W + k;
                } else if (cell < side + top) {
                    hh = (cell - side) / Wp;
                    ww = (cell - side) % Wp;
                } else {
                    hh = H + pad + (cell - side - top) / Wp;
                    ww = (cell - side - top) % Wp;
                }
                int8_t* z = dig + p * plane + (((int64_t(n) * Hp + hh) * CS + 2 * cc + sl) * Wp + ww) * 16;
                *reinterpret_cast<uint4*>(z) = make_uint4(0, 0, 0, 0);
            }
        }
    }
}

// First-layer tap folding (C*KH*KW <= 32, stride 1): the receptive field of
// each output pixel becomes the 32 "channels" of a virtual 1x1 convolution,
// dig[D][N][OH][OW][32] with channel k = (c, ky, kx) (zero past C*KH*KW and
// outside the image).  A thread per output pixel: its gathers are coalesced
// across the warp (consecutive pixels), its 32 digit bytes per plane go out as
// two 16-byte stores.  NaR summaries in the virtual geometry: pos_nar[n][oy][ox]
// (forward rows) and chw_nar[k][oy][ox] (weight-grad rows).
template <int D, typename CodeT>
__global__ void __launch_bounds__(256) im2col_digits_kernel(
    const CodeT* __restrict__ x, int N, int C, int H, int W, int KH, int KW, int pad, int OH,
    int OW, FastDiv fd_p, FastDiv fd_ow, PositFmt f, PositFmt fs, const uint32_t* __restrict__ lut,
    int8_t* __restrict__ dig, uint8_t* __restrict__ pos_nar, uint8_t* __restrict__ chw_nar,
    uint8_t* __restrict__ any, uint8_t* __restrict__ wide = nullptr, int wide_planes = 0,
    int store_planes = D, const uint8_t* __restrict__ only_if = nullptr) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    // completion pass: runs iff a consumer reads the high planes
    if (only_if != nullptr && *only_if == 0) return;
    // 8-bit source codes: the digit table in shared memory
    constexpr bool kSL = sizeof(CodeT) == 1;
    __shared__ uint2 s_dlut[kSL ? 256 : 1];
    if constexpr (kSL)
        if (lut != nullptr)
            for (int i = threadIdx.x; i < (1 << fs.nbits); i += blockDim.x)
                s_dlut[i] = __ldg(reinterpret_cast<const uint2*>(lut) + i);
    const uint32_t* lut_use = kSL && lut != nullptr ? reinterpret_cast<const uint32_t*>(s_dlut) : lut;
    const int ckk = C * KH * KW, khw = KH * KW;
    const uint32_t nar_code = 1u << (fs.nbits - 1);  // fs: the codes' format (lut converts)
    const uint32_t P = uint32_t(OH) * uint32_t(OW);
    const int64_t plane = int64_t(N) * P * 32;
    // receptive-field table: K index k -> (offset of (c, ky - pad, kx - pad) in
    // the image, ky - pad, kx - pad); k >= ckk never loads
    __shared__ int s_off[32];
    __shared__ int16_t s_dy[32], s_dx[32];
    if (threadIdx.x < 32) {
        const int k = threadIdx.x;
        const int c = k / khw, t = k - c * khw, ky = t / KW, kx = t - ky * KW;
        s_off[k] = (c * H + ky - pad) * W + kx - pad;
        s_dy[k] = int16_t(k < ckk ? ky - pad : -32768);  // padding K: never in range
        s_dx[k] = int16_t(kx - pad);
    }
    __syncthreads();
    const uint32_t NP = uint32_t(N) * P;
    for (uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x; pos < NP; pos += gridDim.x * blockDim.x) {
        uint32_t n, pix, oy, ox;
        fd_p.divmod(pos, n, pix);
        fd_ow.divmod(pix, oy, ox);
        const CodeT* xn = x + int64_t(n) * C * H * W + int(oy) * W + int(ox);
        uint32_t words[D][8];
        uint32_t nm = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            uint32_t c4[4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int k = 4 * q + jj;
                const int iy = int(oy) + s_dy[k], ix = int(ox) + s_dx[k];
                c4[jj] = (unsigned(iy) < unsigned(H) && unsigned(ix) < unsigned(W))
                             ? uint32_t(xn[s_off[k]])
                             : 0u;
            }
            nm |= lut_use != nullptr ? digits4_words<D, kSL>(c4, f, nar_code, lut_use, words, q) << (4 * q)
                                     : digits4_words<D>(c4, f, nar_code, nullptr, words, q) << (4 * q);
        }
        if (wide != nullptr && only_if == nullptr) {  // digit planes >= wide_planes in use
            uint32_t o = 0;
#pragma unroll
            for (int p = 0; p < D; ++p)
#pragma unroll
                for (int q = 0; q < 8; ++q) o |= p >= wide_planes ? words[p][q] : 0u;
            if (o && *reinterpret_cast<volatile uint8_t*>(wide) == 0) *wide = 1;  // read first: no same-address store storm
        }
        // slice layout of the virtual [N][OH][2 slices][OW][16] image
        const int64_t row = int64_t(n) * OH + oy;
        int8_t* dst = dig + ((row * 2) * OW + ox) * 16;
#pragma unroll
        for (int p = 0; p < D; ++p) {
            if (p >= store_planes) break;  // high planes: written by the completion pass if used
            *reinterpret_cast<uint4*>(dst + p * plane) =
                make_uint4(words[p][0], words[p][1], words[p][2], words[p][3]);
            *reinterpret_cast<uint4*>(dst + p * plane + int64_t(OW) * 16) =
                make_uint4(words[p][4], words[p][5], words[p][6], words[p][7]);
        }
        if (nm)
            for (int k = 0; k < ckk; ++k)
                if ((nm >> k) & 1) {
                    if (pos_nar) pos_nar[pos] = 1;
                    if (chw_nar) chw_nar[int64_t(k) * P + pix] = 1;
                    *any = 1;
                }
    }
}

// w [F][C][KH][KW] -> K-major weight digits in the slice layout
// dig[D][taps*Kp/16][rows][16] (16 K bytes of one row contiguous):
//   transpose = 0 (forward):    rows = F, element (f, tap, c) = w[f][c][tap]
//   transpose = 1 (input grad): rows = C, element (c, tap, f) = w[f][c][tap]
// Forward: col_add[f] = X(bias[f]), col_nar[f] = NaR in weight row f or bias f.
template <int D, typename CodeT>
__global__ void weight_digits_kernel(const CodeT* __restrict__ w, const CodeT* __restrict__ bias,
                                     int F, int C, int taps, int Kp, int transpose, PositFmt f,
                                     int8_t* __restrict__ dig, int64_t* __restrict__ col_add,
                                     uint8_t* __restrict__ col_nar, uint8_t* __restrict__ any,
                                     uint8_t* __restrict__ wide = nullptr, int wide_planes = 0) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    const int rows = transpose ? C : F;
    const int inner = transpose ? F : C;
    const int64_t total = int64_t(rows) * taps * Kp;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int k = int(i % Kp);
        const int tap = int((i / Kp) % taps);
        const int r = int(i / (int64_t(Kp) * taps));
        const int64_t kg = int64_t(tap) * Kp + k;  // K index; slice layout [D][K/16][rows][16]
        uint32_t code = 0;
        if (k < inner) {
            const int fo = transpose ? k : r, ci = transpose ? r : k;
            code = uint32_t(w[(int64_t(fo) * C + ci) * taps + tap]);
        }
        uint32_t lo, hi;
        bool nar;
        digit_words<D>(code, f, lo, hi, nar);
        if (nar) {
            if (col_nar && !transpose) col_nar[r] = 1;
            *any = 1;
        }
        if (wide != nullptr) {  // a digit plane >= wide_planes in use
            const uint64_t y = (uint64_t(hi) << 32) | lo;
            if ((y >> (8 * wide_planes)) && *reinterpret_cast<volatile uint8_t*>(wide) == 0) *wide = 1;
        }
#pragma unroll
        for (int p = 0; p < D; ++p)
            dig[int64_t(p) * total + ((kg >> 4) * rows + r) * 16 + (kg & 15)] =
                int8_t(((p < 4 ? lo : hi) >> (8 * (p & 3))) & 0xFFu);
    }
    if (!transpose && col_add != nullptr) {
        for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < F;
             r += int64_t(gridDim.x) * blockDim.x) {
            int64_t X = 0;
            const bool nar = bias != nullptr && decode_x(uint32_t(bias[r]), f, X);
            col_add[r] = X;
            if (nar) col_nar[r] = 1;
        }
    }
}

// ------------------------------------------------------------- NaR fix-ups

// Weight-side NaR of the input gradient, exact per output over its valid taps.
// Runs only when the pack pass saw a NaR weight (flag set on device).
template <typename CodeT>
__global__ void dgrad_weight_nar_kernel(CodeT* __restrict__ dx, const CodeT* __restrict__ w,
                                        ConvGeom g, const uint8_t* __restrict__ any_nar_w,
                                        uint32_t nar) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    if (*any_nar_w == 0) return;
    const int64_t total = g.N * g.C * g.H * g.W;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t ix = i % g.W, iy = (i / g.W) % g.H, c = (i / (g.W * g.H)) % g.C;
        bool hit = false;
        for (int64_t f = 0; f < g.F && !hit; ++f)
            for (int64_t ky = 0; ky < g.KH && !hit; ++ky) {
                const int64_t ty = iy + g.pad - ky;
                if (ty < 0 || ty % g.stride || ty / g.stride >= g.OH) continue;
                for (int64_t kx = 0; kx < g.KW; ++kx) {
                    const int64_t tx = ix + g.pad - kx;
                    if (tx < 0 || tx % g.stride || tx / g.stride >= g.OW) continue;
                    if (uint32_t(w[((f * g.C + c) * g.KH + ky) * g.KW + kx]) == nar) {
                        hit = true;
                        break;
                    }
                }
            }
        if (hit) dx[i] = CodeT(nar);
    }
}

// Row NaR of the implicit passes (an output is NaR iff one of its terms has a
// NaR operand, quire.hpp:55); launched always, exit at once unless the
// digitiser saw a NaR.

// forward: y[n][:][oy][ox] = NaR if a tap in range reads a NaR pixel
template <typename CodeT>
__global__ void fwd_nar_fixup_kernel(CodeT* __restrict__ y, const uint8_t* __restrict__ pos_nar,
                                     const uint8_t* __restrict__ any, int64_t N, int F, int H,
                                     int W, int OH, int OW, int KH, int KW, int pad, uint32_t nar,
                                     int relu = 0, CodeT* __restrict__ pre = nullptr) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    if (*any == 0) return;
    const int64_t total = N * OH * OW;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int ox = int(i % OW), oy = int((i / OW) % OH);
        const int64_t n = i / (int64_t(OH) * OW);
        bool hit = false;
        for (int ky = 0; ky < KH && !hit; ++ky)
            for (int kx = 0; kx < KW && !hit; ++kx) {
                const int iy = oy + ky - pad, ix = ox + kx - pad;
                if (unsigned(iy) < unsigned(H) && unsigned(ix) < unsigned(W))
                    hit = pos_nar[(n * H + iy) * W + ix] != 0;
            }
        if (hit)
            for (int fo = 0; fo < F; ++fo) {
                const int64_t o = ((n * F + fo) * OH + oy) * OW + ox;
                y[o] = CodeT(relu ? 0u : nar);  // relu(NaR) = 0
                if (pre) pre[o] = CodeT(nar);
            }
    }
}

// relu in place (+ copy of the pre-activation): the split-K forward path of a
// fused Conv2d + ReLU, after quire_finalize_kernel
template <typename CodeT>
__global__ void relu_codes_kernel(CodeT* __restrict__ y, CodeT* __restrict__ pre, int64_t n, int nbits) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = uint32_t(y[i]);
        if (pre) pre[i] = CodeT(c);
        y[i] = CodeT((c != 0 && ((c >> (nbits - 1)) & 1u) == 0) ? c : 0u);
    }
}

// input grad: dx[n][:][iy][ix] = NaR if a valid tap reads a NaR output gradient
template <typename CodeT>
__global__ void dgrad_nar_fixup_kernel(CodeT* __restrict__ dx, const uint8_t* __restrict__ pos_nar,
                                       const uint8_t* __restrict__ any, int64_t N, int C, int H,
                                       int W, int OH, int OW, int KH, int KW, int pad, uint32_t nar) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    if (*any == 0) return;
    const int64_t total = N * H * W;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int ix = int(i % W), iy = int((i / W) % H);
        const int64_t n = i / (int64_t(H) * W);
        bool hit = false;
        for (int ky = 0; ky < KH && !hit; ++ky)
            for (int kx = 0; kx < KW && !hit; ++kx) {
                const int oy = iy + pad - ky, ox = ix + pad - kx;
                if (unsigned(oy) < unsigned(OH) && unsigned(ox) < unsigned(OW))
                    hit = pos_nar[(n * OH + oy) * OW + ox] != 0;
            }
        if (hit)
            for (int c = 0; c < C; ++c) dx[((n * C + c) * H + iy) * W + ix] = CodeT(nar);
    }
}

// weight grad: dw[:][c][tap] = NaR if the tap's window over channel c holds a NaR
template <typename CodeT>
__global__ void wgrad_nar_fixup_kernel(CodeT* __restrict__ dw, uint8_t* __restrict__ raw_nar,
                                       const uint8_t* __restrict__ chw_nar,
                                       const uint8_t* __restrict__ any, int F, int C, int H, int W,
                                       int OH, int OW, int KH, int KW, int pad, uint32_t nar) {
    pdl_trigger();
    pdl_wait();  // PDL: nothing above touches global memory (pdl.cuh)
    if (*any == 0) return;
    const int taps = KH * KW;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < C * taps; i += gridDim.x * blockDim.x) {
        const int c = i / taps, tap = i % taps, ky = tap / KW, kx = tap % KW;
        bool hit = false;
        for (int oy = 0; oy < OH && !hit; ++oy) {
            const int iy = oy + ky - pad;
            if (unsigned(iy) >= unsigned(H)) continue;
            for (int ox = 0; ox < OW; ++ox) {
                const int ix = ox + kx - pad;
                if (unsigned(ix) < unsigned(W) && chw_nar[(int64_t(c) * H + iy) * W + ix]) {
                    hit = true;
                    break;
                }
            }
        }
        if (hit)
            for (int fo = 0; fo < F; ++fo) {
                const int64_t o = (int64_t(fo) * C + c) * taps + tap;
                if (dw) dw[o] = CodeT(nar);
                if (raw_nar) raw_nar[o] = 1;
            }
    }
}

}  // namespace pnn_b200
