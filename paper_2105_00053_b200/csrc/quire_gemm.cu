// Exact posit-quire GEMM on the 5th-gen tensor cores (tcgen05 kind::i8).
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
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "posit_device.cuh"
#include "quire_gemm.h"
#include "sm100_ptx.cuh"

namespace pnn_b200 {

template <int D>
struct TileCfg;
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

template <int D>
struct Geometry {
    static constexpr int NT = TileCfg<D>::NT;
    static constexpr int KB = TileCfg<D>::KB;
    static constexpr int STAGES = TileCfg<D>::STAGES;
    static constexpr int G = 2 * D - 1;
    static constexpr int NMMA = D * NT;
    static constexpr int A_BYTES = D * kBM * KB;
    static constexpr int B_BYTES = D * NT * KB;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int SMEM = STAGES * STAGE_BYTES + kZeroBytes + 256;
    static_assert((NT / 2) % 8 == 0, "epilogue column split");
    static constexpr uint32_t TMEM_COLS = 512;
    static_assert(G * NT <= 512, "TMEM overflow");
    static_assert(NMMA % 16 == 0 && NMMA <= 256, "bad UMMA N");
    static_assert(KB % 32 == 0, "KB must hold whole i8 MMA k-steps");
};

// ---------------------------------------------------------------- packing

template <typename CodeT>
__device__ __forceinline__ uint32_t load_code(const CodeT* p) {
    return uint32_t(*p);
}

// A[M][K] row-major codes -> A_img[mt][kb][D][16 rowgroups][KB/16][8][16].
template <int D, typename CodeT>
__global__ void __launch_bounds__(256) pack_a_kernel(const CodeT* __restrict__ A, int64_t M,
                                                     int64_t K, int64_t lda, PositFmt f,
                                                     int8_t* __restrict__ img,
                                                     uint8_t* __restrict__ row_nar, int64_t kbt) {
    constexpr int KB = Geometry<D>::KB;
    constexpr int KC = KB / 16;
    const int64_t mtiles = (M + kBM - 1) / kBM;
    const int64_t total = mtiles * kbt * kBM * KC;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int r8 = int(idx & 7);
        int64_t t = idx >> 3;
        const int kc = int(t % KC);
        t /= KC;
        const int rg = int(t % 16);
        t /= 16;
        const int64_t kb = t % kbt;
        const int64_t mt = t / kbt;
        const int64_t row = mt * kBM + rg * 8 + r8;
        const int64_t k0 = kb * KB + kc * 16;
        alignas(16) int8_t dig[D][16];
        bool any_nar = false;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            uint32_t code = 0;
            if (row < M && k0 + j < K) code = load_code(A + row * lda + k0 + j);
            int64_t X;
            any_nar |= decode_x(code, f, X);
            int8_t d8[D];
            balanced_digits<D>(X, d8);
#pragma unroll
            for (int p = 0; p < D; ++p) dig[p][j] = d8[p];
        }
        if (any_nar) row_nar[row] = 1;
        int8_t* chunk = img + (mt * kbt + kb) * int64_t(D * kBM * KB);
#pragma unroll
        for (int p = 0; p < D; ++p) {
            int8_t* dst = chunk + p * (kBM * KB) + rg * (8 * KB) + kc * 128 + r8 * 16;
            *reinterpret_cast<int4*>(dst) = *reinterpret_cast<const int4*>(dig[p]);
        }
    }
}

// B[K][N] row-major codes -> B_img[nt][kb][D][NT/8][KB/16][8][16] (K-major rows
// of the concatenated N dimension: plane p occupies rows [p*NT, (p+1)*NT)).
template <int D, typename CodeT>
__global__ void __launch_bounds__(256) pack_b_kernel(const CodeT* __restrict__ B, int64_t K,
                                                     int64_t N, int64_t ldb, PositFmt f,
                                                     int8_t* __restrict__ img,
                                                     uint8_t* __restrict__ col_nar, int64_t kbt) {
    constexpr int NT = Geometry<D>::NT;
    constexpr int KB = Geometry<D>::KB;
    constexpr int KC = KB / 16;
    const int64_t ntiles = (N + NT - 1) / NT;
    const int64_t total = ntiles * kbt * NT * KC;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int nl = int(idx % NT);
        int64_t t = idx / NT;
        const int kc = int(t % KC);
        t /= KC;
        const int64_t kb = t % kbt;
        const int64_t nt = t / kbt;
        const int64_t n = nt * NT + nl;
        const int64_t k0 = kb * KB + kc * 16;
        alignas(16) int8_t dig[D][16];
        bool any_nar = false;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            uint32_t code = 0;
            if (n < N && k0 + j < K) code = load_code(B + (k0 + j) * ldb + n);
            int64_t X;
            any_nar |= decode_x(code, f, X);
            int8_t d8[D];
            balanced_digits<D>(X, d8);
#pragma unroll
            for (int p = 0; p < D; ++p) dig[p][j] = d8[p];
        }
        if (any_nar) col_nar[n] = 1;
        int8_t* chunk = img + (nt * kbt + kb) * int64_t(D * NT * KB);
#pragma unroll
        for (int p = 0; p < D; ++p) {
            int8_t* dst = chunk + p * (NT * KB) + (nl / 8) * (8 * KB) + kc * 128 + (nl % 8) * 16;
            *reinterpret_cast<int4*>(dst) = *reinterpret_cast<const int4*>(dig[p]);
        }
    }
}

// ------------------------------------------------------------- main kernel

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
        for (int j = 0; j < valid; ++j) dst[j] = CodeT(c[j]);
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

// Raster: tiles grouped by kGroupM m-tiles so the ~148 tiles in flight share
// A and B digit planes in L2.
constexpr int kGroupM = 8;

__device__ __forceinline__ void tile_coords(int64_t t, int64_t mtiles, int64_t ntiles,
                                            int64_t& split, int64_t& mt, int64_t& nt) {
    const int64_t per_split = mtiles * ntiles;
    split = t / per_split;
    const int64_t r = t - split * per_split;
    const int64_t group = r / (kGroupM * ntiles);
    const int64_t within = r - group * (kGroupM * ntiles);
    const int64_t gm = min(int64_t(kGroupM), mtiles - group * kGroupM);
    mt = group * kGroupM + within % gm;
    nt = within / gm;
}

// Persistent, warp-specialized: warp 0 = bulk-copy producer, warp 1 = MMA
// issuer, warps 2..9 = epilogue (2 warps per TMEM lane quarter, each owning
// half of the tile's columns).  The epilogue drains TMEM into registers,
// releases it (tmem_empty), and rounds/stores while the next tile's MMAs run.
template <int D, int QW, typename CodeT>
__global__ void __launch_bounds__(kThreads, 1)
    quire_gemm_tc_kernel(const int8_t* __restrict__ a_img, const int8_t* __restrict__ b_img,
                         int64_t kbt, int64_t kb_per_split, const uint8_t* __restrict__ row_nar,
                         const uint8_t* __restrict__ col_nar, CodeT* __restrict__ C, int64_t M,
                         int64_t N, int64_t ldc, PositFmt f,
                         unsigned __int128* __restrict__ partial, int64_t mtiles, int64_t ntiles,
                         int64_t splits) {
    using Geo = Geometry<D>;
    using QT = typename QuireWord<QW>::T;
    constexpr int NT = Geo::NT, KB = Geo::KB, STAGES = Geo::STAGES, G = Geo::G;
    constexpr int COLS = NT / 2;                 // columns per epilogue thread
    constexpr int GB = G < 8 ? G : 8;            // TMEM loads batched per wait
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* zero_tile = smem + STAGES * Geo::STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(zero_tile + kZeroBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t tiles = mtiles * ntiles * splits;

    for (int i = threadIdx.x; i < kZeroBytes / 16; i += kThreads)
        reinterpret_cast<int4*>(zero_tile)[i] = make_int4(0, 0, 0, 0);
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(tmem_full, 1);
        ptx::mbar_init(tmem_empty, kEpiWarps);
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<Geo::TMEM_COLS>(tmem_slot);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ===== producer: one bulk copy per operand per stage =====
            uint32_t it = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                int64_t split, mt, nt;
                tile_coords(t, mtiles, ntiles, split, mt, nt);
                const int64_t kb0 = split * kb_per_split;
                const int nkb = int(min(kbt, kb0 + kb_per_split) - kb0);
                const int8_t* a_src = a_img + (mt * kbt + kb0) * int64_t(Geo::A_BYTES);
                const int8_t* b_src = b_img + (nt * kbt + kb0) * int64_t(Geo::B_BYTES);
                for (int i = 0; i < nkb; ++i, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    ptx::mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* sa = smem + s * Geo::STAGE_BYTES;
                    ptx::mbar_arrive_expect_tx(&full[s], Geo::STAGE_BYTES);
                    ptx::bulk_g2s(sa, a_src + int64_t(i) * Geo::A_BYTES, Geo::A_BYTES, &full[s]);
                    ptx::bulk_g2s(sa + Geo::A_BYTES, b_src + int64_t(i) * Geo::B_BYTES,
                                  Geo::B_BYTES, &full[s]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ===== MMA issuer =====
            constexpr uint32_t idesc = ptx::idesc_i8(kBM, Geo::NMMA);
            constexpr uint32_t SBO = 8 * KB, LBO = 128;
            const uint64_t zdesc = ptx::smem_desc_kmajor(ptx::smem_u32(zero_tile), LBO, 8 * 32);
            uint32_t it = 0, j = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
                int64_t split, mt, nt;
                tile_coords(t, mtiles, ntiles, split, mt, nt);
                const int64_t kb0 = split * kb_per_split;
                const int nkb = int(min(kbt, kb0 + kb_per_split) - kb0);
                ptx::mbar_wait(tmem_empty, (j & 1) ^ 1);  // epilogue drained the previous tile
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
                        if (first)  // zero groups D-1 .. 2D-2 (plane 0 initialises 0 .. D-1)
                            ptx::mma_i8(tmem + (D - 1) * NT, zdesc, bdesc, idesc, 0);
#pragma unroll
                        for (int p = 0; p < D; ++p) {
                            const uint64_t adesc = ptx::smem_desc_kmajor(
                                a_base + p * (kBM * KB) + ks * 256, LBO, SBO);
                            ptx::mma_i8(tmem + p * NT, adesc, bdesc, idesc,
                                        (first && p == 0) ? 0u : 1u);
                        }
                    }
                    ptx::mma_commit(&empty[s]);
                }
                ptx::mma_commit(tmem_full);
            }
        }
    } else {
        // ===== epilogue: TMEM -> quire words (registers) -> posit codes =====
        const int quarter = warp & 3;
        const int half = (warp - 2) >> 2;
        const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16) + half * COLS;
        const bool vec_ok = (ldc % 8) == 0;
        uint32_t j = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
            int64_t split, mt, nt;
            tile_coords(t, mtiles, ntiles, split, mt, nt);
            ptx::mbar_wait(tmem_full, j & 1);
            ptx::tc_fence_after();
            QT q[COLS];
#pragma unroll
            for (int c = 0; c < COLS; ++c) q[c] = 0;
#pragma unroll
            for (int c0 = 0; c0 < COLS; c0 += 8) {
#pragma unroll
                for (int g0 = 0; g0 < G; g0 += GB) {
                    uint32_t r[GB][8];
#pragma unroll
                    for (int g = 0; g < GB; ++g)
                        if (g0 + g < G) ptx::tmem_ld8(trow + (g0 + g) * NT + c0, r[g]);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int g = 0; g < GB; ++g)
                        if (g0 + g < G)
#pragma unroll
                            for (int x = 0; x < 8; ++x) q[c0 + x] += group_term<QT>(r[g][x], 8 * (g0 + g));
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tmem_empty);

            const int64_t row = mt * kBM + quarter * 32 + lane;
            if (row >= M) continue;
            const bool rnar = row_nar[row] != 0;
            const int64_t colbase = nt * NT + half * COLS;
#pragma unroll
            for (int c0 = 0; c0 < COLS; c0 += 8) {
                const int64_t col0 = colbase + c0;
                if (col0 >= N) break;
                const int valid = int(N - col0 < 8 ? N - col0 : 8);
                if (partial != nullptr) {
                    unsigned __int128* dst = partial + (split * M + row) * N + col0;
#pragma unroll
                    for (int x = 0; x < 8; ++x)
                        if (x < valid) dst[x] = (unsigned __int128)q[c0 + x];
                    continue;
                }
                uint32_t codes[8];
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    const bool nar = rnar || (x < valid && col_nar[col0 + x]);
                    codes[x] = nar ? (1u << (f.nbits - 1)) : quire_word_to_posit(f, q[c0 + x]);
                }
                store_codes8(C + row * ldc + col0, codes, valid, vec_ok);
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

// Sum split-K quire partials (mod 2^W), apply NaR, round once.
template <typename CodeT>
__global__ void quire_finalize_kernel(const unsigned __int128* __restrict__ partial, int splits,
                                      const uint8_t* __restrict__ row_nar,
                                      const uint8_t* __restrict__ col_nar, CodeT* __restrict__ C,
                                      int64_t M, int64_t N, int64_t ldc, PositFmt f) {
    const int64_t total = M * N;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = idx / N, j = idx % N;
        uint32_t code;
        if (row_nar[i] || col_nar[j]) {
            code = 1u << (f.nbits - 1);
        } else {
            unsigned __int128 q = 0;
            for (int s = 0; s < splits; ++s) q += partial[s * total + idx];
            code = quire_word_to_posit(f, q);
        }
        C[i * ldc + j] = CodeT(code);
    }
}

// ------------------------------------------------------------------ host

static int digits_for(const PositFmt& f) {
    // smallest D with balanced capacity 127*(256^D-1)/255 >= 2^(2R)
    for (int D = 1; D <= 8; ++D) {
        const long double cap = 127.0L * (powl(256.0L, D) - 1.0L) / 255.0L;
        if (cap >= powl(2.0L, 2 * f.R)) return D < 2 ? 2 : D;
    }
    return -1;
}

template <int D>
static QuireGemmPlan plan_for(const PositFmt& f, int64_t M, int64_t N, int64_t K,
                              int64_t max_kb_per_split) {
    using Geo = Geometry<D>;
    QuireGemmPlan p{};
    p.D = D;
    p.NT = Geo::NT;
    p.KB = Geo::KB;
    p.mtiles = (M + kBM - 1) / kBM;
    p.ntiles = (N + Geo::NT - 1) / Geo::NT;
    p.kbt = (K + Geo::KB - 1) / Geo::KB;
    // int32 group sums stay exact for K <= 131071 / D (|digit| <= 128); the
    // (8,0)-style quire (W <= 32) is itself mod 2^32, so wrapping is exact.
    int64_t kmax_kb = f.W <= 32 ? p.kbt : (131071 / D) / Geo::KB;
    if (max_kb_per_split > 0 && max_kb_per_split < kmax_kb) kmax_kb = max_kb_per_split;
    if (kmax_kb < 1) kmax_kb = 1;
    p.kb_per_split = p.kbt < kmax_kb ? p.kbt : kmax_kb;
    p.splits = (p.kbt + p.kb_per_split - 1) / p.kb_per_split;
    p.a_img_bytes = size_t(p.mtiles) * p.kbt * Geo::A_BYTES;
    p.b_img_bytes = size_t(p.ntiles) * p.kbt * Geo::B_BYTES;
    p.row_nar_bytes = size_t(p.mtiles) * kBM;
    p.col_nar_bytes = size_t(p.ntiles) * Geo::NT;
    p.partial_bytes = p.splits > 1 ? size_t(p.splits) * M * N * 16 : 0;
    p.smem_bytes = Geo::SMEM;
    return p;
}

int quire_gemm_plan(int nbits, int es, int64_t M, int64_t N, int64_t K, int64_t max_kb_per_split,
                    QuireGemmPlan* plan) {
    const PositFmt f = make_fmt(nbits, es);
    if (nbits < 2 || nbits > 16 || es < 0 || 2 * f.R > 56) return 2;
    const int D = digits_for(f);
    switch (D) {
        case 2: *plan = plan_for<2>(f, M, N, K, max_kb_per_split); break;
        case 3: *plan = plan_for<3>(f, M, N, K, max_kb_per_split); break;
        case 4: *plan = plan_for<4>(f, M, N, K, max_kb_per_split); break;
        case 5: *plan = plan_for<5>(f, M, N, K, max_kb_per_split); break;
        case 6: *plan = plan_for<6>(f, M, N, K, max_kb_per_split); break;
        case 7: *plan = plan_for<7>(f, M, N, K, max_kb_per_split); break;
        case 8: *plan = plan_for<8>(f, M, N, K, max_kb_per_split); break;
        default: return 2;
    }
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    plan->off_a = take(plan->a_img_bytes);
    plan->off_b = take(plan->b_img_bytes);
    plan->off_row_nar = take(plan->row_nar_bytes);
    plan->off_col_nar = take(plan->col_nar_bytes);
    plan->off_partial = take(plan->partial_bytes);
    plan->workspace_bytes = off;
    return 0;
}

static int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

static int grid_for(int64_t items, int threads) {
    int64_t b = (items + threads - 1) / threads;
    if (b > 148 * 64) b = 148 * 64;
    if (b < 1) b = 1;
    return int(b);
}

template <int D, typename CodeT>
static cudaError_t launch_typed(const QuireGemmPlan& p, const PositFmt& f, const CodeT* A,
                                const CodeT* B, CodeT* C, int64_t M, int64_t N, int64_t K,
                                int64_t lda, int64_t ldb, int64_t ldc, uint8_t* ws,
                                cudaStream_t st, QuireGemmStats* stats) {
    using Geo = Geometry<D>;
    int8_t* a_img = reinterpret_cast<int8_t*>(ws + p.off_a);
    int8_t* b_img = reinterpret_cast<int8_t*>(ws + p.off_b);
    uint8_t* rnar = ws + p.off_row_nar;
    uint8_t* cnar = ws + p.off_col_nar;
    auto* partial = p.splits > 1 ? reinterpret_cast<unsigned __int128*>(ws + p.off_partial) : nullptr;
    cudaError_t e;
    if ((e = cudaMemsetAsync(rnar, 0, p.row_nar_bytes, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(cnar, 0, p.col_nar_bytes, st)) != cudaSuccess) return e;
    const int64_t a_items = p.mtiles * p.kbt * kBM * (Geo::KB / 16);
    const int64_t b_items = p.ntiles * p.kbt * Geo::NT * (Geo::KB / 16);
    if (stats) cudaEventRecord(stats->ev[0], st);
    pack_a_kernel<D, CodeT><<<grid_for(a_items, 256), 256, 0, st>>>(A, M, K, lda, f, a_img, rnar,
                                                                     p.kbt);
    pack_b_kernel<D, CodeT><<<grid_for(b_items, 256), 256, 0, st>>>(B, K, N, ldb, f, b_img, cnar,
                                                                     p.kbt);
    if (stats) cudaEventRecord(stats->ev[1], st);
    // D <= 3 implies R <= 11, hence W <= 64: no 128-bit instantiation needed.
    void (*kern)(const int8_t*, const int8_t*, int64_t, int64_t, const uint8_t*, const uint8_t*,
                 CodeT*, int64_t, int64_t, int64_t, PositFmt, unsigned __int128*, int64_t, int64_t,
                 int64_t);
    if constexpr (D <= 3)
        kern = f.W <= 32 ? quire_gemm_tc_kernel<D, 1, CodeT> : quire_gemm_tc_kernel<D, 2, CodeT>;
    else
        kern = f.W <= 64 ? quire_gemm_tc_kernel<D, 2, CodeT> : quire_gemm_tc_kernel<D, 4, CodeT>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM)) !=
        cudaSuccess)
        return e;
    const int64_t tiles = p.mtiles * p.ntiles * p.splits;
    const int grid = int(tiles < num_sms() ? tiles : num_sms());
    kern<<<grid, kThreads, Geo::SMEM, st>>>(a_img, b_img, p.kbt, p.kb_per_split, rnar, cnar, C, M,
                                            N, ldc, f, partial, p.mtiles, p.ntiles, p.splits);
    if (stats) cudaEventRecord(stats->ev[2], st);
    if (p.splits > 1) {
        quire_finalize_kernel<CodeT><<<grid_for(M * N, 256), 256, 0, st>>>(
            partial, int(p.splits), rnar, cnar, C, M, N, ldc, f);
    }
    if (stats) cudaEventRecord(stats->ev[3], st);
    return cudaGetLastError();
}

int quire_gemm_launch(int nbits, int es, const void* A, const void* B, void* C, int64_t M,
                      int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc, void* workspace,
                      size_t workspace_bytes, int64_t max_kb_per_split, cudaStream_t st,
                      QuireGemmStats* stats) {
    QuireGemmPlan p;
    int rc = quire_gemm_plan(nbits, es, M, N, K, max_kb_per_split, &p);
    if (rc) return rc;
    if (workspace_bytes < p.workspace_bytes) return 3;
    const PositFmt f = make_fmt(nbits, es);
    auto* ws = static_cast<uint8_t*>(workspace);
    cudaError_t e = cudaSuccess;
#define PNN_CASE(DD)                                                                              \
    case DD:                                                                                      \
        e = nbits <= 8 ? launch_typed<DD, uint8_t>(p, f, (const uint8_t*)A, (const uint8_t*)B,   \
                                                   (uint8_t*)C, M, N, K, lda, ldb, ldc, ws, st,  \
                                                   stats)                                         \
                       : launch_typed<DD, uint16_t>(p, f, (const uint16_t*)A, (const uint16_t*)B, \
                                                    (uint16_t*)C, M, N, K, lda, ldb, ldc, ws, st, \
                                                    stats);                                       \
        break;
    switch (p.D) {
        PNN_CASE(2)
        PNN_CASE(3)
        PNN_CASE(4)
        PNN_CASE(5)
        PNN_CASE(6)
        PNN_CASE(7)
        PNN_CASE(8)
        default: return 2;
    }
#undef PNN_CASE
    return e == cudaSuccess ? 0 : 4;
}

}  // namespace pnn_b200
