// Host side of the implicit-GEMM convolution path: eligibility, workspace
// plan, digitising launches, TMA tensor maps, kernel dispatch, NaR fix-ups.
// See igemm_core.cuh for the kernel; conv.cu routes the C-ABI calls here.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "igemm.h"
#include "igemm_core.cuh"

namespace pnn_b200 {

static int g_conv_algo = 0;
int conv_algo() { return g_conv_algo; }
int set_conv_algo(int a) {
    const int prev = g_conv_algo;
    g_conv_algo = a;
    return prev;
}

namespace {

// N tile: modes 0/1 two CTAs per SM (small_nt), mode 2 the one-CTA TileCfg tile
int nt_for(int D, int mode) {
    if (mode != 2 && D <= 4) return small_nt(D);
    return D == 2 ? TileCfg<2>::NT : D <= 4 ? TileCfg<4>::NT : TileCfg<8>::NT;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Output-pixel raster tiles of 128 rows: whole rows of width Wt; either an
// image spans tiles of Hb rows or a tile holds 128 / (Ht*Wt) whole images.
bool tile_geom(int64_t Ht, int64_t Wt, int* tpi, int* ipt, int* Hb) {
    if (Wt < 1 || Wt > 128 || Ht < 1) return false;
    const int64_t P = Ht * Wt;
    if (P >= 128) {
        if (128 % Wt || Ht % (128 / Wt)) return false;
        *Hb = int(128 / Wt);
        *tpi = int(P / 128);
        *ipt = 0;
    } else {
        if (128 % P) return false;
        *Hb = int(Ht);
        *tpi = 0;
        *ipt = int(128 / P);
    }
    return true;
}

struct ImplPlan {
    int mode, D, NT;
    IgemmArgs a;
    int64_t Ca, Wa, Ha;     // A digit tensor [D][N][Ha][Wa][Ca]
    uint32_t boxA[5];       // slice-layout box {2 * w, h, n, slices, planes}
    int64_t Kp, brows;      // modes 0/1: B digits [D][brows][taps * Kp]
    int64_t Fpw;            // mode 2: B digits [D][N][OH][OW][Fpw]
    size_t adig, bdig;      // bytes
    size_t off_adig, off_bdig, off_col_add, off_lut, off_maps, maps_bytes, off_pos_nar, off_chw_nar,
        off_col_nar, off_flags, off_partial, total;
    bool fold;    // first-layer tap folding: planned on the virtual 1x1 geometry gv
    int ckk;      // C * KH * KW of the real layer
    ConvGeom gv;  // geometry the plan runs on (== the real one unless folded)
};

// A first layer with few input channels (C*KH*KW <= 32, stride 1) runs as a
// 1x1 convolution over the folded receptive fields (im2col_digits_kernel):
// one 32-wide K block for the forward pass, one 32-row M tile for the weight
// gradient.  (Its input gradient is never needed, so pass 1 does not fold.)
bool fold_geom(int pass, const ConvGeom& g, ConvGeom* gv) {
    if (pass == 1 || g.stride != 1 || g.C % 32 == 0 || g.C * g.KH * g.KW > 32) return false;
    *gv = g;
    gv->C = 32;
    gv->H = g.OH;
    gv->W = g.OW;
    gv->KH = gv->KW = 1;
    gv->pad = 0;
    return true;
}

bool make_plan(int pass, const PositFmt& f, const ConvGeom& g_real, bool raw, ImplPlan* p) {
    if (conv_algo() == 1 || g_real.stride != 1) return false;
    if (g_real.N < 1 || g_real.N > (1 << 30)) return false;
    const int D = digits_for(f);
    if (D < 2 || D > 8) return false;
    *p = ImplPlan{};
    p->ckk = int(g_real.C * g_real.KH * g_real.KW);
    p->gv = g_real;
    p->fold = fold_geom(pass, g_real, &p->gv);
    const ConvGeom& g = p->gv;
    p->mode = pass;
    p->D = D;
    p->NT = nt_for(D, pass);
    IgemmArgs& a = p->a;
    a.f = f;
    static const int debug = getenv("PNN_IGEMM_DEBUG") ? atoi(getenv("PNN_IGEMM_DEBUG")) : 0;
    a.debug = debug;  // profiling experiments only: results are wrong when set
    a.KW = int(g.KW);
    a.pad = g.pad;
    const int64_t taps = g.KH * g.KW;
    a.taps = int(taps);
    size_t pos_nar = 0, chw_nar = 0, col_nar = 0, col_add = 0;
    if (pass == 0 || pass == 1) {
        const int64_t Cin = pass == 0 ? g.C : g.F;         // contracted channels
        const int64_t Cout = pass == 0 ? g.F : g.C;
        const int64_t Ht = pass == 0 ? g.OH : g.H, Wt = pass == 0 ? g.OW : g.W;
        const int64_t Hs = pass == 0 ? g.H : g.OH, Ws = pass == 0 ? g.W : g.OW;
        if (Cin % 32 || Ws > 256) return false;
        int tpi, ipt, Hb;
        if (!tile_geom(Ht, Wt, &tpi, &ipt, &Hb)) return false;
        a.tiles_per_img = tpi;
        a.imgs_per_tile = ipt;
        a.Hb = Hb;
        a.cch = int(Cin / 32);
        a.M = g.N * Ht * Wt;
        a.N = Cout;
        a.mtiles = tpi > 0 ? g.N * tpi : cdiv(g.N, ipt);
        a.ntiles = cdiv(Cout, p->NT);
        a.kbt = taps * Cin / 32;
        p->Ca = Cin;
        p->Wa = Ws;
        p->Ha = Hs;
        p->boxA[0] = uint32_t(2 * Wt);
        p->boxA[1] = uint32_t(Hb);
        p->boxA[2] = uint32_t(tpi > 0 ? 1 : ipt);
        p->boxA[3] = 2;  // one 32-channel K step
        p->boxA[4] = uint32_t(D);
        p->Kp = Cin;
        p->brows = Cout;
        p->adig = size_t(D) * g.N * Hs * Ws * Cin;
        p->bdig = size_t(D) * Cout * taps * Cin;
        pos_nar = size_t(g.N) * Hs * Ws;
        if (pass == 0) {
            col_nar = size_t(Cout);
            col_add = size_t(Cout) * 8;
        }
    } else {
        if (g.C % 32 || g.W > 256 || g.OW > 256) return false;
        int OWb, OHb;
        if (g.OW >= 32) {
            if (g.OW % 32) return false;
            OWb = 32;
            OHb = 1;
        } else {
            if (32 % g.OW || g.OH % (32 / g.OW)) return false;
            OWb = int(g.OW);
            OHb = int(32 / g.OW);
        }
        a.OWb = OWb;
        a.OHb = OHb;
        a.C = int(g.C);
        a.kpr = int(g.OW / OWb);
        a.kpi = int((g.OH / OHb) * a.kpr);
        a.KH = int(g.KH);
        a.kgroups = int((g.KW + 3) / 4);
        a.cgroups = int(g.C / 32);
        a.Hp = int(g.H + 2 * g.pad);
        a.mtiles = int64_t(a.KH) * a.kgroups * a.cgroups;
        a.M = a.mtiles * kBM;  // padding rows (kx >= KW, folded c >= C*KH*KW) not stored
        a.N = g.F;
        p->Fpw = cdiv(g.F, p->NT) * p->NT;
        a.ntiles = p->Fpw / p->NT;
        a.kbt = g.N * a.kpi;
        p->Ca = g.C;
        p->Wa = g.W + 2 * g.pad;  // zero-padded x digits
        p->Ha = g.H + 2 * g.pad;
        p->boxA[0] = uint32_t(2 * OWb);
        p->boxA[1] = uint32_t(OHb);
        p->boxA[2] = 4;   // kx taps of one group
        p->boxA[3] = 2;   // one 32-channel group
        p->boxA[4] = uint32_t(D);
        // + margin: the dummy kx taps of the last row read up to 3 pixels past it
        p->adig = size_t(D) * g.N * p->Ha * p->Wa * g.C + 64;
        p->bdig = size_t(D) * g.N * g.OH * g.OW * p->Fpw;
        chw_nar = size_t(g.C) * g.H * g.W;
        col_nar = size_t(p->Fpw);
    }
    // split-K: int32 group sums exact for <= 131071 / D terms (W > 32), SM fill
    const int64_t cap = f.W <= 32 ? a.kbt : (131071 / D) / kIKB;
    const int64_t kbps = split_kblocks(a.kbt, cap < 1 ? 1 : cap, a.mtiles * a.ntiles,
                                       num_sms() * ((pass == 2 || D >= 5) ? 1 : 2));  // CTAs in flight
    a.kb_per_split = a.kbt < kbps ? a.kbt : kbps;
    a.splits = cdiv(a.kbt, a.kb_per_split);
    a.fd_split = FastDiv(uint32_t(a.mtiles * a.ntiles));
    a.fd_group = FastDiv(uint32_t(kGroupM * a.ntiles));
    a.fd_g8 = FastDiv(uint32_t(kGroupM));
    a.fd_glast = FastDiv(uint32_t(a.mtiles % kGroupM ? a.mtiles % kGroupM : kGroupM));
    if (a.mtiles * a.ntiles * a.splits >= (int64_t(1) << 31) || a.M >= (int64_t(1) << 31)) return false;
    const size_t partial = (a.splits > 1 || raw) ? size_t(a.splits) * a.M * a.N * 16 : 0;

    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    };
    p->off_adig = take(p->adig);
    p->off_bdig = take(p->bdig);
    p->off_col_add = take(col_add);
    p->off_lut = take(f.nbits <= kActLutBits ? size_t(8) << f.nbits : 0);
    p->off_maps = off;  // NaR maps and flags: zeroed by one memset
    p->off_pos_nar = take(pos_nar);
    p->off_chw_nar = take(chw_nar);
    p->off_col_nar = take(col_nar);
    p->off_flags = take(16);
    p->maps_bytes = off - p->off_maps;
    p->off_partial = take(partial);
    p->total = off;
    return true;
}

uint32_t* lut_of(const ImplPlan& p, uint8_t* ws) {
    return p.a.f.nbits <= kActLutBits ? reinterpret_cast<uint32_t*>(ws + p.off_lut) : nullptr;
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (fn == nullptr) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &ptr, 12000, cudaEnableDefault,
                                             &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

// Slice layout dig[D][N][H][C/16][W][16] (int8 digits, 16 channels per 16-byte
// cell) as a 5-D map of 8-byte elements {2W, H, N, C/16, D}: a box row is a run
// of pixels of one 16-channel slice, contiguous in HBM.  No swizzle: the
// canonical 8 x 16-byte core matrices of the UMMA layouts are exactly 8
// consecutive pixels of a slice.  box = {2 * pixels, h, n, slices, planes}.
bool map_act(CUtensorMap* m, void* base, int D, int64_t N, int64_t H, int64_t W, int64_t C,
             const uint32_t box[5]) {
    auto enc = encoder();
    if (!enc) return false;
    const int64_t CS = C / 16;
    const cuuint64_t dims[5] = {cuuint64_t(2 * W), cuuint64_t(H), cuuint64_t(N), cuuint64_t(CS),
                                cuuint64_t(D)};
    const cuuint64_t strides[4] = {cuuint64_t(CS * W * 16), cuuint64_t(H * CS * W * 16),
                                   cuuint64_t(W * 16), cuuint64_t(N * H * CS * W * 16)};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Zero-padded x digits dig[D][N][Hp][C/16][Wp][16] for the weight gradient as
// {2 * Wp, N * Hp, 4, C/16, D}: rows of all images stacked (the pad rows make
// that safe), and a 4-wide kx dimension of stride one 16-byte pixel -- an
// overlapping view, so ONE box {pixels, rows, 4 kx, 2 slices, D} holds the
// operand of 4 taps x 32 channels x D planes.
bool map_wgrad_x(CUtensorMap* m, void* base, int D, int64_t N, int64_t Hp, int64_t Wp, int64_t C,
                 const uint32_t box[5]) {
    auto enc = encoder();
    if (!enc) return false;
    const int64_t CS = C / 16;
    const cuuint64_t dims[5] = {cuuint64_t(2 * Wp), cuuint64_t(N * Hp), 4, cuuint64_t(CS),
                                cuuint64_t(D)};
    const cuuint64_t strides[4] = {cuuint64_t(CS * Wp * 16), 16, cuuint64_t(Wp * 16),
                                   cuuint64_t(N * Hp * CS * Wp * 16)};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Weight digits dig[D][K/16][rows][16] as a 3-D map {2 * rows, D, K/16} of
// 8-byte elements; box {2 * NT, D, 2} -> smem [2 slices][D][NT][16 B], i.e. the
// D planes concatenated along N with a uniform 128-byte 8-row stride.
bool map_weights(CUtensorMap* m, void* base, int D, int64_t rows, int64_t K, int NT) {
    auto enc = encoder();
    if (!enc) return false;
    const int64_t KS = K / 16;
    const cuuint64_t dims[3] = {cuuint64_t(2 * rows), cuuint64_t(D), cuuint64_t(KS)};
    const cuuint64_t strides[2] = {cuuint64_t(KS * rows * 16), cuuint64_t(rows * 16)};
    const cuuint32_t boxd[3] = {cuuint32_t(2 * NT), cuuint32_t(D), 2};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims, strides, boxd, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tile shape per pass (measured on B200, profiles/README.md):
//  * modes 0/1, D <= 4: two CTAs per SM, 256 TMEM columns each, small N tile --
//    one CTA's drain/rounding overlaps the other's MMAs;
//  * modes 0/1, D >= 5 and mode 2: one CTA per SM, full-TMEM N tile, one
//    accumulator buffer.  (Two CTAs per SM leave too few stages for D >= 5;
//    two accumulator buffers in one CTA need the small N tile, which doubles
//    the tiles and the per-tile TMEM drain -- TMEM reads run at 64 B/cycle/SM
//    -- and measured 25% slower.)
template <int MODE, int D>
constexpr int cps_of() { return (MODE == 2 || D >= 5) ? 1 : 2; }
template <int MODE, int D>
constexpr int acc_of() { return 1; }
template <int MODE, int D>
constexpr int nt_of() { return cps_of<MODE, D>() == 2 ? small_nt(D) : TileCfg<D>::NT; }

template <int D, typename CodeT, int MODE>
cudaError_t launch_kernel(const CUtensorMap& tA, const CUtensorMap& tB, const IgemmArgs& a,
                          OutMap<CodeT> out, cudaStream_t st) {
    constexpr int NTT = nt_of<MODE, D>(), CPS = cps_of<MODE, D>(), ACC = acc_of<MODE, D>();
    using Geo = ImplGeo<D, NTT, CPS, ACC>;
    void (*k)(CUtensorMap, CUtensorMap, IgemmArgs, OutMap<CodeT>);
    if constexpr (D <= 3)
        k = a.f.W <= 32 ? igemm_kernel<D, NTT, CPS, ACC, 1, CodeT, MODE>
                        : igemm_kernel<D, NTT, CPS, ACC, 2, CodeT, MODE>;
    else
        k = a.f.W <= 64 ? igemm_kernel<D, NTT, CPS, ACC, 2, CodeT, MODE>
                        : igemm_kernel<D, NTT, CPS, ACC, 4, CodeT, MODE>;
    // BASELINE formats: epilogue specialised on the compile-time format
    const int fid = fixed_fmt_id(a.f);
    if constexpr (D == 2 && sizeof(CodeT) == 1)
        if (fid == 1) k = igemm_kernel<2, NTT, CPS, ACC, 1, CodeT, MODE, 1>;
    if constexpr (D == 4 && sizeof(CodeT) == 1)
        if (fid == 2) k = igemm_kernel<4, NTT, CPS, ACC, 2, CodeT, MODE, 2>;
    if constexpr (D == 6 && sizeof(CodeT) == 2)
        if (fid == 3) k = igemm_kernel<6, NTT, CPS, ACC, 4, CodeT, MODE, 3>;
    if constexpr (D == 8 && sizeof(CodeT) == 2)
        if (fid == 4) k = igemm_kernel<8, NTT, CPS, ACC, 4, CodeT, MODE, 4>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM);
    if (e != cudaSuccess) return e;
    const int64_t tiles = a.mtiles * a.ntiles * a.splits;
    const int64_t slots = int64_t(CPS) * num_sms();
    const int grid = int(tiles < slots ? tiles : slots);
    k<<<grid, Geo::THREADS, Geo::SMEM, st>>>(tA, tB, a, out);
    return cudaGetLastError();
}

template <typename CodeT, int MODE>
cudaError_t dispatch(int D, const CUtensorMap& tA, const CUtensorMap& tB, const IgemmArgs& a,
                     OutMap<CodeT> out, cudaStream_t st) {
    switch (D) {
        case 2: return launch_kernel<2, CodeT, MODE>(tA, tB, a, out, st);
        case 3: return launch_kernel<3, CodeT, MODE>(tA, tB, a, out, st);
        case 4: return launch_kernel<4, CodeT, MODE>(tA, tB, a, out, st);
        case 5: return launch_kernel<5, CodeT, MODE>(tA, tB, a, out, st);
        case 6: return launch_kernel<6, CodeT, MODE>(tA, tB, a, out, st);
        case 7: return launch_kernel<7, CodeT, MODE>(tA, tB, a, out, st);
        case 8: return launch_kernel<8, CodeT, MODE>(tA, tB, a, out, st);
        default: return cudaErrorInvalidValue;
    }
}

template <typename CodeT>
cudaError_t act_digits(int D, const CodeT* x, int64_t N, int64_t C, int64_t H, int64_t W,
                       int64_t Cp, int pad, const PositFmt& f, uint32_t* lut, bool build_lut, int8_t* dig,
                       uint8_t* pos_nar, uint8_t* chw_nar, uint8_t* chan_nar, uint8_t* any,
                       cudaStream_t st) {
    // thread per (pixel, 32 channels): grid (pixel blocks, 32-channel chunks)
    if (N * H * W >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    const dim3 grid(unsigned((grid_for(N * H * W * (Cp / 32), 256) + Cp / 32 - 1) / (Cp / 32)),
                    unsigned(Cp / 32));
    const FastDiv fd_hw{uint32_t(H * W)}, fd_w{uint32_t(W)};
    if (lut == nullptr) build_lut = false;
#define PNN_ACT(DD)                                                                              \
    if (build_lut) digit_lut_kernel<DD><<<16, 256, 0, st>>>(f, lut);                             \
    act_digits_kernel<DD, CodeT><<<grid, 256, 0, st>>>(x, int(N), int(C), int(H), int(W), int(Cp), \
                                                       pad, fd_hw, fd_w, f, lut, dig, pos_nar,   \
                                                       chw_nar, chan_nar, any)
    switch (D) {
        case 2: PNN_ACT(2); break;
        case 3: PNN_ACT(3); break;
        case 4: PNN_ACT(4); break;
        case 5: PNN_ACT(5); break;
        case 6: PNN_ACT(6); break;
        case 7: PNN_ACT(7); break;
        case 8: PNN_ACT(8); break;
        default: return cudaErrorInvalidValue;
    }
#undef PNN_ACT
    return cudaGetLastError();
}

template <typename CodeT>
cudaError_t im2col_digits(int D, const CodeT* x, const ConvGeom& g, const PositFmt& f, uint32_t* lut,
                          int8_t* dig, uint8_t* pos_nar, uint8_t* chw_nar, uint8_t* any,
                          cudaStream_t st) {
    const int grid = grid_for(g.N * g.OH * g.OW, 256);  // thread per output pixel
    if (g.N * g.OH * g.OW >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    const FastDiv fd_p{uint32_t(g.OH * g.OW)}, fd_ow{uint32_t(g.OW)};
#define PNN_I2C(DD)                                                                          \
    if (lut) digit_lut_kernel<DD><<<16, 256, 0, st>>>(f, lut);                               \
    im2col_digits_kernel<DD, CodeT><<<grid, 256, 0, st>>>(                                   \
        x, int(g.N), int(g.C), int(g.H), int(g.W), int(g.KH), int(g.KW), g.pad, int(g.OH),   \
        int(g.OW), fd_p, fd_ow, f, lut, dig, pos_nar, chw_nar, any)
    switch (D) {
        case 2: PNN_I2C(2); break;
        case 3: PNN_I2C(3); break;
        case 4: PNN_I2C(4); break;
        case 5: PNN_I2C(5); break;
        case 6: PNN_I2C(6); break;
        case 7: PNN_I2C(7); break;
        case 8: PNN_I2C(8); break;
        default: return cudaErrorInvalidValue;
    }
#undef PNN_I2C
    return cudaGetLastError();
}

template <typename CodeT>
cudaError_t weight_digits(int D, const CodeT* w, const CodeT* bias, int64_t F, int64_t C,
                          int64_t taps, int64_t Kp, int transpose, const PositFmt& f, int8_t* dig,
                          int64_t* col_add, uint8_t* col_nar, uint8_t* any, cudaStream_t st) {
    const int64_t total = (transpose ? C : F) * taps * Kp;
    const int grid = grid_for(total > F ? total : F, 256);
#define PNN_WD(DD)                                                                              \
    weight_digits_kernel<DD, CodeT><<<grid, 256, 0, st>>>(w, bias, int(F), int(C), int(taps),  \
                                                          int(Kp), transpose, f, dig, col_add, \
                                                          col_nar, any)
    switch (D) {
        case 2: PNN_WD(2); break;
        case 3: PNN_WD(3); break;
        case 4: PNN_WD(4); break;
        case 5: PNN_WD(5); break;
        case 6: PNN_WD(6); break;
        case 7: PNN_WD(7); break;
        case 8: PNN_WD(8); break;
        default: return cudaErrorInvalidValue;
    }
#undef PNN_WD
    return cudaGetLastError();
}

int rc_of(cudaError_t e) { return e == cudaSuccess ? 0 : 4; }

template <typename CodeT>
int run_fwd(const ImplPlan& p, const ConvGeom& g, const CodeT* x, const CodeT* w,
            const CodeT* bias, CodeT* y, uint8_t* ws, cudaStream_t st) {
    const PositFmt& f = p.a.f;
    auto* adig = reinterpret_cast<int8_t*>(ws + p.off_adig);
    auto* bdig = reinterpret_cast<int8_t*>(ws + p.off_bdig);
    auto* col_add = reinterpret_cast<int64_t*>(ws + p.off_col_add);
    uint8_t* pos_nar = ws + p.off_pos_nar;
    uint8_t* col_nar = ws + p.off_col_nar;
    uint8_t* flags = ws + p.off_flags;
    cudaError_t e;
    if ((e = cudaMemsetAsync(ws + p.off_maps, 0, p.maps_bytes, st)) != cudaSuccess) return 4;
    const ConvGeom& gv = p.gv;  // virtual 1x1 geometry when the first layer is folded
    if (p.fold)
        e = im2col_digits<CodeT>(p.D, x, g, f, lut_of(p, ws), adig, pos_nar, nullptr, flags, st);
    else
        e = act_digits<CodeT>(p.D, x, g.N, g.C, g.H, g.W, p.Ca, 0, f, lut_of(p, ws), true, adig,
                              pos_nar, nullptr, nullptr, flags, st);
    if (e != cudaSuccess) return 4;
    const int64_t taps = gv.KH * gv.KW;  // weights: [F][C*KH*KW] read as [F][ckk][1][1] if folded
    if ((e = weight_digits<CodeT>(p.D, w, bias, g.F, p.fold ? p.ckk : g.C, taps, p.Kp, 0, f, bdig,
                                  col_add, col_nar, flags + 1, st)) != cudaSuccess)
        return 4;
    CUtensorMap tA, tB;
    if (!map_act(&tA, adig, p.D, gv.N, gv.H, gv.W, p.Ca, p.boxA) ||
        !map_weights(&tB, bdig, p.D, p.brows, taps * p.Kp, p.NT))
        return 5;
    IgemmArgs a = p.a;
    a.col_add = bias ? col_add : nullptr;
    a.col_nar = col_nar;
    const bool use_partial = a.splits > 1;
    a.partial = use_partial ? reinterpret_cast<unsigned __int128*>(ws + p.off_partial) : nullptr;
    const OutMap<CodeT> out = out_nchw<CodeT>(y, g.OH * g.OW, g.F);
    if ((e = dispatch<CodeT, 0>(p.D, tA, tB, a, out, st)) != cudaSuccess) return 4;
    if (use_partial)
        quire_finalize_kernel<CodeT><<<grid_for(a.M * a.N, 256), 256, 0, st>>>(
            a.partial, int(a.splits), nullptr, col_nar, out, a.M, a.N, f, nullptr, nullptr);
    fwd_nar_fixup_kernel<CodeT><<<grid_for(a.M, 256), 256, 0, st>>>(
        y, pos_nar, flags, g.N, int(g.F), int(gv.H), int(gv.W), int(g.OH), int(g.OW), int(gv.KH),
        int(gv.KW), gv.pad, 1u << (f.nbits - 1));
    return rc_of(cudaGetLastError());
}

template <typename CodeT>
int run_dgrad(const ImplPlan& p, const ConvGeom& g, const CodeT* dy, const CodeT* w, CodeT* dx,
              uint8_t* ws, cudaStream_t st) {
    const PositFmt& f = p.a.f;
    auto* adig = reinterpret_cast<int8_t*>(ws + p.off_adig);
    auto* bdig = reinterpret_cast<int8_t*>(ws + p.off_bdig);
    uint8_t* pos_nar = ws + p.off_pos_nar;
    uint8_t* flags = ws + p.off_flags;
    if (cudaMemsetAsync(ws + p.off_maps, 0, p.maps_bytes, st) != cudaSuccess) return 4;
    if (act_digits<CodeT>(p.D, dy, g.N, g.F, g.OH, g.OW, p.Ca, 0, f, lut_of(p, ws), true, adig, pos_nar, nullptr, nullptr,
                          flags, st) != cudaSuccess)
        return 4;
    const int64_t taps = g.KH * g.KW;
    if (weight_digits<CodeT>(p.D, w, nullptr, g.F, g.C, taps, p.Kp, 1, f, bdig, nullptr, nullptr,
                             flags + 1, st) != cudaSuccess)
        return 4;
    CUtensorMap tA, tB;
    if (!map_act(&tA, adig, p.D, g.N, g.OH, g.OW, p.Ca, p.boxA) ||
        !map_weights(&tB, bdig, p.D, p.brows, taps * p.Kp, p.NT))
        return 5;
    IgemmArgs a = p.a;
    a.col_add = nullptr;
    a.col_nar = nullptr;
    const bool use_partial = a.splits > 1;
    a.partial = use_partial ? reinterpret_cast<unsigned __int128*>(ws + p.off_partial) : nullptr;
    const OutMap<CodeT> out = out_nchw<CodeT>(dx, g.H * g.W, g.C);
    if (dispatch<CodeT, 1>(p.D, tA, tB, a, out, st) != cudaSuccess) return 4;
    if (use_partial)
        quire_finalize_kernel<CodeT><<<grid_for(a.M * a.N, 256), 256, 0, st>>>(
            a.partial, int(a.splits), nullptr, nullptr, out, a.M, a.N, f, nullptr, nullptr);
    const uint32_t nar = 1u << (f.nbits - 1);
    dgrad_nar_fixup_kernel<CodeT><<<grid_for(a.M, 256), 256, 0, st>>>(
        dx, pos_nar, flags, g.N, int(g.C), int(g.H), int(g.W), int(g.OH), int(g.OW), int(g.KH),
        int(g.KW), g.pad, nar);
    dgrad_weight_nar_kernel<CodeT><<<grid_for(a.M * a.N, 256), 256, 0, st>>>(dx, w, g, flags + 1,
                                                                             nar);
    return rc_of(cudaGetLastError());
}

template <typename CodeT>
int run_wgrad(const ImplPlan& p, const ConvGeom& g, const CodeT* dy, const CodeT* x, CodeT* dw,
              unsigned __int128* raw_words, uint8_t* raw_nar, uint8_t* ws, cudaStream_t st) {
    const PositFmt& f = p.a.f;
    auto* adig = reinterpret_cast<int8_t*>(ws + p.off_adig);
    auto* bdig = reinterpret_cast<int8_t*>(ws + p.off_bdig);
    uint8_t* chw_nar = ws + p.off_chw_nar;
    uint8_t* col_nar = ws + p.off_col_nar;
    uint8_t* flags = ws + p.off_flags;
    if (cudaMemsetAsync(ws + p.off_maps, 0, p.maps_bytes, st) != cudaSuccess) return 4;
    const ConvGeom& gv = p.gv;  // virtual 1x1 geometry when the first layer is folded
    cudaError_t e;
    if (p.fold)
        e = im2col_digits<CodeT>(p.D, x, g, f, lut_of(p, ws), adig, nullptr, chw_nar, flags, st);
    else
        e = act_digits<CodeT>(p.D, x, g.N, g.C, g.H, g.W, p.Ca, g.pad, f, lut_of(p, ws), true,
                              adig, nullptr, chw_nar, nullptr, flags, st);
    if (e != cudaSuccess) return 4;
    if (!p.fold && g.pad > 0) {  // zero the pad ring of the padded x digits
        const int64_t cells = int64_t(p.D) * g.N * (p.Ca / 16) *
                              (int64_t(2 * g.pad) * (g.W + 2 * g.pad) + g.H * 2 * g.pad);
        pad_zero_kernel<<<grid_for(cells, 256), 256, 0, st>>>(reinterpret_cast<uint4*>(adig),
                                                              int64_t(p.D) * g.N, int(g.H), int(g.W),
                                                              int(p.Ca / 16), g.pad);
    }
    if (act_digits<CodeT>(p.D, dy, g.N, g.F, g.OH, g.OW, p.Fpw, 0, f, lut_of(p, ws), false, bdig, nullptr, nullptr, col_nar,
                          flags + 1, st) != cudaSuccess)
        return 4;
    CUtensorMap tA, tB;
    const uint32_t boxB[5] = {uint32_t(2 * p.a.OWb), uint32_t(p.a.OHb), 1, uint32_t(p.NT / 16),
                              uint32_t(p.D)};
    if (!map_wgrad_x(&tA, adig, p.D, gv.N, p.Ha, p.Wa, p.Ca, p.boxA) ||
        !map_act(&tB, bdig, p.D, g.N, g.OH, g.OW, p.Fpw, boxB))
        return 5;
    IgemmArgs a = p.a;
    a.col_add = nullptr;
    a.col_nar = col_nar;
    const bool use_partial = a.splits > 1 || raw_words != nullptr;
    a.partial = use_partial ? reinterpret_cast<unsigned __int128*>(ws + p.off_partial) : nullptr;
    OutMap<CodeT> out{};
    out.base = dw;
    out.ldc = p.ckk;    // dw[f][(c,ky,kx)]
    out.mode = 3;       // rows: tiles (ky, kx group, 32-channel group) x (slice, kx, c16)
    out.kh = int(gv.KH);
    out.kw = int(gv.KW);
    out.kgroups = p.a.kgroups;
    out.cgroups = p.a.cgroups;
    out.cvalid = p.fold ? p.ckk : int(g.C);
    if (dispatch<CodeT, 2>(p.D, tA, tB, a, out, st) != cudaSuccess) return 4;
    if (use_partial)
        quire_finalize_kernel<CodeT><<<grid_for(a.M * a.N, 256), 256, 0, st>>>(
            a.partial, int(a.splits), nullptr, col_nar, out, a.M, a.N, f, raw_words, raw_nar);
    wgrad_nar_fixup_kernel<CodeT><<<grid_for(p.ckk, 128), 128, 0, st>>>(
        dw, raw_nar, chw_nar, flags, int(g.F), p.fold ? p.ckk : int(g.C), int(gv.H), int(gv.W),
        int(g.OH), int(g.OW), int(gv.KH), int(gv.KW), gv.pad, 1u << (f.nbits - 1));
    return rc_of(cudaGetLastError());
}

}  // namespace

bool igemm_eligible(int pass, const PositFmt& f, const ConvGeom& g, bool raw, size_t* bytes) {
    ImplPlan p;
    if (!make_plan(pass, f, g, raw, &p)) return false;
    if (bytes) *bytes = p.total;
    return true;
}

int igemm_conv_fwd(const PositFmt& f, const ConvGeom& g, const void* x, const void* w,
                   const void* bias, void* y, void* ws, size_t ws_bytes, cudaStream_t st) {
    ImplPlan p;
    if (!make_plan(0, f, g, false, &p)) return 2;
    if (ws_bytes < p.total) return 3;
    auto* b = static_cast<uint8_t*>(ws);
    if (f.nbits <= 8)
        return run_fwd<uint8_t>(p, g, (const uint8_t*)x, (const uint8_t*)w, (const uint8_t*)bias,
                                (uint8_t*)y, b, st);
    return run_fwd<uint16_t>(p, g, (const uint16_t*)x, (const uint16_t*)w, (const uint16_t*)bias,
                             (uint16_t*)y, b, st);
}

int igemm_conv_dgrad(const PositFmt& f, const ConvGeom& g, const void* dy, const void* w, void* dx,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
    ImplPlan p;
    if (!make_plan(1, f, g, false, &p)) return 2;
    if (ws_bytes < p.total) return 3;
    auto* b = static_cast<uint8_t*>(ws);
    if (f.nbits <= 8)
        return run_dgrad<uint8_t>(p, g, (const uint8_t*)dy, (const uint8_t*)w, (uint8_t*)dx, b, st);
    return run_dgrad<uint16_t>(p, g, (const uint16_t*)dy, (const uint16_t*)w, (uint16_t*)dx, b, st);
}

int igemm_conv_wgrad(const PositFmt& f, const ConvGeom& g, const void* dy, const void* x, void* dw,
                     unsigned __int128* raw_words, uint8_t* raw_nar, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
    ImplPlan p;
    if (!make_plan(2, f, g, raw_words != nullptr, &p)) return 2;
    if (ws_bytes < p.total) return 3;
    auto* b = static_cast<uint8_t*>(ws);
    if (f.nbits <= 8)
        return run_wgrad<uint8_t>(p, g, (const uint8_t*)dy, (const uint8_t*)x, (uint8_t*)dw,
                                  raw_words, raw_nar, b, st);
    return run_wgrad<uint16_t>(p, g, (const uint16_t*)dy, (const uint16_t*)x, (uint16_t*)dw,
                               raw_words, raw_nar, b, st);
}

}  // namespace pnn_b200

extern "C" int pnn_conv_algo(int algo) {
    if (algo < 0 || algo > 2) return -1;
    return pnn_b200::set_conv_algo(algo);
}
