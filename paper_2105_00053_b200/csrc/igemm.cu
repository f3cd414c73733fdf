// Host side of the implicit-GEMM convolution path: eligibility, workspace
// plan, digitising launches, TMA tensor maps, kernel dispatch, NaR fix-ups.
// See igemm_core.cuh for the kernel; conv.cu routes the C-ABI calls here.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "igemm.h"
#include "tables.h"
#include "pdl.cuh"
#include "igemm_core.cuh"

namespace pnn_b200 {

static int g_conv_algo = 0;
static int64_t g_variant_min_work = int64_t(1) << 27;  // MACs below which no reduced variant launches
int64_t variant_min_work() { return g_variant_min_work; }
int64_t set_variant_min_work(int64_t v) {
    const int64_t prev = g_variant_min_work;
    g_variant_min_work = v;
    return prev;
}
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
    int DA, OFF;            // A digit planes / group offset (mode 2 from saved digits; else D, 0)
    IgemmArgs a;
    int64_t Ca, Wa, Ha;     // A digit tensor [D][N][Ha][Wa][Ca]
    uint32_t boxA[5];       // slice-layout box {2 * w, h, n, slices, planes}
    int64_t Kp, brows;      // modes 0/1: B digits [D][brows][taps * Kp]
    int64_t Fpw;            // mode 2: B digits [D][N][OH][OW][Fpw]
    size_t adig, bdig;      // bytes
    size_t off_adig, off_bdig, off_col_add, off_lut, off_lut2, off_maps, maps_bytes, off_pos_nar,
        off_chw_nar, off_col_nar, off_flags, off_partial, total;
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

bool make_plan(int pass, const PositFmt& f, const ConvGeom& g_real, bool raw, ImplPlan* p,
               int DA = 0, int OFF = 0, bool saved_x = false) {
    if (conv_algo() == 1 || g_real.stride != 1) return false;
    if (g_real.N < 1 || g_real.N > (1 << 30)) return false;
    // Linear layers (1x1 over 1x1 images): a TMA box would gather one 16-byte
    // pixel cell per image; the explicit path's contiguous bulk copies win
    // (fc1 of the CIFAR CNN: ~3x).  Forced implicit (algo 2) still allowed.
    if (conv_algo() == 0 && g_real.H == 1 && g_real.W == 1 && g_real.KH == 1 && g_real.KW == 1)
        return false;
    const int D = digits_for(f);
    if (D < 2 || D > 8) return false;
    *p = ImplPlan{};
    p->DA = DA > 0 ? DA : D;
    p->OFF = OFF;
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
        // forward: the x digits carry a stored zero ring (the weight gradient's
        // layout, so the same digits serve both passes); input grad: TMA OOB fill
        const int apad = pass == 0 ? g.pad : 0;
        a.apad = apad;
        a.M = g.N * Ht * Wt;
        a.N = Cout;
        a.mtiles = tpi > 0 ? g.N * tpi : cdiv(g.N, ipt);
        a.ntiles = cdiv(Cout, p->NT);
        a.kbt = taps * Cin / 32;
        p->Ca = Cin;
        p->Wa = Ws + 2 * apad;
        p->Ha = Hs + 2 * apad;
        p->boxA[0] = uint32_t(2 * Wt);
        p->boxA[1] = uint32_t(Hb);
        p->boxA[2] = uint32_t(tpi > 0 ? 1 : ipt);
        p->boxA[3] = 2;  // one 32-channel K step
        p->boxA[4] = uint32_t(D);
        p->Kp = Cin;
        p->brows = Cout;
        // + margin: the weight gradient's dummy kx taps read up to 3 pixels past the end
        p->adig = size_t(D) * g.N * p->Ha * p->Wa * Cin + 64;
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
        p->boxA[4] = uint32_t(p->DA);
        // + margin: the dummy kx taps of the last row read up to 3 pixels past it
        p->adig = size_t(p->DA) * g.N * p->Ha * p->Wa * g.C + 64;
        p->bdig = size_t(D) * g.N * g.OH * g.OW * p->Fpw;
        chw_nar = size_t(g.C) * g.H * g.W;
        col_nar = size_t(p->Fpw);
    }
    // split-K: int32 group sums exact for <= 131071 / D terms (W > 32), SM fill
    const int64_t cap = f.W <= 32 ? a.kbt : (131071 / D) / kIKB;
    // CTAs in flight: two per SM for the two-CTA kernels -- including the weight
    // gradient's reduced-digit variant (saved (8,1) digits under (12,1)), which
    // needs the second CTA's stages to keep enough TMA boxes in flight
    const bool wg_pair = pass == 2 && saved_x &&
                         ((D == 6 && ((p->DA == 4 && p->OFF == 1) || (p->DA == 6 && p->OFF == 0))) ||
                          (D == 8 && p->DA == 8 && p->OFF == 0));
    const int64_t kbps = split_kblocks(a.kbt, cap < 1 ? 1 : cap, a.mtiles * a.ntiles,
                                       num_sms() * (((pass == 2 && !wg_pair) || (pass != 2 && D >= 5)) ? 1 : 2));
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
    p->off_lut = take(size_t(8) << kActLutBits);   // digit LUTs by source code (<= 12 bits)
    p->off_lut2 = take(size_t(8) << kActLutBits);
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

// digit LUT for codes of format fs digitised in the plan's format (null: decode
// in registers, only when fs == f)
uint32_t* lut_of(const ImplPlan& p, uint8_t* ws, const PositFmt& fs, int which = 0) {
    return fs.nbits <= kActLutBits ? reinterpret_cast<uint32_t*>(ws + (which ? p.off_lut2 : p.off_lut))
                                   : nullptr;
}

bool same_fmt(const PositFmt& a, const PositFmt& b) { return a.nbits == b.nbits && a.es == b.es; }

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
bool map_weights(CUtensorMap* m, void* base, int D, int64_t rows, int64_t K, int NT, int box_planes = 0) {
    auto enc = encoder();
    if (!enc) return false;
    const int64_t KS = K / 16;
    const cuuint64_t dims[3] = {cuuint64_t(2 * rows), cuuint64_t(D), cuuint64_t(KS)};
    const cuuint64_t strides[2] = {cuuint64_t(KS * rows * 16), cuuint64_t(rows * 16)};
    const cuuint32_t boxd[3] = {cuuint32_t(2 * NT), cuuint32_t(box_planes > 0 ? box_planes : D), 2};
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

// PNN_WGRAD_NT64=0: the reduced weight gradient on 32-column tiles for wide layers too (A/B)
inline bool wgrad_nt64() {
    static const bool on = [] {
        const char* v = getenv("PNN_WGRAD_NT64");
        return v == nullptr || v[0] != '0';
    }();
    return on;
}

// PNN_IGEMM_ACC2=1: the reduced-digit forward / input-gradient kernels as ONE CTA
// per SM with two TMEM accumulator buffers and 16 epilogue warps (instead of
// two single-buffer CTAs): the MMA thread runs a whole tile ahead of the epilogue
inline bool igemm_acc2() {
    static const bool on = [] {
        const char* v = getenv("PNN_IGEMM_ACC2");
        return v != nullptr && v[0] == '1';
    }();
    return on;
}

template <int D, typename CodeT, int MODE, int DA, int OFF, int DB, int QWF, int NTT, int CPS, int ACC>
cudaError_t launch_kernel_geo(const CUtensorMap& tA, const CUtensorMap& tB, const IgemmArgs& a,
                              OutMap<CodeT> out, cudaStream_t st);

template <int D, typename CodeT, int MODE, int DA = D, int OFF = 0, int DB = D, int QWF = 0>
cudaError_t launch_kernel(const CUtensorMap& tA, const CUtensorMap& tB, const IgemmArgs& a,
                          OutMap<CodeT> out, cudaStream_t st) {
    // reduced-digit input gradient: (DA + DB - 1) * 32 <= 256 TMEM columns, so
    // two CTAs per SM overlap one's TMEM drain with the other's MMAs
    constexpr bool kPairSM = DB < D && (DA + DB - 1) * 32 <= 256;
    constexpr int NTT = kPairSM ? 32 : nt_of<MODE, D>();
    constexpr int CPS = kPairSM ? 2 : cps_of<MODE, D>(), ACC = acc_of<MODE, D>();
    if constexpr (kPairSM && MODE != 2)
        if (igemm_acc2()) return launch_kernel_geo<D, CodeT, MODE, DA, OFF, DB, QWF, NTT, 1, 2>(tA, tB, a, out, st);
    return launch_kernel_geo<D, CodeT, MODE, DA, OFF, DB, QWF, NTT, CPS, ACC>(tA, tB, a, out, st);
}

template <int D, typename CodeT, int MODE, int DA, int OFF, int DB, int QWF, int NTT, int CPS, int ACC>
cudaError_t launch_kernel_geo(const CUtensorMap& tA, const CUtensorMap& tB, const IgemmArgs& a_in,
                              OutMap<CodeT> out, cudaStream_t st) {
    using Geo = ImplGeo<D, NTT, CPS, ACC, DA, DB>;
    void (*k)(CUtensorMap, CUtensorMap, IgemmArgs, OutMap<CodeT>);
    IgemmArgs a = a_in;
    // 64-bit words of a W < 64 quire: with DA / DB-digit operands (|X| <= 128 *
    // (256^D - 1) / 255) the exact sum of K products (+ the bias term) stays
    // below 2^(W-1) for short K -- then the word is the value, no wrap to undo
    {
        const double ma = std::log2(128.0 * (std::pow(256.0, DA) - 1.0) / 255.0);
        const double mb = std::log2(128.0 * (std::pow(256.0, DB) - 1.0) / 255.0);
        const double k_terms = double(a.kbt) * kIKB + 1.0;
        a.nowrap = (MODE != 2 && a.f.W < 64 && ma + mb + std::log2(k_terms) < double(a.f.W - 1) - 0.01) ? 1 : 0;
    }
    const int fid = fixed_fmt_id(a.f);
    if constexpr (QWF != 0) {  // quire word forced by the caller (reduced-digit variants)
        k = igemm_kernel<D, NTT, CPS, ACC, QWF, CodeT, MODE, 0, DA, OFF, DB>;
        if constexpr (D == 6 && sizeof(CodeT) == 2)
            if (fid == 3) k = igemm_kernel<6, NTT, CPS, ACC, QWF, CodeT, MODE, 3, DA, OFF, DB>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM);
        if (e != cudaSuccess) return e;
        const int64_t tiles = a.mtiles * a.ntiles * a.splits;
        const int64_t slots = int64_t(CPS) * num_sms();
        return launch_pdl(k, dim3(unsigned(tiles < slots ? tiles : slots)), dim3(Geo::THREADS), Geo::SMEM, st,
                          tA, tB, a, out);
    }
    if constexpr (D <= 3)
        k = a.f.W <= 32 ? igemm_kernel<D, NTT, CPS, ACC, 1, CodeT, MODE, 0, DA, OFF, DB>
                        : igemm_kernel<D, NTT, CPS, ACC, 2, CodeT, MODE, 0, DA, OFF, DB>;
    else
        k = a.f.W <= 64 ? igemm_kernel<D, NTT, CPS, ACC, 2, CodeT, MODE, 0, DA, OFF, DB>
                        : igemm_kernel<D, NTT, CPS, ACC, 4, CodeT, MODE, 0, DA, OFF, DB>;
    // BASELINE formats: epilogue specialised on the compile-time format
    if constexpr (DA == D && DB == D) {
        if constexpr (D == 2 && sizeof(CodeT) == 1)
            if (fid == 1) k = igemm_kernel<2, NTT, CPS, ACC, 1, CodeT, MODE, 1>;
        if constexpr (D == 8 && sizeof(CodeT) == 2)
            if (fid == 4) k = igemm_kernel<8, NTT, CPS, ACC, 4, CodeT, MODE, 4>;
    }
    if constexpr (D == 4 && sizeof(CodeT) == 1)
        if (fid == 2) k = igemm_kernel<4, NTT, CPS, ACC, 2, CodeT, MODE, 2, DA, OFF, DB>;
    if constexpr (D == 6 && sizeof(CodeT) == 2)
        if (fid == 3) k = igemm_kernel<6, NTT, CPS, ACC, 4, CodeT, MODE, 3, DA, OFF, DB>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo::SMEM);
    if (e != cudaSuccess) return e;
    const int64_t tiles = a.mtiles * a.ntiles * a.splits;
    const int64_t slots = int64_t(CPS) * num_sms();
    const int grid = int(tiles < slots ? tiles : slots);
    return launch_pdl(k, dim3(unsigned(grid)), dim3(Geo::THREADS), Geo::SMEM, st, tA, tB, a, out);
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

// Weight-gradient A operands of DA planes at group offset OFF that have a
// kernel: the symmetric case, and posit(8,1) forward digits under a posit(12,1)
// gradient (BASELINE config 3: R 12 -> 20, one digit up).
// Input gradients whose weights all fit kDgradDB digits (|X_w| within the
// 3-digit balanced capacity, i.e. |w| < 8 in posit(12,1)): a variant with
// DB = 3 weight planes (half the MMAs, 8 instead of 11 TMEM groups) runs;
// the weight digitiser's flag selects it on the device (both variants are
// launched, the other exits at once), so no host round trip is needed.
constexpr int kDgradDB = 3;
// digit planes of the reduced variants: 3 (posit(8,1) / posit(12,1) classes),
// 4 for the 8-digit posit(16,1) class (|X| < 2^31: |v| < 8)
inline int red_planes(int D) { return D == 8 ? 4 : kDgradDB; }
bool dgrad_reduced(int D) { return D == 6 || D == 8; }
// the variants cost an extra (exiting) launch: only for passes with real work
inline bool variant_worthy(const IgemmArgs& a) { return a.M * a.N * a.kbt * kIKB >= variant_min_work(); }

template <typename CodeT>
cudaError_t dispatch_dgrad_reduced(int D, const CUtensorMap& tA, const CUtensorMap& tB, const IgemmArgs& a,
                                   OutMap<CodeT> out, cudaStream_t st) {
    if constexpr (sizeof(CodeT) == 2)
        if (D == 6) return launch_kernel<6, CodeT, 1, 6, 0, kDgradDB>(tA, tB, a, out, st);
    return cudaErrorInvalidValue;
}

// Both operands within 3 digits (dy too: |dy| < 8 in posit(12,1)): 3 x 3 digit
// MMAs, 5 TMEM groups; the exact sum then fits 64 bits for chunks below 2^17
// terms (|X| < 2^23 each), so a 64-bit quire word serves (single split only:
// split-K partials are 128-bit words).
template <typename CodeT>
cudaError_t dispatch_dgrad_33(int D, bool narrow_word, const CUtensorMap& tA, const CUtensorMap& tB,
                              const IgemmArgs& a, OutMap<CodeT> out, cudaStream_t st) {
    if constexpr (sizeof(CodeT) == 2)
        if (D == 6)
            return narrow_word ? launch_kernel<6, CodeT, 1, kDgradDB, 0, kDgradDB, 2>(tA, tB, a, out, st)
                               : launch_kernel<6, CodeT, 1, kDgradDB, 0, kDgradDB, 4>(tA, tB, a, out, st);
    return cudaErrorInvalidValue;
}

bool wgrad_variant(int D, int DA, int OFF) {
    return (DA == D && OFF == 0) || (D == 6 && DA == 4 && OFF == 1);
}

template <typename CodeT>
cudaError_t dispatch_wgrad(int D, int DA, int OFF, const CUtensorMap& tA, const CUtensorMap& tB,
                           const IgemmArgs& a, OutMap<CodeT> out, cudaStream_t st) {
    if (DA == D && OFF == 0) return dispatch<CodeT, 2>(D, tA, tB, a, out, st);
    if constexpr (sizeof(CodeT) == 2)
        if (D == 6 && DA == 4 && OFF == 1) return launch_kernel<6, CodeT, 2, 4, 1>(tA, tB, a, out, st);
    return cudaErrorInvalidValue;
}

// ---- digitisers: codes of format fs (uint8 for nbits <= 8, else uint16) ->
// digits of the plan format f (through the conversion LUT when fs != f)

// The digit table of (D, fs -> f) for the life of the process (tables.h);
// nullptr: build the per-call table in the workspace instead.
uint32_t* cached_digit_lut(int D, const PositFmt& fs, const PositFmt& f, cudaStream_t st) {
    if (D < 2 || D > 8) return nullptr;
    return static_cast<uint32_t*>(persistent_table(
        table_key(1, D, fs.nbits, fs.es, f.nbits, f.es), (size_t(2) << fs.nbits) * 4, st,
        [&](void* p, cudaStream_t s) {
            auto* l = static_cast<uint32_t*>(p);
            switch (D) {
                case 2: digit_lut_conv_kernel<2><<<16, 256, 0, s>>>(fs, f, l); break;
                case 3: digit_lut_conv_kernel<3><<<16, 256, 0, s>>>(fs, f, l); break;
                case 4: digit_lut_conv_kernel<4><<<16, 256, 0, s>>>(fs, f, l); break;
                case 5: digit_lut_conv_kernel<5><<<16, 256, 0, s>>>(fs, f, l); break;
                case 6: digit_lut_conv_kernel<6><<<16, 256, 0, s>>>(fs, f, l); break;
                case 7: digit_lut_conv_kernel<7><<<16, 256, 0, s>>>(fs, f, l); break;
                default: digit_lut_conv_kernel<8><<<16, 256, 0, s>>>(fs, f, l); break;
            }
        }));
}

template <typename SrcT>
cudaError_t act_digits_t(int D, const SrcT* x, int64_t N, int64_t C, int64_t H, int64_t W, int64_t Cp,
                         int pad, const PositFmt& f, const PositFmt& fs, uint32_t* lut, bool build_lut,
                         int8_t* dig, uint8_t* pos_nar, uint8_t* chw_nar, uint8_t* chan_nar,
                         uint8_t* any, cudaStream_t st, const DigitGate& gt, uint8_t* wide, int wide_planes,
                         int store_planes, const uint8_t* only_if, const uint8_t* only_if2) {
    // thread per (pixel, 32 channels): grid (pixel blocks, 32-channel chunks)
    if (N * H * W >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    const int64_t gx = (grid_for(N * H * W * (Cp / 32), 256) + Cp / 32 - 1) / (Cp / 32);
    const dim3 grid(unsigned(only_if != nullptr && gx > 148 ? 148 : gx), unsigned(Cp / 32));
    const FastDiv fd_hw{uint32_t(H * W)}, fd_w{uint32_t(W)};
    if (lut == nullptr) build_lut = false;
    // whole 256-pixel tiles per image, 16-byte aligned channel rows: staged loads
    const bool tiled = (H * W) % 256 == 0 && (256 % W == 0 || W % 256 == 0) &&
                       (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(gt.gate) & 15) == 0;
    const int64_t ntiles = N * H * W / 256;
    // a completion pass (only_if) usually exits at once: few blocks (grid-stride
    // loops cover the work when it does run)
    const int64_t tcap = only_if != nullptr ? 148 : 148 * 8;
    const dim3 tgrid(unsigned(ntiles < tcap ? ntiles : tcap), unsigned(Cp / 32));
#define PNN_ACT(DD)                                                                                  \
    if (build_lut) digit_lut_conv_kernel<DD><<<16, 256, 0, st>>>(fs, f, lut);                        \
    if (tiled && gt.gate == nullptr)                                                                 \
        launch_pdl(act_digits_tiled_kernel<DD, SrcT, 0>, dim3(tgrid), dim3(256), 0, st,                                  \
            x, int(N), int(C), int(H), int(W), int(Cp), pad, fd_hw, fd_w, f, fs, lut, dig, pos_nar,  \
            chw_nar, chan_nar, any, gt, wide, wide_planes, store_planes, only_if, only_if2);         \
    else if (tiled && gt.gb == 1)                                                                    \
        launch_pdl(act_digits_tiled_kernel<DD, SrcT, 1>, dim3(tgrid), dim3(256), 0, st,                                  \
            x, int(N), int(C), int(H), int(W), int(Cp), pad, fd_hw, fd_w, f, fs, lut, dig, pos_nar,  \
            chw_nar, chan_nar, any, gt, wide, wide_planes, store_planes, only_if, only_if2);         \
    else if (tiled)                                                                                  \
        launch_pdl(act_digits_tiled_kernel<DD, SrcT, 2>, dim3(tgrid), dim3(256), 0, st,                                  \
            x, int(N), int(C), int(H), int(W), int(Cp), pad, fd_hw, fd_w, f, fs, lut, dig, pos_nar,  \
            chw_nar, chan_nar, any, gt, wide, wide_planes, store_planes, only_if, only_if2);         \
    else                                                                                             \
        launch_pdl(act_digits_kernel<DD, SrcT>, dim3(grid), dim3(256), 0, st, x, int(N), int(C), int(H), int(W), int(Cp), \
                                                          pad, fd_hw, fd_w, f, fs, lut, dig, pos_nar, \
                                                          chw_nar, chan_nar, any, gt, wide, wide_planes, \
                                                          store_planes, only_if, only_if2)
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

cudaError_t act_digits(int D, const void* x, int64_t N, int64_t C, int64_t H, int64_t W, int64_t Cp,
                       int pad, const PositFmt& f, const PositFmt& fs, uint32_t* lut, bool build_lut,
                       int8_t* dig, uint8_t* pos_nar, uint8_t* chw_nar, uint8_t* chan_nar, uint8_t* any,
                       cudaStream_t st, const DigitGate& gt = DigitGate{}, uint8_t* wide = nullptr,
                       int wide_planes = 0, bool reduce_stores = false, const uint8_t* also_if = nullptr,
                       const uint8_t* only_if = nullptr) {
    if (lut == nullptr && !same_fmt(f, fs)) return cudaErrorInvalidValue;  // no in-register convert
    if (lut != nullptr && build_lut)
        if (uint32_t* c = cached_digit_lut(D, fs, f, st)) {
            lut = c;
            build_lut = false;
        }
    // reduce_stores (every consumer of these digits is a flag-selected variant):
    // store only the planes the reduced-digit kernels read, then a completion
    // pass (exits at once unless the wide flag is set) writes all planes
    // (also_if: a second flag whose consumers read the high planes too.)
    // only_if alone: a single full pass that runs iff *only_if (a later completion).
    const int sp = reduce_stores && wide != nullptr && wide_planes > 0 && wide_planes < D ? wide_planes : D;
    for (int pass = 0; pass < (sp < D ? 2 : 1); ++pass) {
        const int store = pass == 0 ? sp : D;
        const uint8_t* oi = pass == 0 ? only_if : wide;
        const uint8_t* oi2 = pass == 0 ? nullptr : also_if;
        const bool lut_now = build_lut && pass == 0;
        cudaError_t e =
            fs.nbits <= 8
                ? act_digits_t(D, static_cast<const uint8_t*>(x), N, C, H, W, Cp, pad, f, fs, lut, lut_now, dig,
                               pos_nar, chw_nar, chan_nar, any, st, gt, wide, wide_planes, store, oi, oi2)
                : act_digits_t(D, static_cast<const uint16_t*>(x), N, C, H, W, Cp, pad, f, fs, lut, lut_now, dig,
                               pos_nar, chw_nar, chan_nar, any, st, gt, wide, wide_planes, store, oi, oi2);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <typename SrcT>
cudaError_t im2col_digits_t(int D, const SrcT* x, const ConvGeom& g, const PositFmt& f,
                            const PositFmt& fs, uint32_t* lut, int8_t* dig, uint8_t* pos_nar,
                            uint8_t* chw_nar, uint8_t* any, cudaStream_t st, uint8_t* wide, int wide_planes) {
    const int grid = grid_for(g.N * g.OH * g.OW, 256);  // thread per output pixel
    if (g.N * g.OH * g.OW >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    const FastDiv fd_p{uint32_t(g.OH * g.OW)}, fd_ow{uint32_t(g.OW)};
    bool build = lut != nullptr;
    if (build)
        if (uint32_t* c = cached_digit_lut(D, fs, f, st)) {
            lut = c;
            build = false;
        }
#define PNN_I2C(DD)                                                                          \
    if (build) digit_lut_conv_kernel<DD><<<16, 256, 0, st>>>(fs, f, lut);                    \
    launch_pdl(im2col_digits_kernel<DD, SrcT>, dim3(grid), dim3(256), 0, st,                                    \
        x, int(g.N), int(g.C), int(g.H), int(g.W), int(g.KH), int(g.KW), g.pad, int(g.OH),   \
        int(g.OW), fd_p, fd_ow, f, fs, lut, dig, pos_nar, chw_nar, any, wide, wide_planes, DD,     \
        static_cast<const uint8_t*>(nullptr))
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

cudaError_t im2col_digits(int D, const void* x, const ConvGeom& g, const PositFmt& f, const PositFmt& fs,
                          uint32_t* lut, int8_t* dig, uint8_t* pos_nar, uint8_t* chw_nar, uint8_t* any,
                          cudaStream_t st, uint8_t* wide = nullptr, int wide_planes = 0) {
    if (lut == nullptr && !same_fmt(f, fs)) return cudaErrorInvalidValue;
    if (fs.nbits <= 8)
        return im2col_digits_t(D, static_cast<const uint8_t*>(x), g, f, fs, lut, dig, pos_nar, chw_nar, any, st,
                               wide, wide_planes);
    return im2col_digits_t(D, static_cast<const uint16_t*>(x), g, f, fs, lut, dig, pos_nar, chw_nar, any, st,
                           wide, wide_planes);
}

template <typename CodeT>
cudaError_t weight_digits(int D, const CodeT* w, const CodeT* bias, int64_t F, int64_t C,
                          int64_t taps, int64_t Kp, int transpose, const PositFmt& f, int8_t* dig,
                          int64_t* col_add, uint8_t* col_nar, uint8_t* any, cudaStream_t st,
                          uint8_t* wide = nullptr, int wide_planes = 0) {
    const int64_t total = (transpose ? C : F) * taps * Kp;
    const int grid = grid_for(total > F ? total : F, 256);
#define PNN_WD(DD)                                                                              \
    launch_pdl(weight_digits_kernel<DD, CodeT>, dim3(grid), dim3(256), 0, st, w, bias, int(F), int(C), int(taps),  \
                                                          int(Kp), transpose, f, dig, col_add, \
                                                          col_nar, any, wide, wide_planes)
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

// The forward pass's activation digits, kept for the weight gradient (the
// "saved tensor" of the layer): [D_f][N][Ha][Ca/16][Wa][16] digits of x in the
// forward format (zero ring stored; Ha/Wa/Ca of the wgrad plan), the NaR map
// chw_nar (any image) and an any-NaR flag.
struct SavedX {
    int8_t* dig;
    uint8_t* chw;
    uint8_t* flag;  // [0] any NaR in x, [1] x uses digit planes >= kDgradDB
};

struct SaveLayout {
    size_t dig, chw, total;  // offsets: chw at dig, flag at chw + chw bytes
    size_t chw_bytes;
};

bool save_layout(const PositFmt& f, const ConvGeom& g, SaveLayout* L) {
    ImplPlan pf, pw;
    if (!make_plan(0, f, g, false, &pf) || !make_plan(2, f, g, false, &pw)) return false;
    if (pf.fold != pw.fold) return false;
    auto r256 = [](size_t b) { return (b + 255) & ~size_t(255); };
    L->dig = r256(pf.adig);
    L->chw_bytes = pw.fold ? size_t(pw.ckk) * g.OH * g.OW : size_t(g.C) * g.H * g.W;
    L->chw = r256(L->chw_bytes);
    L->total = L->dig + L->chw + 256;
    return true;
}

SavedX saved_of(void* base, const SaveLayout& L) {
    auto* b = static_cast<uint8_t*>(base);
    return SavedX{reinterpret_cast<int8_t*>(b), b + L.dig, b + L.dig + L.chw};
}

template <typename CodeT>
int run_fwd(const ImplPlan& p, const ConvGeom& g, const CodeT* x, const CodeT* w,
            const CodeT* bias, CodeT* y, uint8_t* ws, cudaStream_t st, const SavedX* sv,
            size_t sv_clear, int relu = 0, CodeT* pre = nullptr) {
    const PositFmt& f = p.a.f;
    auto* adig = sv ? sv->dig : reinterpret_cast<int8_t*>(ws + p.off_adig);
    auto* bdig = reinterpret_cast<int8_t*>(ws + p.off_bdig);
    auto* col_add = reinterpret_cast<int64_t*>(ws + p.off_col_add);
    uint8_t* pos_nar = ws + p.off_pos_nar;
    uint8_t* col_nar = ws + p.off_col_nar;
    uint8_t* flags = ws + p.off_flags;
    uint8_t* xflag = sv ? sv->flag : flags;  // any NaR in x
    cudaError_t e;
    if ((e = cudaMemsetAsync(ws + p.off_maps, 0, p.maps_bytes, st)) != cudaSuccess) return 4;
    if (sv && (e = cudaMemsetAsync(sv->chw, 0, sv_clear, st)) != cudaSuccess) return 4;
    const ConvGeom& gv = p.gv;  // virtual 1x1 geometry when the first layer is folded
    // x's digit-plane flag (the reduced-digit variants of this pass and of the weight gradient)
    uint8_t* xwide = sv ? sv->flag + 1 : flags + 3;
    if (p.fold)
        e = im2col_digits(p.D, x, g, f, f, lut_of(p, ws, f), adig, pos_nar, sv ? sv->chw : nullptr, xflag, st,
                          xwide, red_planes(p.D));
    else
        e = act_digits(p.D, x, g.N, g.C, g.H, g.W, p.Ca, g.pad, f, f, lut_of(p, ws, f), true, adig,
                       pos_nar, sv ? sv->chw : nullptr, nullptr, xflag, st, DigitGate{}, xwide, red_planes(p.D));
    if (e != cudaSuccess) return 4;
    const int64_t taps = gv.KH * gv.KW;  // weights: [F][C*KH*KW] read as [F][ckk][1][1] if folded
    // reduced-digit variant (posit(8,1) / posit(12,1): x and w within 3 balanced digits)
    const bool reduced = ((p.D == 4 && sizeof(CodeT) == 1) ||
                          ((p.D == 6 || p.D == 8) && sizeof(CodeT) == 2)) && variant_worthy(p.a);
    const int RP = red_planes(p.D);
    uint8_t* wwide = flags + 2;
    if ((e = weight_digits<CodeT>(p.D, w, bias, g.F, p.fold ? p.ckk : g.C, taps, p.Kp, 0, f, bdig,
                                  col_add, col_nar, flags + 1, st, reduced ? wwide : nullptr, RP)) !=
        cudaSuccess)
        return 4;
    CUtensorMap tA, tB, tA3, tB3;
    uint32_t boxA3[5];
    for (int i = 0; i < 5; ++i) boxA3[i] = p.boxA[i];
    boxA3[4] = RP;
    if (!map_act(&tA, adig, p.D, gv.N, p.Ha, p.Wa, p.Ca, p.boxA) ||
        !map_weights(&tB, bdig, p.D, p.brows, taps * p.Kp, p.NT) ||
        (reduced && (!map_act(&tA3, adig, p.D, gv.N, p.Ha, p.Wa, p.Ca, boxA3) ||
                     !map_weights(&tB3, bdig, p.D, p.brows, taps * p.Kp, p.NT, RP))))
        return 5;
    IgemmArgs a = p.a;
    a.col_add = bias ? col_add : nullptr;
    a.col_nar = col_nar;
    const bool use_partial = a.splits > 1;
    a.partial = use_partial ? reinterpret_cast<unsigned __int128*>(ws + p.off_partial) : nullptr;
    a.relu = relu;
    a.pre_out = pre;
    const OutMap<CodeT> out = out_nchw<CodeT>(y, g.OH * g.OW, g.F);
    if (reduced) {  // both launched; the x / w plane flags let exactly one run
        a.vflag = xwide;
        a.vflag2 = wwide;
        a.vexpect = a.vexpect2 = 0;
        if constexpr (sizeof(CodeT) == 1) {
            // >= 64 output channels: 64-column tiles on one CTA per SM read each activation
            // box once per 64 channels (conv3 / conv4 of the CIFAR CNN: 56.2 -> 53.3 and
            // 82.8 -> 80.1 us); PNN_FWD_NT64=0: 32-column tiles on two CTAs per SM
            static const bool nt64 = [] {
                const char* v = getenv("PNN_FWD_NT64");
                return v == nullptr || v[0] != '0';
            }();
            if (nt64 && p.D == 4 && p.NT == 32 && a.ntiles % 2 == 0 && a.splits == 1) {
                IgemmArgs a2 = a;
                a2.ntiles = a.ntiles / 2;
                a2.fd_split = FastDiv(uint32_t(a2.mtiles * a2.ntiles));
                a2.fd_group = FastDiv(uint32_t(kGroupM * a2.ntiles));
                CUtensorMap tB64;
                if (!map_weights(&tB64, bdig, p.D, p.brows, taps * p.Kp, 64, RP)) return 5;
                e = launch_kernel_geo<4, CodeT, 0, kDgradDB, 0, kDgradDB, 0, 64, 1, 1>(tA3, tB64, a2, out, st);
            } else {
                e = launch_kernel<4, CodeT, 0, kDgradDB, 0, kDgradDB>(tA3, tB3, a, out, st);
            }
            if (e != cudaSuccess) return 4;
        }
        if constexpr (sizeof(CodeT) == 2) {
            if (p.D == 6) {  // 64-bit quire word when a single chunk's exact sum fits
                const bool narrow_word = a.splits == 1 && a.kb_per_split * kIKB < (int64_t(1) << 17);
                e = narrow_word ? launch_kernel<6, CodeT, 0, kDgradDB, 0, kDgradDB, 2>(tA3, tB3, a, out, st)
                                : launch_kernel<6, CodeT, 0, kDgradDB, 0, kDgradDB, 4>(tA3, tB3, a, out, st);
            } else {
                e = launch_kernel<8, CodeT, 0, 4, 0, 4, 4>(tA3, tB3, a, out, st);
            }
            if (e != cudaSuccess) return 4;
        }
        a.vor = 1;
        a.vexpect = 1;
    }
    if ((e = dispatch<CodeT, 0>(p.D, tA, tB, a, out, st)) != cudaSuccess) return 4;
    if (use_partial) {
        launch_finalize<CodeT>(a.partial, int(a.splits), nullptr, col_nar, out, a.M, a.N, f, nullptr, nullptr, st);
        if (relu)
            launch_pdl(relu_codes_kernel<CodeT>, dim3(grid_for(a.M * a.N, 256)), dim3(256), 0, st, y, pre, a.M * a.N, f.nbits);
    }
    launch_pdl(fwd_nar_fixup_kernel<CodeT>, dim3(grid_fixup(a.M)), dim3(256), 0, st, 
        y, pos_nar, xflag, g.N, int(g.F), int(gv.H), int(gv.W), int(g.OH), int(g.OW), int(gv.KH),
        int(gv.KW), gv.pad, 1u << (f.nbits - 1), relu, pre);
    return rc_of(cudaGetLastError());
}

// Input gradient.  pre: dy already digitised in the plan's layout by the
// weight-gradient pass (shared operand) -- its digits, pixel NaR map and
// any-NaR flag; otherwise dy is digitised here.
struct DyDigits {
    const int8_t* dig;
    const uint8_t* pos_nar;
    const uint8_t* any;
    const uint8_t* wide;  // dy uses digit planes >= kDgradDB (null: unknown)
};

template <typename CodeT>
int run_dgrad(const ImplPlan& p, const ConvGeom& g, const CodeT* dy, const CodeT* w, CodeT* dx,
              uint8_t* ws, cudaStream_t st, const DyDigits* pre = nullptr,
              const DigitGate& gt = DigitGate{}) {
    const PositFmt& f = p.a.f;
    auto* adig = reinterpret_cast<int8_t*>(ws + p.off_adig);
    auto* bdig = reinterpret_cast<int8_t*>(ws + p.off_bdig);
    uint8_t* pos_nar = ws + p.off_pos_nar;
    uint8_t* flags = ws + p.off_flags;
    // (with pre, the caller cleared the maps before dy's digitiser filled pos_nar)
    if (pre == nullptr && cudaMemsetAsync(ws + p.off_maps, 0, p.maps_bytes, st) != cudaSuccess) return 4;
    const bool reduced = dgrad_reduced(p.D) && sizeof(CodeT) == 2 && variant_worthy(p.a);
    const int RP = red_planes(p.D);
    if (pre == nullptr &&
        act_digits(p.D, dy, g.N, g.F, g.OH, g.OW, p.Ca, 0, f, f, lut_of(p, ws, f), true, adig, pos_nar,
                   nullptr, nullptr, flags, st, gt, reduced ? flags + 3 : nullptr, RP, reduced) != cudaSuccess)
        return 4;
    const int8_t* a_dig = pre ? pre->dig : adig;
    const uint8_t* a_pos = pre ? pre->pos_nar : pos_nar;
    const uint8_t* a_any = pre ? pre->any : flags;
    const uint8_t* dy_wide = pre ? pre->wide : (reduced ? flags + 3 : nullptr);
    const int64_t taps = g.KH * g.KW;
    uint8_t* wide = flags + 2;  // weights need more than kDgradDB digit planes
    if (weight_digits<CodeT>(p.D, w, nullptr, g.F, g.C, taps, p.Kp, 1, f, bdig, nullptr, nullptr,
                             flags + 1, st, reduced ? wide : nullptr, RP) != cudaSuccess)
        return 4;
    // dy's digits were stored without the high planes (narrow dy): the full
    // variant, selected by wide weights, reads them -- complete dy then
    if (reduced && dy_wide != nullptr &&
        act_digits(p.D, dy, g.N, g.F, g.OH, g.OW, p.Ca, 0, f, f, lut_of(p, ws, f), true,
                   const_cast<int8_t*>(a_dig), nullptr, nullptr, nullptr, flags + 4, st, gt, nullptr, 0, false,
                   nullptr, wide) != cudaSuccess)
        return 4;
    CUtensorMap tA, tA3, tB, tB3;
    uint32_t box3[5];
    for (int i = 0; i < 5; ++i) box3[i] = p.boxA[i];
    box3[4] = RP;  // A box of the reduced variant: dy's low digit planes
    if (!map_act(&tA, const_cast<int8_t*>(a_dig), p.D, g.N, g.OH, g.OW, p.Ca, p.boxA) ||
        !map_weights(&tB, bdig, p.D, p.brows, taps * p.Kp, p.NT) ||
        (reduced && !map_weights(&tB3, bdig, p.D, p.brows, taps * p.Kp, p.NT, RP)) ||
        (reduced && dy_wide && !map_act(&tA3, const_cast<int8_t*>(a_dig), p.D, g.N, g.OH, g.OW, p.Ca, box3)))
        return 5;
    IgemmArgs a = p.a;
    a.col_add = nullptr;
    a.col_nar = nullptr;
    const bool use_partial = a.splits > 1;
    a.partial = use_partial ? reinterpret_cast<unsigned __int128*>(ws + p.off_partial) : nullptr;
    const OutMap<CodeT> out = out_nchw<CodeT>(dx, g.H * g.W, g.C);
    if (reduced && p.D == 6) {  // all variants launched; the digitisers' flags let exactly one run
        a.vflag = wide;  // weights need more than 3 planes?
        a.vexpect = 0;
        if (dy_wide) {
            a.vflag2 = dy_wide;  // dy needs more than 3 planes?
            a.vexpect2 = 0;
            const bool narrow_word = a.splits == 1 && a.kb_per_split * kIKB < (int64_t(1) << 17);
            if (dispatch_dgrad_33<CodeT>(p.D, narrow_word, tA3, tB3, a, out, st) != cudaSuccess) return 4;
            a.vexpect2 = 1;
        }
        if (dispatch_dgrad_reduced<CodeT>(p.D, tA, tB3, a, out, st) != cudaSuccess) return 4;
        a.vflag2 = nullptr;
        a.vexpect = 1;
    } else if (reduced && dy_wide) {  // posit(16,1) class: 4 x 4 digits or the full kernel
        a.vflag = wide;
        a.vflag2 = dy_wide;
        a.vexpect = a.vexpect2 = 0;
        if constexpr (sizeof(CodeT) == 2)
            if (launch_kernel<8, CodeT, 1, 4, 0, 4, 4>(tA3, tB3, a, out, st) != cudaSuccess) return 4;
        a.vor = 1;
        a.vexpect = 1;
    }
    if (dispatch<CodeT, 1>(p.D, tA, tB, a, out, st) != cudaSuccess) return 4;
    if (use_partial)
        launch_finalize<CodeT>(a.partial, int(a.splits), nullptr, nullptr, out, a.M, a.N, f, nullptr, nullptr, st);
    const uint32_t nar = 1u << (f.nbits - 1);
    launch_pdl(dgrad_nar_fixup_kernel<CodeT>, dim3(grid_fixup(a.M)), dim3(256), 0, st, 
        dx, a_pos, a_any, g.N, int(g.C), int(g.H), int(g.W), int(g.OH), int(g.OW), int(g.KH),
        int(g.KW), g.pad, nar);
    launch_pdl(dgrad_weight_nar_kernel<CodeT>, dim3(grid_fixup(a.M * a.N)), dim3(256), 0, st, dx, w, g, flags + 1,
                                                                             nar);
    return rc_of(cudaGetLastError());
}

// Weight gradient in the plan's format f.  x: codes of format fx (digitised
// here, converting through the LUT) unless sv holds the forward pass's saved
// digits (p.DA planes at group offset p.OFF).  dy: codes of format fdy;
// share_pos_nar != null also records dy's pixel NaR map for an input-gradient
// pass that reuses these dy digits.
template <typename CodeT>
int run_wgrad(const ImplPlan& p, const ConvGeom& g, const void* dy, const PositFmt& fdy,
              const void* x, const PositFmt& fx, CodeT* dw, unsigned __int128* raw_words,
              uint8_t* raw_nar, uint8_t* ws, cudaStream_t st, const SavedX* sv = nullptr,
              uint8_t* share_pos_nar = nullptr, const DigitGate& gt = DigitGate{},
              uint8_t* dy_wide = nullptr, bool share_gated = true) {
    const PositFmt& f = p.a.f;
    auto* adig = sv ? sv->dig : reinterpret_cast<int8_t*>(ws + p.off_adig);
    auto* bdig = reinterpret_cast<int8_t*>(ws + p.off_bdig);
    uint8_t* chw_nar = sv ? sv->chw : ws + p.off_chw_nar;
    uint8_t* col_nar = ws + p.off_col_nar;
    uint8_t* flags = ws + p.off_flags;
    uint8_t* xflag = sv ? sv->flag : flags;
    if (cudaMemsetAsync(ws + p.off_maps, 0, p.maps_bytes, st) != cudaSuccess) return 4;
    const ConvGeom& gv = p.gv;  // virtual 1x1 geometry when the first layer is folded
    cudaError_t e = cudaSuccess;
    if (sv == nullptr) {
        if (p.fold)
            e = im2col_digits(p.D, x, g, f, fx, lut_of(p, ws, fx), adig, nullptr, chw_nar, flags, st);
        else
            e = act_digits(p.D, x, g.N, g.C, g.H, g.W, p.Ca, g.pad, f, fx, lut_of(p, ws, fx), true, adig,
                           nullptr, chw_nar, nullptr, flags, st);
        if (e != cudaSuccess) return 4;
    }
    // reduced-digit variant: saved (8,1)-format x one digit up, both operands in 3 planes
    // ((8,1) saved digits one digit up, or same-format (12,1) saved digits)
    const bool reduced = sv != nullptr && sizeof(CodeT) == 2 &&
                         ((p.D == 6 && ((p.DA == 4 && p.OFF == 1) || (p.DA == 6 && p.OFF == 0))) ||
                          (p.D == 8 && p.DA == 8 && p.OFF == 0)) &&
                         variant_worthy(p.a);
    const int RP = red_planes(p.D);
    if (reduced && dy_wide == nullptr) dy_wide = flags + 3;
    // dy's high digit planes only when used: every consumer (this pass, and the
    // input gradient sharing the digits) is a flag-selected variant
    const bool reduce_dy = reduced && (share_pos_nar == nullptr || share_gated);
    // (the full weight-gradient variant also runs when x alone is wide: complete dy then too)
    if (act_digits(p.D, dy, g.N, g.F, g.OH, g.OW, p.Fpw, 0, f, fdy, lut_of(p, ws, fdy, 1), true, bdig,
                   share_pos_nar, nullptr, col_nar, flags + 1, st, gt, dy_wide, RP, reduce_dy,
                   reduced ? sv->flag + 1 : nullptr) != cudaSuccess)
        return 4;
    CUtensorMap tA, tB, tA3, tB3;
    const uint32_t boxB[5] = {uint32_t(2 * p.a.OWb), uint32_t(p.a.OHb), 1, uint32_t(p.NT / 16),
                              uint32_t(p.D)};
    uint32_t boxA3[5], boxB3[5];
    for (int i = 0; i < 5; ++i) {
        boxA3[i] = p.boxA[i];
        boxB3[i] = boxB[i];
    }
    boxA3[4] = boxB3[4] = RP;
    if (!map_wgrad_x(&tA, adig, p.DA, gv.N, p.Ha, p.Wa, p.Ca, p.boxA) ||
        !map_act(&tB, bdig, p.D, g.N, g.OH, g.OW, p.Fpw, boxB) ||
        (reduced && (!map_wgrad_x(&tA3, adig, p.DA, gv.N, p.Ha, p.Wa, p.Ca, boxA3) ||
                     !map_act(&tB3, bdig, p.D, g.N, g.OH, g.OW, p.Fpw, boxB3))))
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
    if (reduced) {  // both launched; the x / dy plane flags let exactly one run
        a.vflag = sv->flag + 1;
        a.vflag2 = dy_wide;
        a.vexpect = a.vexpect2 = 0;
        if constexpr (sizeof(CodeT) == 2) {
            cudaError_t er;
            // 64 output channels or more: the 3-digit variant on 64-column tiles (5 groups x
            // 64 = 320 TMEM columns, one CTA per SM) reads each A box once per 64 channels
            // instead of once per 32 -- the pass is L2 -> shared-memory traffic bound.
            // Same splits and partial layout, so the finalize pass does not care which ran.
            if (p.D == 6 && p.Fpw % 64 == 0 && p.NT == 32 && wgrad_nt64()) {
                IgemmArgs a2 = a;
                a2.ntiles = p.Fpw / 64;
                a2.fd_split = FastDiv(uint32_t(a2.mtiles * a2.ntiles));
                a2.fd_group = FastDiv(uint32_t(kGroupM * a2.ntiles));
                CUtensorMap tB64;
                uint32_t boxB64[5];
                for (int i = 0; i < 5; ++i) boxB64[i] = boxB3[i];
                boxB64[3] = 4;  // 64 channels = 4 slices
                if (!map_act(&tB64, bdig, p.D, g.N, g.OH, g.OW, p.Fpw, boxB64)) return 5;
                er = p.OFF == 1
                         ? launch_kernel_geo<6, CodeT, 2, kDgradDB, 1, kDgradDB, 4, 64, 1, 1>(tA3, tB64, a2, out, st)
                         : launch_kernel_geo<6, CodeT, 2, kDgradDB, 0, kDgradDB, 4, 64, 1, 1>(tA3, tB64, a2, out, st);
            } else {
                er = p.D == 8 ? launch_kernel<8, CodeT, 2, 4, 0, 4, 4>(tA3, tB3, a, out, st)
                     : p.OFF == 1 ? launch_kernel<6, CodeT, 2, kDgradDB, 1, kDgradDB, 4>(tA3, tB3, a, out, st)
                                  : launch_kernel<6, CodeT, 2, kDgradDB, 0, kDgradDB, 4>(tA3, tB3, a, out, st);
            }
            if (er != cudaSuccess) return 4;
        }
        a.vor = 1;
        a.vexpect = 1;
    }
    if (dispatch_wgrad<CodeT>(p.D, p.DA, p.OFF, tA, tB, a, out, st) != cudaSuccess) return 4;
    if (use_partial)
        launch_finalize<CodeT>(a.partial, int(a.splits), nullptr, col_nar, out, a.M, a.N, f, raw_words, raw_nar, st);
    launch_pdl(wgrad_nar_fixup_kernel<CodeT>, dim3(grid_for(p.ckk, 128)), dim3(128), 0, st, 
        dw, raw_nar, chw_nar, xflag, int(g.F), p.fold ? p.ckk : int(g.C), int(gv.H), int(gv.W),
        int(g.OH), int(g.OW), int(gv.KH), int(gv.KW), gv.pad, 1u << (f.nbits - 1));
    return rc_of(cudaGetLastError());
}

// A saved forward digit tensor of format ff usable as the weight gradient's A
// operand in format fg: same format, or an exact widening (same es, more bits)
// by a whole number of digits with a kernel variant.  *DA / *OFF on success.
bool saved_usable(const PositFmt& ff, const PositFmt& fg, int* DA, int* OFF) {
    const int DF = digits_for(ff), DG = digits_for(fg);
    if (same_fmt(ff, fg)) {
        *DA = DG;
        *OFF = 0;
        return true;
    }
    if (ff.es != fg.es || fg.nbits <= ff.nbits) return false;
    const int shift = fg.R - ff.R;  // X_g = X_f * 2^shift exactly
    if (shift % 8) return false;
    if (!wgrad_variant(DG, DF, shift / 8)) return false;
    *DA = DF;
    *OFF = shift / 8;
    return true;
}

// Plans of the fused backward: weight gradient (format fg, A from the saved
// digits when usable) and, when wanted, the input gradient (format fb).
struct BwdPlan {
    ImplPlan pw, pd;
    bool has_dx, use_saved, share_dy;
    size_t off_d, total;
};

bool make_bwd_plan(const PositFmt& ff, const PositFmt& fb, const PositFmt& fg, const ConvGeom& g,
                   bool raw, bool has_dx, bool saved, BwdPlan* b) {
    *b = BwdPlan{};
    int DA = 0, OFF = 0;
    b->use_saved = saved && saved_usable(ff, fg, &DA, &OFF);
    if (!make_plan(2, fg, g, raw, &b->pw, b->use_saved ? DA : 0, b->use_saved ? OFF : 0, b->use_saved))
        return false;
    // x / dy codes of another format are digitised through a conversion LUT
    if (!b->use_saved && !same_fmt(ff, fg) && ff.nbits > kActLutBits) return false;
    if (!same_fmt(fb, fg) && fb.nbits > kActLutBits) return false;
    b->has_dx = has_dx;
    if (has_dx && !make_plan(1, fb, g, false, &b->pd)) return false;
    // dy digits shared when both passes see the same digits in the same layout
    b->share_dy = has_dx && same_fmt(fb, fg) && b->pw.Fpw == g.F && b->pd.Ca == g.F;
    b->off_d = (b->pw.total + 255) & ~size_t(255);
    b->total = b->off_d + (has_dx ? b->pd.total : 0);
    return true;
}

template <typename GT, typename BT>
int run_backward(const BwdPlan& b, const ConvGeom& g, const PositFmt& ff, const PositFmt& fb,
                 const void* dy, const void* x, const SavedX* sv, const void* w_bwd, void* dx, void* dw,
                 unsigned __int128* raw_words, uint8_t* raw_nar, uint8_t* ws, cudaStream_t st,
                 const DigitGate& gt) {
    uint8_t* wsd = ws + b.off_d;
    if (b.share_dy && cudaMemsetAsync(wsd + b.pd.off_maps, 0, b.pd.maps_bytes, st) != cudaSuccess) return 4;
    uint8_t* dy_wide = b.share_dy ? wsd + b.pd.off_flags + 3 : nullptr;  // cleared with the dgrad maps
    const bool dgrad_gated = dgrad_reduced(b.pd.D) && sizeof(BT) == 2 && variant_worthy(b.pd.a);
    int rc = run_wgrad<GT>(b.pw, g, dy, fb, x, ff, static_cast<GT*>(dw), raw_words, raw_nar, ws, st,
                           b.use_saved ? sv : nullptr,
                           b.share_dy ? wsd + b.pd.off_pos_nar : nullptr, gt, dy_wide, dgrad_gated);
    if (rc != 0 || !b.has_dx) return rc;
    const DigitGate gd = gt;  // the input gradient digitises dy itself unless it shares the digits
    if (b.share_dy) {
        const DyDigits pre{reinterpret_cast<const int8_t*>(ws + b.pw.off_bdig), wsd + b.pd.off_pos_nar,
                           ws + b.pw.off_flags + 1, dy_wide};
        return run_dgrad<BT>(b.pd, g, static_cast<const BT*>(dy), static_cast<const BT*>(w_bwd),
                             static_cast<BT*>(dx), wsd, st, &pre, gd);
    }
    return run_dgrad<BT>(b.pd, g, static_cast<const BT*>(dy), static_cast<const BT*>(w_bwd),
                         static_cast<BT*>(dx), wsd, st, nullptr, gd);
}

}  // namespace

bool igemm_eligible(int pass, const PositFmt& f, const ConvGeom& g, bool raw, size_t* bytes) {
    ImplPlan p;
    if (!make_plan(pass, f, g, raw, &p)) return false;
    if (bytes) *bytes = p.total;
    return true;
}

int igemm_conv_fwd(const PositFmt& f, const ConvGeom& g, const void* x, const void* w,
                   const void* bias, void* y, void* ws, size_t ws_bytes, cudaStream_t st,
                   void* saved, size_t saved_bytes, int relu, void* pre) {
    ImplPlan p;
    if (!make_plan(0, f, g, false, &p)) return 2;
    if (ws_bytes < p.total) return 3;
    SaveLayout L{};
    SavedX sv{};
    if (saved != nullptr) {
        if (!save_layout(f, g, &L)) return 2;
        if (saved_bytes < L.total) return 3;
        sv = saved_of(saved, L);
    }
    auto* b = static_cast<uint8_t*>(ws);
    const SavedX* svp = saved ? &sv : nullptr;
    const size_t clear = L.chw + 16;  // NaR map + flag
    if (f.nbits <= 8)
        return run_fwd<uint8_t>(p, g, (const uint8_t*)x, (const uint8_t*)w, (const uint8_t*)bias,
                                (uint8_t*)y, b, st, svp, clear, relu, (uint8_t*)pre);
    return run_fwd<uint16_t>(p, g, (const uint16_t*)x, (const uint16_t*)w, (const uint16_t*)bias,
                             (uint16_t*)y, b, st, svp, clear, relu, (uint16_t*)pre);
}

size_t igemm_saved_bytes(const PositFmt& f, const ConvGeom& g) {
    SaveLayout L;
    return save_layout(f, g, &L) ? L.total : 0;
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
        return run_wgrad<uint8_t>(p, g, dy, f, x, f, (uint8_t*)dw, raw_words, raw_nar, b, st);
    return run_wgrad<uint16_t>(p, g, dy, f, x, f, (uint16_t*)dw, raw_words, raw_nar, b, st);
}

bool igemm_backward_eligible(const PositFmt& ff, const PositFmt& fb, const PositFmt& fg,
                             const ConvGeom& g, bool raw, bool has_dx, bool saved, size_t* bytes) {
    BwdPlan b;
    if (!make_bwd_plan(ff, fb, fg, g, raw, has_dx, saved, &b)) return false;
    if (bytes) *bytes = b.total;
    return true;
}

int igemm_conv_backward(const PositFmt& ff, const PositFmt& fb, const PositFmt& fg, const ConvGeom& g,
                        const void* dy, const void* x, const void* saved, size_t saved_bytes,
                        const void* w_bwd, void* dx, void* dw, unsigned __int128* raw_words,
                        uint8_t* raw_nar, void* ws, size_t ws_bytes, cudaStream_t st,
                        const void* gate, int gate_nbits, void* dy_gated) {
    BwdPlan b;
    if (!make_bwd_plan(ff, fb, fg, g, raw_words != nullptr, dx != nullptr, saved != nullptr, &b)) return 2;
    if (ws_bytes < b.total) return 3;
    if (!b.use_saved && x == nullptr) return 2;  // saved digits unusable for this format pair
    SavedX sv{};
    if (b.use_saved) {
        SaveLayout L;
        if (!save_layout(ff, g, &L)) return 2;
        if (saved_bytes < L.total) return 3;
        sv = saved_of(const_cast<void*>(saved), L);
    }
    auto* w = static_cast<uint8_t*>(ws);
    DigitGate gt{};
    if (gate != nullptr) {
        gt.gate = gate;
        gt.gb = gate_nbits <= 8 ? 1 : 2;
        gt.gnbits = gate_nbits;
    }
    if (dy_gated != nullptr) {  // the ReLU's input gradient itself (recording / the bias gradient)
        const int64_t total = g.N * g.F * g.OH * g.OW;
        if (fb.nbits <= 8)
            launch_pdl(gate_codes_kernel<uint8_t>, dim3(grid_for(total, 256)), dim3(256), 0, st, 
                static_cast<const uint8_t*>(dy), gt, static_cast<uint8_t*>(dy_gated), total);
        else
            launch_pdl(gate_codes_kernel<uint16_t>, dim3(grid_for(total, 256)), dim3(256), 0, st, 
                static_cast<const uint16_t*>(dy), gt, static_cast<uint16_t*>(dy_gated), total);
    }
    const bool g8 = fg.nbits <= 8, b8 = fb.nbits <= 8;
    if (g8 && b8)
        return run_backward<uint8_t, uint8_t>(b, g, ff, fb, dy, x, &sv, w_bwd, dx, dw, raw_words, raw_nar, w, st, gt);
    if (g8)
        return run_backward<uint8_t, uint16_t>(b, g, ff, fb, dy, x, &sv, w_bwd, dx, dw, raw_words, raw_nar, w, st, gt);
    if (b8)
        return run_backward<uint16_t, uint8_t>(b, g, ff, fb, dy, x, &sv, w_bwd, dx, dw, raw_words, raw_nar, w, st, gt);
    return run_backward<uint16_t, uint16_t>(b, g, ff, fb, dy, x, &sv, w_bwd, dx, dw, raw_words, raw_nar, w, st, gt);
}

}  // namespace pnn_b200

extern "C" int64_t pnn_variant_min_work(int64_t macs) {
    return macs < 0 ? pnn_b200::variant_min_work() : pnn_b200::set_variant_min_work(macs);
}

extern "C" int pnn_conv_algo(int algo) {
    if (algo < 0 || algo > 2) return -1;
    return pnn_b200::set_conv_algo(algo);
}
