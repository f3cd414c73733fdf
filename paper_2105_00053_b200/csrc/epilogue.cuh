// Register-lean quire epilogue pieces for the tcgen05 kernels:
//
//  * QAcc2<QW>: one output's quire word Q = sum_g S_g 256^g (mod the word)
//    accumulated straight from the int32 TMEM group sums -- one IMAD.WIDE
//    per group into the word position it lands in (<= 3 words live);
//  * a per-CTA rounding table (one entry per posit scale): the regime and
//    exponent bits of pack_round32_bf tabulated, so the per-output rounding
//    is a table load, a shift, and the guard/sticky round -- the same
//    arithmetic as pack_round32_bf (posit.cpp:93-132), entry for entry;
//  * qN_to_posit_lut: W-bit two's-complement quire word (N = 32/64/128-bit
//    container) -> posit code with the table.
#pragma once

#include <cstdint>

#include "posit_device.cuh"

namespace pnn_b200 {

constexpr int kPackLutEntries = 64;  // 2R + 2 <= 58 for every supported format (2R <= 56)

// Entry i: i = 0 saturates to minpos, i = 2R + 1 to maxpos, otherwise scale
// s = i - 1 - R in [-R, R-1]: {regime|exponent bits left-aligned, head =
// regime length + es, (1 << head) - 1, 0}.
__device__ __forceinline__ void build_pack_lut(const PositFmt& f, uint4* lut, int tid, int nthr) {
    const int n = 2 * f.R + 2;
    for (int i = tid; i < n; i += nthr) {
        uint4 v;
        if (i == 0 || i == n - 1) {
            const uint32_t pat = i == 0 ? 1u : (1u << (f.nbits - 1)) - 1u;
            v = make_uint4(pat << (33 - f.nbits), 31u, 0x7FFFFFFFu, 0u);
        } else {
            const int sc = i - 1 - f.R;
            const int k = sc >> f.es;
            const int e = sc - (k << f.es);
            const bool kpos = k >= 0;
            const int rl = kpos ? k + 2 : 1 - k;
            const uint32_t regime = kpos ? (((1u << (k + 1)) - 1u) << 1) : 1u;
            const int head = rl + f.es;
            uint32_t w = regime << (32 - rl);
            if (f.es > 0) w |= uint32_t(e) << (32 - head);
            v = make_uint4(w, uint32_t(head), (1u << head) - 1u, 0u);
        }
        lut[i] = v;
    }
}

// pack_round32_bf through the table: sig32 has its leading one at bit 31.
__device__ __forceinline__ uint32_t pack_lut(const PositFmt& f, const uint4* lut, int scale,
                                             uint32_t sig32, bool sticky, bool neg) {
    int idx = scale + f.R + 1;
    idx = idx < 0 ? 0 : (idx > 2 * f.R + 1 ? 2 * f.R + 1 : idx);
    const uint4 e = lut[idx];
    const uint32_t frac = sig32 << 1;
    const uint32_t w = e.x | (frac >> e.y);
    const uint32_t lowm = (1u << (32 - f.nbits)) - 1u;
    const bool st = sticky || ((frac & e.z) | (w & lowm)) != 0;
    uint32_t pat = w >> (33 - f.nbits);
    const uint32_t guard = (w >> (32 - f.nbits)) & 1u;
    pat += guard & (uint32_t(st) | (pat & 1u));
    const uint32_t mask = (1u << f.nbits) - 1u;
    return neg ? ((0u - pat) & mask) : pat;
}

__device__ __forceinline__ uint32_t q_to_posit_lut(const PositFmt& f, uint32_t q, const uint4* lut) {
    const int32_t v = f.W < 32 ? int32_t(q << (32 - f.W)) >> (32 - f.W) : int32_t(q);
    const uint32_t s = uint32_t(v >> 31);
    const uint32_t mag = (uint32_t(v) ^ s) - s;
    const int lz = __clz(mag);
    const uint32_t c = pack_lut(f, lut, 31 - lz - 2 * f.R, mag << (lz & 31), false, s != 0);
    return mag == 0 ? 0u : c;
}

// 64-bit word as two 32-bit halves (the SM has no 64-bit integer ALU): sign
// extension from W bits touches the high half only, |q| by xor + add-carry,
// the leading one by two FLOs, the top 32 bits by one funnel shift.
__device__ __forceinline__ uint32_t q_to_posit_lut(const PositFmt& f, uint64_t q, const uint4* lut) {
    uint32_t lo = uint32_t(q);
    int32_t hi = int32_t(q >> 32);
    if (f.W <= 32) {  // the whole word lives in the low half (no shift by >= 32)
        lo = uint32_t(int32_t(lo << (32 - f.W)) >> (32 - f.W));
        hi = int32_t(lo) >> 31;
    } else if (f.W < 64) {
        hi = (hi << (64 - f.W)) >> (64 - f.W);
    }
    const uint32_t s = uint32_t(hi >> 31);  // 0 or ~0
    uint32_t ml = lo ^ s, mh = uint32_t(hi) ^ s;
    asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(ml), "+r"(mh) : "r"(s & 1u));
    const bool hz = mh == 0;
    const int lzh = __clz(mh), lzl = __clz(ml);
    const uint32_t sig = hz ? (ml << (lzl & 31)) : __funnelshift_l(ml, mh, lzh);
    const bool sticky = !hz && (ml << (lzh & 31)) != 0;  // lzh < 32 when mh != 0
    const int top = hz ? 31 - lzl : 63 - lzh;
    const uint32_t c = pack_lut(f, lut, top - 2 * f.R, sig, sticky, s != 0);
    return (ml | mh) == 0 ? 0u : c;
}

// The same rounding of a 64-bit word (W <= 64) with the leading-one search and
// the normalisation done by the FP64 converter: I2F.F64 (toward zero) of the
// W-bit value gives |q|'s exponent and its top 53 bits; the bits it drops
// (|q| >= 2^53) are detected by converting back (exact for an integral double)
// and OR-ed into the sticky bit.  Same pack_lut call, same result
// (tests/test_epilogue_gpu.py compares both on edge and random words).
__device__ __forceinline__ uint32_t q_to_posit_lut_f64(const PositFmt& f, uint64_t q, const uint4* lut) {
    int64_t v = int64_t(q);
    if (f.W < 64) v = (v << (64 - f.W)) >> (64 - f.W);
    const double d = __ll2double_rz(v);
    const bool lost = __double2ll_rz(d) != v;
    const uint32_t hi = uint32_t(__double2hiint(d)), lo = uint32_t(__double2loint(d));
    const int top = int((hi >> 20) & 0x7FFu) - 1023;
    const uint32_t sig = 0x80000000u | ((hi & 0xFFFFFu) << 11) | (lo >> 21);
    const bool sticky = (lo & 0x1FFFFFu) != 0 || lost;
    const uint32_t c = pack_lut(f, lut, top - 2 * f.R, sig, sticky, (hi >> 31) != 0);
    return v == 0 ? 0u : c;
}

// The same conversion with what the caller knows folded in:
//  * kNoWrap: q already is the exact value (the pass's |sum| bound is below
//    2^(W-1)), so no sign extension from W bits;
//  * kRelu: the caller stores relu(code) only: negative values and zero give 0,
//    so the rounding runs on the magnitude path alone (the sign of a nonzero
//    converted integer is the sign of the double's high word; zero has hi == 0);
//  * a value of 2^53 or more saturates to +-maxpos whenever 3R <= 52 (maxpos =
//    2^R is 2^(3R) quire units), so the dropped-bit check is skipped there.
// Same codes as q_to_posit_lut_f64 (tests/test_epilogue_gpu.py, conv tests).
template <bool kRelu, bool kNoWrap>
__device__ __forceinline__ uint32_t q_to_posit_lut_f64x(const PositFmt& f, uint64_t q, const uint4* lut) {
    int64_t v = int64_t(q);
    if (!kNoWrap && f.W < 64) v = (v << (64 - f.W)) >> (64 - f.W);
    const double d = __ll2double_rz(v);
    const uint32_t hi = uint32_t(__double2hiint(d)), lo = uint32_t(__double2loint(d));
    const bool lost = 3 * f.R > 52 && __double2ll_rz(d) != v;
    const int top = int((hi >> 20) & 0x7FFu) - 1023;
    const uint32_t sig = 0x80000000u | ((hi & 0xFFFFFu) << 11) | (lo >> 21);
    const bool sticky = (lo & 0x1FFFFFu) != 0 || lost;
    if constexpr (kRelu) {
        const uint32_t c = pack_lut(f, lut, top - 2 * f.R, sig, sticky, false);
        return int32_t(hi) > 0 ? c : 0u;
    } else {
        const uint32_t c = pack_lut(f, lut, top - 2 * f.R, sig, sticky, (hi >> 31) != 0);
        return hi == 0 ? 0u : c;
    }
}

// 8-bit output formats: the whole of pack_lut tabulated.  pack_lut's result
// depends on the significand only through its top FB = 6 - es fraction bits
// (the bits that can reach the pattern or the guard position: head >= 2 + es)
// and on whether anything below them is set, so
//     code = tab[((scale index) * 2^FB + top FB fraction bits) * 2 + (rest != 0)]
// with every entry computed by pack_lut itself (build_pack_tab8, after
// build_pack_lut and a barrier).  (scale index, top bits) is one field of the
// double's high word: (hi >> (20 - FB)) minus a constant, clamped -- the rows at
// both ends are the constant minpos / maxpos saturations.
// (2R + 2) * 2^FB * 2 = (12 * 2^es + 2) * 2^(7 - es) <= 1792 entries for nbits <= 8
constexpr int kTab8Bytes = 2048;
__device__ __forceinline__ void build_pack_tab8(const PositFmt& f, const uint4* lut, uint8_t* tab, int tid,
                                                int nthr) {
    const int FB = 6 - f.es, rows = 2 * f.R + 2;
    for (int i = tid; i < (rows << FB) * 2; i += nthr) {
        const int st = i & 1, m = (i >> 1) & ((1 << FB) - 1), row = i >> (FB + 1);
        const uint32_t sig = 0x80000000u | (uint32_t(m) << (31 - FB));
        tab[i] = uint8_t(pack_lut(f, lut, row - 1 - f.R, sig, st != 0, false));
    }
}

// 64-bit quire word -> 8-bit posit code through the FP64 converter and the
// table (same codes as q_to_posit_lut_f64; flags as q_to_posit_lut_f64x).
template <bool kRelu, bool kNoWrap>
__device__ __forceinline__ uint32_t q_to_posit_tab8(const PositFmt& f, uint64_t q, const uint8_t* tab) {
    int64_t v = int64_t(q);
    if (!kNoWrap && f.W < 64) v = (v << (64 - f.W)) >> (64 - f.W);
    const double d = __ll2double_rz(v);
    const uint32_t hi = uint32_t(__double2hiint(d)), lo = uint32_t(__double2loint(d));
    const int FB = 6 - f.es;
    const bool lost = 3 * f.R > 52 && __double2ll_rz(d) != v;
    const uint32_t mag = kRelu ? hi : (hi & 0x7FFFFFFFu);  // (relu: negative values are discarded)
    // row = top - 2R + R + 1 with top = exponent - 1023
    int idx = int(mag >> (20 - FB)) - ((1023 + f.R - 1) << FB);
    const int last = ((2 * f.R + 2) << FB) - 1;
    idx = idx < 0 ? 0 : (idx > last ? last : idx);
    const uint32_t rest = (hi & ((1u << (20 - FB)) - 1u)) | lo | uint32_t(lost);
    const uint32_t c = tab[2 * idx + int(rest != 0)];
    if constexpr (kRelu) return int32_t(hi) > 0 ? c : 0u;
    else return hi == 0 ? 0u : ((hi >> 31) ? ((0u - c) & ((1u << f.nbits) - 1u)) : c);
}

// 32-bit quire word (W <= 32) -> 8-bit posit code: the same table through the
// FP32 converter (24-bit significand, toward zero; a value of 2^24 or more
// saturates whenever 3R <= 23, otherwise the dropped bits join the rest bit).
template <bool kRelu>
__device__ __forceinline__ uint32_t q32_to_posit_tab8(const PositFmt& f, uint32_t q, const uint8_t* tab) {
    const int32_t v = f.W < 32 ? int32_t(q << (32 - f.W)) >> (32 - f.W) : int32_t(q);
    const float fl = __int2float_rz(v);
    const uint32_t bits = __float_as_uint(fl);
    const int FB = 6 - f.es;
    const bool lost = 3 * f.R > 23 && __float2int_rz(fl) != v;
    const uint32_t mag = kRelu ? bits : (bits & 0x7FFFFFFFu);
    int idx = int(mag >> (23 - FB)) - ((127 + f.R - 1) << FB);
    const int last = ((2 * f.R + 2) << FB) - 1;
    idx = idx < 0 ? 0 : (idx > last ? last : idx);
    const uint32_t rest = (bits & ((1u << (23 - FB)) - 1u)) | uint32_t(lost);
    const uint32_t c = tab[2 * idx + int(rest != 0)];
    if constexpr (kRelu) return int32_t(bits) > 0 ? c : 0u;
    else return bits == 0 ? 0u : ((bits >> 31) ? ((0u - c) & ((1u << f.nbits) - 1u)) : c);
}

// 128-bit word as four 32-bit limbs (sign extension from W bits, |q| by xor +
// carry chain, leading limb selected, top 32 bits by one funnel shift).
__device__ __forceinline__ uint32_t q_to_posit_lut(const PositFmt& f, unsigned __int128 q,
                                                   const uint4* lut) {
    uint32_t w0 = uint32_t(q), w1 = uint32_t(uint64_t(q) >> 32);
    const uint64_t qh = uint64_t(q >> 64);
    uint32_t w2 = uint32_t(qh);
    int32_t w3 = int32_t(qh >> 32);
    if (f.W <= 96) {  // 64 < W <= 96: the sign lives in w2
        w2 = uint32_t(int32_t(w2 << (96 - f.W)) >> (96 - f.W));
        w3 = int32_t(w2) >> 31;
    } else if (f.W < 128) {
        w3 = (w3 << (128 - f.W)) >> (128 - f.W);
    }
    const uint32_t s = uint32_t(w3 >> 31);
    uint32_t m0 = w0 ^ s, m1 = w1 ^ s, m2 = w2 ^ s, m3 = uint32_t(w3) ^ s;
    asm("add.cc.u32 %0, %0, %4;\n\taddc.cc.u32 %1, %1, 0;\n\taddc.cc.u32 %2, %2, 0;\n\taddc.u32 %3, %3, 0;"
        : "+r"(m0), "+r"(m1), "+r"(m2), "+r"(m3)
        : "r"(s & 1u));
    // |q| <= 2^(W-1): for W <= 96 the top limb is zero (compile-time for the
    // specialised formats).  Leading limb by selects, not branches (the lanes of
    // a warp disagree on it): (hi, lo, below) = the limb holding the leading
    // one, the next limb, the OR of the rest.
    const bool n3 = f.W > 96 && m3 != 0, n2 = m2 != 0, n1 = m1 != 0;
    const uint32_t hi = n3 ? m3 : n2 ? m2 : n1 ? m1 : m0;
    const uint32_t lo = n3 ? m2 : n2 ? m1 : n1 ? m0 : 0u;
    const uint32_t below = n3 ? (m1 | m0) : n2 ? m0 : 0u;
    const int base = n3 ? 127 : n2 ? 95 : n1 ? 63 : 31;
    const int lz = __clz(hi);
    const uint32_t sig = __funnelshift_l(lo, hi, lz);
    const bool sticky = (lo << (lz & 31)) != 0 || below != 0;  // lz < 32 unless q == 0
    const uint32_t c = pack_lut(f, lut, base - lz - 2 * f.R, sig, sticky, s != 0);
    return hi == 0 ? 0u : c;
}

// Quire word of one output, accumulated group by group (mod the word size;
// the quire is only defined mod 2^W <= word bits).
template <int QW>
struct QAcc2;
template <>
struct QAcc2<1> {  // W <= 32
    uint32_t q = 0;
    __device__ __forceinline__ void add(int g, uint32_t s) {
        if (8 * g < 32) q += s << (8 * g);
    }
    __device__ __forceinline__ uint32_t get() const { return q; }
};
template <>
struct QAcc2<2> {  // W <= 64: groups 0-3 by IMAD.WIDE, 4-7 into the high word only
    int64_t q = 0;
    uint32_t hi = 0;
    __device__ __forceinline__ void add(int g, uint32_t s) {
        if (g < 4) q += int64_t(int32_t(s)) * int64_t(1u << (8 * g));
        else if (g < 8) hi += s << (8 * g - 32);
    }
    __device__ __forceinline__ uint64_t get() const { return uint64_t(q) + (uint64_t(hi) << 32); }
};
template <>
struct QAcc2<4> {  // W <= 128: three overlapping 64-bit words at bit 0, 32, 64
    int64_t w0 = 0, w1 = 0;
    uint64_t w2 = 0;
    __device__ __forceinline__ void add(int g, uint32_t s) {
        const int64_t x = int64_t(int32_t(s));
        if (g < 4) w0 += x * int64_t(1u << (8 * g));
        else if (g < 8) w1 += x * int64_t(1u << (8 * g - 32));
        else if (g < 16) w2 += uint64_t(x) << (8 * g - 64);
    }
    __device__ __forceinline__ unsigned __int128 get() const {
        const unsigned __int128 a = (unsigned __int128)(__int128)w0;
        const unsigned __int128 b = (unsigned __int128)(__int128)w1 << 32;
        return a + b + ((unsigned __int128)w2 << 64);
    }
};

}  // namespace pnn_b200
