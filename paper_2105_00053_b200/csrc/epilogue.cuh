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

__device__ __forceinline__ uint32_t q_to_posit_lut(const PositFmt& f, uint64_t q, const uint4* lut) {
    const int64_t v = f.W < 64 ? int64_t(q << (64 - f.W)) >> (64 - f.W) : int64_t(q);
    const uint64_t s = uint64_t(v >> 63);
    const uint64_t mag = (uint64_t(v) ^ s) - s;
    const int lz = __clzll(mag);
    const uint64_t sig = mag << (lz & 63);
    const uint32_t c = pack_lut(f, lut, 63 - lz - 2 * f.R, uint32_t(sig >> 32), uint32_t(sig) != 0,
                                s != 0);
    return mag == 0 ? 0u : c;
}

__device__ __forceinline__ uint32_t q_to_posit_lut(const PositFmt& f, unsigned __int128 q,
                                                   const uint4* lut) {
    uint64_t lo = uint64_t(q), hi = uint64_t(q >> 64);
    if (f.W < 128) hi = uint64_t(int64_t(hi << (128 - f.W)) >> (128 - f.W));  // W > 64
    const uint64_t s = uint64_t(int64_t(hi) >> 63);
    const unsigned __int128 S = ((unsigned __int128)s << 64) | s;
    const unsigned __int128 m = ((((unsigned __int128)hi << 64) | lo) ^ S) - S;
    lo = uint64_t(m);
    hi = uint64_t(m >> 64);
    const bool hz = hi == 0;
    const int lzh = __clzll(hi), lzl = __clzll(lo);
    const uint64_t sig_h = (hi << (lzh & 63)) | ((lo >> 1) >> ((63 - lzh) & 63));
    const bool st_h = (lo << (lzh & 63)) != 0;
    const uint64_t sig = hz ? (lo << (lzl & 63)) : sig_h;
    const bool sticky = (!hz && st_h) || uint32_t(sig) != 0;
    const int top = hz ? 63 - lzl : 127 - lzh;
    const uint32_t c = pack_lut(f, lut, top - 2 * f.R, uint32_t(sig >> 32), sticky, s != 0);
    return (hz && lo == 0) ? 0u : c;
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
