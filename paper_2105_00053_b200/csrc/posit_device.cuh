// Device posit core: decode to the exact integer image, balanced int8 digit
// split, and quire -> posit rounding.  sm_100a only.
//
// Reference semantics:
//   decode        : detail::unpack            proj/src/posit.cpp:67-91
//                   DecodeTables::Fixed        proj/src/posit_tables.cpp:43-64
//   pack_round    : detail::pack_round         proj/src/posit.cpp:93-132
//   quire readout : Quire::to_posit            proj/src/quire.cpp:105-146
//
// Integer image.  For format (n, es) with R = (n-2)<<es every posit x is
// x = X * 2^-R with X an exact integer, |X| <= 2^(2R).  The reference quire
// (W = 4R + n bits, LSB weight 2^-2R, quire.hpp:20-30) after accumulating
// products holds exactly  sum(X_a * X_b) mod 2^W.  Everything below works on X.
#pragma once

#include <cstdint>

namespace pnn_b200 {

struct PositFmt {
    int nbits;
    int es;
    int R;  // max_scale
    int W;  // quire bits
};

__host__ __device__ inline PositFmt make_fmt(int nbits, int es) {
    PositFmt f;
    f.nbits = nbits;
    f.es = es;
    f.R = (nbits - 2) << es;
    f.W = 4 * f.R + nbits;
    return f;
}

// Compile-time formats of the BASELINE configs, for kernel specialisations
// whose epilogues then constant-fold every mask and shift; 0 = the runtime
// format argument.
template <int FMT>
__device__ __forceinline__ PositFmt fixed_fmt(const PositFmt& rt) {
    if constexpr (FMT == 1) return PositFmt{8, 0, 6, 32};
    else if constexpr (FMT == 2) return PositFmt{8, 1, 12, 56};
    else if constexpr (FMT == 3) return PositFmt{12, 1, 20, 92};
    else if constexpr (FMT == 4) return PositFmt{16, 1, 28, 128};
    else return rt;
}
inline int fixed_fmt_id(const PositFmt& f) {
    if (f.es == 0 && f.nbits == 8) return 1;
    if (f.es == 1 && f.nbits == 8) return 2;
    if (f.es == 1 && f.nbits == 12) return 3;
    if (f.es == 1 && f.nbits == 16) return 4;
    return 0;
}

// Decode one code into X (two's complement int64).  Returns true for NaR.
// Valid for 2 <= nbits <= 32 and 2R <= 62 (X fits int64).
__device__ __forceinline__ bool decode_x(uint32_t code, const PositFmt& f, int64_t& X) {
    const uint32_t mask = f.nbits == 32 ? 0xFFFFFFFFu : ((1u << f.nbits) - 1u);
    code &= mask;
    X = 0;
    if (code == 0) return false;
    const uint32_t nar = 1u << (f.nbits - 1);
    if (code == nar) return true;
    const bool neg = (code & nar) != 0;
    const uint32_t mag = neg ? ((0u - code) & mask) : code;
    // payload (nbits-1 bits) left-aligned in 32 bits; low bits are zero
    const uint32_t p = mag << (33 - f.nbits);
    const bool first = (p >> 31) != 0;
    int run = first ? __clz(~p) : __clz(p);
    if (run > f.nbits - 1) run = f.nbits - 1;
    const int k = first ? run - 1 : -run;
    const int used = run + 1;
    int rem = f.nbits - 1 - used;
    if (rem < 0) rem = 0;
    const uint32_t tail = used < 32 ? (p << used) : 0u;
    const int ebits = f.es < rem ? f.es : rem;
    uint32_t e = ebits > 0 ? (tail >> (32 - ebits)) : 0u;
    e <<= (f.es - ebits);
    const int fb = rem - ebits;
    const uint32_t frac = fb > 0 ? ((tail << ebits) >> (32 - fb)) : 0u;
    const int scale = k * (1 << f.es) + int(e);
    const uint64_t sig = (uint64_t(1) << fb) | frac;
    const int pos = scale - fb + f.R;  // >= 0 for every finite posit
    const int64_t mx = int64_t(sig << pos);
    X = neg ? -mx : mx;
    return false;
}

// decode_x without branches (the digitisers' per-code hot path): the same X
// for every code (zero and NaR give X = 0; returns true for NaR).  The regime
// run comes from one FLO of the payload XOR its first bit, the significand is
// kept left-aligned (leading one at bit 31) and placed by one 64-bit right
// shift of S * 2^32 by 63 - R - scale (in [63 - 2R, 63]: pos >= 0 for every
// finite posit, so only zeros are shifted out).  Valid for nbits <= 32, 2R <= 62.
__device__ __forceinline__ bool decode_x_bf(uint32_t code, const PositFmt& f, int64_t& X) {
    const uint32_t narc = 1u << (f.nbits - 1);
    code &= narc | (narc - 1u);
    const uint32_t sgn = 0u - (code >> (f.nbits - 1));      // 0 or ~0
    const uint32_t mag = ((code ^ sgn) - sgn) & (narc - 1u);  // payload; 0 for zero and NaR
    const uint32_t p = mag << (33 - f.nbits);
    const uint32_t inv = uint32_t(int32_t(p) >> 31);          // ~0 when the regime is a run of ones
    const int run = __clz(int(p ^ inv));                      // <= nbits - 1 (32 only when mag == 0)
    const uint32_t tail = (p << (run & 31)) << 1;             // past the regime and its terminator
    const uint32_t e = f.es > 0 ? tail >> (32 - f.es) : 0u;
    const uint32_t S = ((tail << f.es) >> 1) | 0x80000000u;   // 1.fraction, leading one at bit 31
    const int k = (run - 1) ^ int(~inv);                      // run - 1, or -run for a run of zeros
    const int scale = k * (1 << f.es) + int(e);
    uint64_t mx = (uint64_t(S) << 32) >> (63 - f.R - scale);
    mx = mag == 0 ? 0ull : mx;
    const uint64_t s64 = uint64_t(int64_t(int32_t(sgn)));
    X = int64_t((mx ^ s64) - s64);
    return code == narc;
}

// Same, into a 128-bit image: valid for 2R <= 124 (the elementwise formats up
// to posit(12,2), R = 40, used by the posit(8,2)* optimizer and loss stages).
__device__ __forceinline__ bool decode_x128(uint32_t code, const PositFmt& f, __int128& X) {
    const uint32_t mask = f.nbits == 32 ? 0xFFFFFFFFu : ((1u << f.nbits) - 1u);
    code &= mask;
    X = 0;
    if (code == 0) return false;
    const uint32_t nar = 1u << (f.nbits - 1);
    if (code == nar) return true;
    const bool neg = (code & nar) != 0;
    const uint32_t mag = neg ? ((0u - code) & mask) : code;
    const uint32_t p = mag << (33 - f.nbits);
    const bool first = (p >> 31) != 0;
    int run = first ? __clz(~p) : __clz(p);
    if (run > f.nbits - 1) run = f.nbits - 1;
    const int k = first ? run - 1 : -run;
    const int used = run + 1;
    int rem = f.nbits - 1 - used;
    if (rem < 0) rem = 0;
    const uint32_t tail = used < 32 ? (p << used) : 0u;
    const int ebits = f.es < rem ? f.es : rem;
    uint32_t e = ebits > 0 ? (tail >> (32 - ebits)) : 0u;
    e <<= (f.es - ebits);
    const int fb = rem - ebits;
    const uint32_t frac = fb > 0 ? ((tail << ebits) >> (32 - fb)) : 0u;
    const int scale = k * (1 << f.es) + int(e);
    const unsigned __int128 sig = (unsigned __int128)((uint64_t(1) << fb) | frac);
    const __int128 mx = (__int128)(sig << (scale - fb + f.R));
    X = neg ? -mx : mx;
    return false;
}

// Balanced base-256 digits: X = sum_d digit[d] * 256^d, digit in [-128, 127].
template <int D>
__device__ __forceinline__ void balanced_digits(int64_t X, int8_t (&dig)[D]) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
        const int8_t t = int8_t(uint8_t(uint64_t(X) & 0xFF));
        dig[d] = t;
        X = (X - int64_t(t)) >> 8;
    }
}

// detail::pack_round restated with a 64-bit window (nbits <= 32, so regime +
// exponent + guard always fit): round-to-nearest, ties to the even pattern,
// saturate at maxpos, never round to zero.
__device__ __forceinline__ uint32_t pack_round(const PositFmt& f, bool neg, int scale,
                                               uint64_t sig, bool sticky) {
    if (sig == 0) return 0;
    uint32_t pat;
    if (scale >= f.R) {
        pat = (1u << (f.nbits - 1)) - 1u;
    } else if (scale < -f.R) {
        pat = 1u;
    } else {
        const int k = scale >> f.es;                  // floor division
        const int e = scale - (k << f.es);
        const int rl = k >= 0 ? k + 2 : 1 - k;        // regime incl. terminator
        const uint64_t regime = k >= 0 ? (((uint64_t(1) << (k + 1)) - 1) << 1) : 1;
        const int head = rl + f.es;                   // < 64
        uint64_t w = regime << (64 - rl);
        if (f.es > 0) w |= uint64_t(e) << (64 - head);
        const uint64_t frac = sig << 1;               // 63 fraction bits, left-aligned
        w |= frac >> head;
        bool st = sticky || (frac << (64 - head)) != 0;
        pat = uint32_t(w >> (65 - f.nbits));
        const bool guard = (w >> (64 - f.nbits)) & 1;
        st = st || (w << f.nbits) != 0;
        if (guard && (st || (pat & 1))) ++pat;
    }
    const uint32_t mask = f.nbits == 32 ? 0xFFFFFFFFu : ((1u << f.nbits) - 1u);
    return neg ? ((0u - pat) & mask) : pat;
}

// pack_round with a 32-bit window for nbits <= 16 (regime <= 15 bits, es <= 4):
// identical results to pack_round with sig = sig32 << 32 | low, sticky |= low != 0.
__device__ __forceinline__ uint32_t pack_round32(const PositFmt& f, bool neg, int scale,
                                                 uint32_t sig32, bool sticky) {
    uint32_t pat;
    if (scale >= f.R) {
        pat = (1u << (f.nbits - 1)) - 1u;
    } else if (scale < -f.R) {
        pat = 1u;
    } else {
        const int k = scale >> f.es;
        const int e = scale - (k << f.es);
        const int rl = k >= 0 ? k + 2 : 1 - k;
        const uint32_t regime = k >= 0 ? (((1u << (k + 1)) - 1u) << 1) : 1u;
        const int head = rl + f.es;  // in [2, 19]
        uint32_t w = regime << (32 - rl);
        if (f.es > 0) w |= uint32_t(e) << (32 - head);
        const uint32_t frac = sig32 << 1;
        w |= frac >> head;
        bool st = sticky || (frac << (32 - head)) != 0;
        pat = w >> (33 - f.nbits);
        const bool guard = (w >> (32 - f.nbits)) & 1u;
        st = st || (w << f.nbits) != 0;
        if (guard && (st || (pat & 1u))) ++pat;
    }
    const uint32_t mask = (1u << f.nbits) - 1u;
    return neg ? ((0u - pat) & mask) : pat;
}

// Branch-free pack_round32 (same result): saturation and the round-up are
// selects, shifts are kept in range by clamping the scale, so the GEMM
// epilogue can interleave the conversions of its 8 columns.
__device__ __forceinline__ uint32_t pack_round32_bf(const PositFmt& f, bool neg, int scale,
                                                    uint32_t sig32, bool sticky) {
    const bool hi_sat = scale >= f.R, lo_sat = scale < -f.R;
    const int sc = scale < -f.R ? -f.R : (scale > f.R - 1 ? f.R - 1 : scale);
    const int k = sc >> f.es;
    const int e = sc - (k << f.es);
    const bool kpos = k >= 0;
    const int rl = kpos ? k + 2 : 1 - k;
    const uint32_t regime = kpos ? (((1u << (k + 1)) - 1u) << 1) : 1u;
    const int head = rl + f.es;
    uint32_t w = regime << (32 - rl);
    if (f.es > 0) w |= uint32_t(e) << (32 - head);
    const uint32_t frac = sig32 << 1;
    w |= frac >> head;
    const bool st = sticky || (frac << (32 - head)) != 0 || (w << f.nbits) != 0;
    uint32_t pat = w >> (33 - f.nbits);
    const uint32_t guard = (w >> (32 - f.nbits)) & 1u;
    pat += guard & (uint32_t(st) | (pat & 1u));
    pat = hi_sat ? (1u << (f.nbits - 1)) - 1u : (lo_sat ? 1u : pat);
    const uint32_t mask = (1u << f.nbits) - 1u;
    return neg ? ((0u - pat) & mask) : pat;
}

// Branch-free quire word -> posit (same results as quire_word_to_posit).
__device__ __forceinline__ uint32_t quire_word_to_posit_bf(const PositFmt& f, uint32_t q) {
    const uint32_t m = f.W >= 32 ? 0xFFFFFFFFu : ((1u << f.W) - 1u);
    q &= m;
    const bool neg = ((q >> (f.W - 1)) & 1u) != 0;
    const uint32_t mag = neg ? ((0u - q) & m) : q;
    const int lz = __clz(mag);
    const uint32_t c = pack_round32_bf(f, neg, 31 - lz - 2 * f.R, mag << (lz & 31), false);
    return mag == 0 ? 0u : c;
}
__device__ __forceinline__ uint32_t quire_word_to_posit_bf(const PositFmt& f, uint64_t q) {
    const uint64_t m = f.W >= 64 ? ~uint64_t(0) : ((uint64_t(1) << f.W) - 1);
    q &= m;
    const bool neg = ((q >> (f.W - 1)) & 1) != 0;
    const uint64_t mag = neg ? ((0 - q) & m) : q;
    const int lz = __clzll(mag);
    const uint64_t sig = mag << (lz & 63);
    const uint32_t c =
        pack_round32_bf(f, neg, 63 - lz - 2 * f.R, uint32_t(sig >> 32), uint32_t(sig) != 0);
    return mag == 0 ? 0u : c;
}
__device__ __forceinline__ uint32_t quire_word_to_posit_bf(const PositFmt& f, unsigned __int128 q) {
    uint64_t lo = uint64_t(q), hi = uint64_t(q >> 64);
    const uint64_t hmask = f.W >= 128 ? ~uint64_t(0) : ((uint64_t(1) << (f.W - 64)) - 1);  // W > 64
    hi &= hmask;
    const bool neg = ((hi >> (f.W - 65)) & 1) != 0;
    const uint64_t nlo = 0 - lo, nhi = (~hi + (lo == 0 ? 1 : 0)) & hmask;
    lo = neg ? nlo : lo;
    hi = neg ? nhi : hi;
    const bool hz = hi == 0;
    const int lzh = __clzll(hi), lzl = __clzll(lo);
    const uint64_t sig_h = (hi << (lzh & 63)) | ((lo >> 1) >> ((63 - lzh) & 63));
    const bool st_h = (lo << (lzh & 63)) != 0;
    const uint64_t sig = hz ? (lo << (lzl & 63)) : sig_h;
    const bool sticky = (!hz && st_h) || uint32_t(sig) != 0;
    const int top = hz ? 63 - lzl : 127 - lzh;
    const uint32_t c = pack_round32_bf(f, neg, top - 2 * f.R, uint32_t(sig >> 32), sticky);
    return (hz && lo == 0) ? 0u : c;
}

// Quire word (W <= 32 / 64 / 128 bits held in uint32 / uint64 / u128) -> posit,
// nbits <= 16.  Same result as quire_to_posit.
__device__ __forceinline__ uint32_t quire_word_to_posit(const PositFmt& f, uint32_t q) {
    const uint32_t m = f.W >= 32 ? 0xFFFFFFFFu : ((1u << f.W) - 1u);
    q &= m;
    const bool neg = ((q >> (f.W - 1)) & 1u) != 0;
    const uint32_t mag = neg ? ((0u - q) & m) : q;
    if (mag == 0) return 0;
    const int top = 31 - __clz(mag);
    return pack_round32(f, neg, top - 2 * f.R, mag << (31 - top), false);
}
__device__ __forceinline__ uint32_t quire_word_to_posit(const PositFmt& f, uint64_t q) {
    const uint64_t m = f.W >= 64 ? ~uint64_t(0) : ((uint64_t(1) << f.W) - 1);
    q &= m;
    const bool neg = ((q >> (f.W - 1)) & 1) != 0;
    const uint64_t mag = neg ? ((0 - q) & m) : q;
    if (mag == 0) return 0;
    const int top = 63 - __clzll(mag);
    const uint64_t sig = mag << (63 - top);
    return pack_round32(f, neg, top - 2 * f.R, uint32_t(sig >> 32), uint32_t(sig) != 0);
}
__device__ __forceinline__ uint32_t quire_word_to_posit(const PositFmt& f, unsigned __int128 q) {
    const unsigned __int128 one = 1;
    const unsigned __int128 m = f.W >= 128 ? ~(unsigned __int128)0 : ((one << f.W) - 1);
    q &= m;
    const bool neg = ((q >> (f.W - 1)) & 1) != 0;
    const unsigned __int128 mag = neg ? ((0 - q) & m) : q;
    if (mag == 0) return 0;
    const uint64_t hi = uint64_t(mag >> 64), lo = uint64_t(mag);
    int top;
    uint64_t sig;
    bool sticky;
    if (hi) {
        const int lz = __clzll(hi);
        top = 127 - lz;
        sig = lz ? ((hi << lz) | (lo >> (64 - lz))) : hi;
        sticky = lz ? (lo << lz) != 0 : lo != 0;
    } else {
        const int lz = __clzll(lo);
        top = 63 - lz;
        sig = lo << lz;
        sticky = false;
    }
    return pack_round32(f, neg, top - 2 * f.R, uint32_t(sig >> 32), sticky || uint32_t(sig) != 0);
}

// Quire::to_posit on a W-bit two's complement value held in 128 bits
// (W <= 128).  LSB weight 2^-2R.
__device__ __forceinline__ uint32_t quire_to_posit(const PositFmt& f, unsigned __int128 q) {
    const unsigned __int128 one = 1;
    const unsigned __int128 m = f.W >= 128 ? ~(unsigned __int128)0 : ((one << f.W) - 1);
    q &= m;
    const bool neg = ((q >> (f.W - 1)) & 1) != 0;
    const unsigned __int128 mag = neg ? ((0 - q) & m) : q;
    if (mag == 0) return 0;
    const uint64_t hi = uint64_t(mag >> 64), lo = uint64_t(mag);
    const int top = hi ? 127 - __clzll(hi) : 63 - __clzll(lo);
    uint64_t sig;
    bool sticky;
    if (top >= 63) {
        const int drop = top - 63;
        sig = uint64_t(mag >> drop);
        sticky = drop > 0 && (mag & ((one << drop) - 1)) != 0;
    } else {
        sig = lo << (63 - top);
        sticky = false;
    }
    return pack_round(f, neg, top - 2 * f.R, sig, sticky);
}

// 64-bit variant for W <= 64 (e.g. posit(8,0) W=32, posit(8,1) W=56).
__device__ __forceinline__ uint32_t quire_to_posit64(const PositFmt& f, uint64_t q) {
    const uint64_t m = f.W >= 64 ? ~uint64_t(0) : ((uint64_t(1) << f.W) - 1);
    q &= m;
    const bool neg = ((q >> (f.W - 1)) & 1) != 0;
    const uint64_t mag = neg ? ((0 - q) & m) : q;
    if (mag == 0) return 0;
    const int top = 63 - __clzll(mag);
    return pack_round(f, neg, top - 2 * f.R, mag << (63 - top), false);
}

}  // namespace pnn_b200
