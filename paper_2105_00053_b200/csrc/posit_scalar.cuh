// Device scalar posit arithmetic for the elementwise kernels (ReLU, max-pool,
// softmax cross-entropy, SGD, stage conversions).  Bit-exact with the
// reference's scalar ALU for nbits <= 16 and 2*max_scale <= 60:
//   add/sub/mul/div   proj/src/posit.cpp:393-416 (exact kernels :172-228)
//   convert           posit.cpp:487-495
//   compare           posit.cpp:514-520
//   from_float64      posit.cpp:243-260, 502-508
//   ldexp_posit       posit.cpp:522-532
//   round_to_int      posit.cpp:534-553,  to_int64 :555-563
//   from_int64        posit_math.cpp:51-57
//   exp_posit         posit_math.cpp:67-85,  log_posit :87-107
// add/sub/mul round the exact result (held in the integer image, LSB 2^-R or
// 2^-2R) once; div follows the reference's 128/64 long division with a sticky.
#pragma once

#include <cstdint>

#include "posit_device.cuh"

namespace pnn_b200 {

struct Unp {
    int cls;  // 0 zero, 1 NaR, 2 finite
    bool neg;
    int scale;
    uint64_t sig;  // normalized, bit 63 set
};

__device__ __forceinline__ uint32_t code_mask(const PositFmt& f) {
    return f.nbits == 32 ? 0xFFFFFFFFu : ((1u << f.nbits) - 1u);
}
__device__ __forceinline__ uint32_t nar_of(const PositFmt& f) { return 1u << (f.nbits - 1); }

__device__ __forceinline__ Unp unpack(const PositFmt& f, uint32_t code) {
    Unp u;
    code &= code_mask(f);
    u.neg = false;
    u.scale = 0;
    u.sig = 0;
    if (code == 0) { u.cls = 0; return u; }
    if (code == nar_of(f)) { u.cls = 1; return u; }
    u.cls = 2;
    u.neg = (code & nar_of(f)) != 0;
    const uint32_t mag = u.neg ? ((0u - code) & code_mask(f)) : code;
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
    u.scale = k * (1 << f.es) + int(e);
    u.sig = (uint64_t(1) << 63) | (fb > 0 ? uint64_t(frac) << (63 - fb) : 0);
    return u;
}

// Round an exact nonzero magnitude mag * 2^lsb_exp (sign neg) to a posit.
__device__ __forceinline__ uint32_t round_mag128(const PositFmt& f, bool neg,
                                                 unsigned __int128 mag, int lsb_exp) {
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
    return pack_round(f, neg, top + lsb_exp, sig, sticky);
}

__device__ __forceinline__ uint32_t p_negate(const PositFmt& f, uint32_t a) {
    return (0u - a) & code_mask(f);
}

// add/sub/mul for the wide elementwise formats (56 < 2R <= 124, e.g. the
// posit(12,2) optimizer and posit(10,2) loss of the posit(8,2)* preset):
// add/sub on 128-bit integer images (|X| <= 2^(2R) < 2^125, exact); mul on
// the significands (two <= 16-bit significands, exact 128-bit product).
// Either way the exact result is rounded once, as in the narrow path.
static __device__ __noinline__ uint32_t p_op_wide(const PositFmt& f, int op, uint32_t a,
                                                  uint32_t b) {
    if (op == 2) {
        const Unp ua = unpack(f, a), ub = unpack(f, b);
        if (ua.cls == 0 || ub.cls == 0) return 0;
        const unsigned __int128 pr = (unsigned __int128)ua.sig * ub.sig;  // value * 2^(126-sa-sb)
        return round_mag128(f, ua.neg != ub.neg, pr, ua.scale + ub.scale - 126);
    }
    __int128 xa, xb;
    decode_x128(a, f, xa);
    decode_x128(b, f, xb);
    if (op == 1) xb = -xb;
    if (xb == 0) return a;                          // x + 0 == x (posit.cpp:400)
    if (xa == 0) return op == 1 ? p_negate(f, b) : b;
    const __int128 s = xa + xb;
    if (s == 0) return 0;
    const bool neg = s < 0;
    return round_mag128(f, neg, (unsigned __int128)(neg ? -s : s), -f.R);
}

// op: 0 add, 1 sub, 2 mul, 3 div
__device__ __forceinline__ uint32_t p_op(const PositFmt& f, int op, uint32_t a, uint32_t b) {
    const uint32_t m = code_mask(f), nar = nar_of(f);
    a &= m;
    b &= m;
    if (a == nar || b == nar) return nar;
    if (op == 3) {
        if (b == 0) return nar;
        if (a == 0) return 0;
        const Unp ua = unpack(f, a), ub = unpack(f, b);
        const unsigned __int128 num = (unsigned __int128)ua.sig << 64;
        const unsigned __int128 q = num / ub.sig;
        const unsigned __int128 rem = num - q * ub.sig;
        int scale = ua.scale - ub.scale;
        uint64_t sig;
        bool sticky;
        if (q >> 64) {
            sig = uint64_t(q >> 1);
            sticky = (q & 1) != 0 || rem != 0;
        } else {
            sig = uint64_t(q);
            sticky = rem != 0;
            scale -= 1;
        }
        return pack_round(f, ua.neg != ub.neg, scale, sig, sticky);
    }
    if (2 * f.R > 56) return p_op_wide(f, op, a, b);
    int64_t xa, xb;
    decode_x(a, f, xa);
    decode_x(b, f, xb);
    if (op == 2) {
        if (xa == 0 || xb == 0) return 0;
        const bool neg = (xa < 0) != (xb < 0);
        const unsigned __int128 pa = (unsigned __int128)(xa < 0 ? -xa : xa);
        const unsigned __int128 pb = (unsigned __int128)(xb < 0 ? -xb : xb);
        return round_mag128(f, neg, pa * pb, -2 * f.R);
    }
    if (op == 1) xb = -xb;
    if (xb == 0) return a;                          // x + 0 == x (posit.cpp:400)
    if (xa == 0) return op == 1 ? p_negate(f, b) : b;
    const __int128 s = (__int128)xa + xb;
    if (s == 0) return 0;
    const bool neg = s < 0;
    return round_mag128(f, neg, (unsigned __int128)(neg ? -s : s), -f.R);
}

__device__ __forceinline__ uint32_t p_add(const PositFmt& f, uint32_t a, uint32_t b) { return p_op(f, 0, a, b); }
__device__ __forceinline__ uint32_t p_sub(const PositFmt& f, uint32_t a, uint32_t b) { return p_op(f, 1, a, b); }
__device__ __forceinline__ uint32_t p_mul(const PositFmt& f, uint32_t a, uint32_t b) { return p_op(f, 2, a, b); }
__device__ __forceinline__ uint32_t p_div(const PositFmt& f, uint32_t a, uint32_t b) { return p_op(f, 3, a, b); }

__device__ __forceinline__ uint32_t p_convert(const PositFmt& src, const PositFmt& dst, uint32_t c) {
    const Unp u = unpack(src, c);
    if (u.cls == 0) return 0;
    if (u.cls == 1) return nar_of(dst);
    return pack_round(dst, u.neg, u.scale, u.sig, false);
}

// Signed pattern comparison (NaR lowest).
__device__ __forceinline__ int p_compare(const PositFmt& f, uint32_t a, uint32_t b) {
    const int sh = 32 - f.nbits;
    const int32_t ia = int32_t(a << sh) >> sh, ib = int32_t(b << sh) >> sh;
    return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

__device__ __forceinline__ uint32_t p_from_float64(const PositFmt& f, double x) {
    if (x == 0.0) return 0;
    const uint64_t b = uint64_t(__double_as_longlong(x));
    const int be = int((b >> 52) & 0x7FF);
    if (be == 0x7FF) return nar_of(f);
    const bool neg = (b >> 63) != 0;
    const uint64_t mant = b & ((uint64_t(1) << 52) - 1);
    uint64_t sig;
    int scale;
    if (be == 0) {
        const int lead = __clzll(mant);
        sig = mant << lead;
        scale = -1023 - (lead - 11);
    } else {
        sig = ((uint64_t(1) << 52) | mant) << 11;
        scale = be - 1023;
    }
    return pack_round(f, neg, scale, sig, false);
}

__device__ __forceinline__ uint32_t p_ldexp(const PositFmt& f, uint32_t c, int k) {
    const Unp u = unpack(f, c);
    if (u.cls != 2) return c & code_mask(f);
    long s = long(u.scale) + k;
    if (s > f.R) s = f.R;
    if (s < -f.R - 1) s = -f.R - 1;
    return pack_round(f, u.neg, int(s), u.sig, false);
}

__device__ __forceinline__ uint32_t p_round_to_int(const PositFmt& f, uint32_t c) {
    const Unp u = unpack(f, c);
    if (u.cls != 2) return c & code_mask(f);
    if (u.scale >= 63) return c & code_mask(f);
    if (u.scale < -1) return 0;
    if (u.scale == -1) {
        if (u.sig == (uint64_t(1) << 63)) return 0;
        return pack_round(f, u.neg, 0, uint64_t(1) << 63, false);
    }
    const int fb = 63 - u.scale;
    uint64_t ip = u.sig >> fb;
    const uint64_t rem = u.sig & ((uint64_t(1) << fb) - 1);
    const uint64_t half = uint64_t(1) << (fb - 1);
    if (rem > half || (rem == half && (ip & 1))) ++ip;
    const int lead = __clzll(ip);
    return pack_round(f, u.neg, 63 - lead, ip << lead, false);
}

__device__ __forceinline__ int64_t p_to_int64(const PositFmt& f, uint32_t c) {
    const Unp u = unpack(f, c);
    if (u.cls != 2 || u.scale < 0) return 0;
    if (u.scale >= 62) return u.neg ? INT64_MIN : INT64_MAX;
    const int64_t mag = int64_t(u.sig >> (63 - u.scale));
    return u.neg ? -mag : mag;
}

__device__ __forceinline__ uint32_t p_from_int64(const PositFmt& f, int64_t v) {
    if (v == 0) return 0;
    const bool neg = v < 0;
    const uint64_t mag = neg ? (~uint64_t(v) + 1) : uint64_t(v);
    const int lead = __clzll(mag);
    return pack_round(f, neg, 63 - lead, mag << lead, false);
}

// exp_posit: k = round(x * log2e); r = x - k*ln2; degree-10 Horner in posit
// ops with 1/k! quantized by from_float64; ldexp by k.
static __device__ __noinline__ uint32_t p_exp(const PositFmt& f, uint32_t x) {
    x &= code_mask(f);
    if (x == nar_of(f)) return x;
    if (x == 0) return p_from_int64(f, 1);
    const uint32_t log2e = p_from_float64(f, 1.4426950408889634);
    const uint32_t ln2 = p_from_float64(f, 0.6931471805599453);
    const uint32_t kp = p_round_to_int(f, p_mul(f, x, log2e));
    const int64_t k = p_to_int64(f, kp);
    if (k > f.R) return nar_of(f) - 1;
    if (k < -f.R - 1) return 1;
    const uint32_t r = p_sub(f, x, p_mul(f, kp, ln2));
    double fact = 1.0;
    for (int i = 1; i <= 10; ++i) fact *= i;  // 10!
    uint32_t p = p_from_float64(f, 1.0 / fact);
    for (int i = 9; i >= 0; --i) {
        fact /= (i + 1);  // i!  (exact in double for i <= 10, same value as the ascending product)
        p = p_add(f, p_mul(f, p, r), p_from_float64(f, 1.0 / fact));
    }
    return p_ldexp(f, p, int(k));
}

// log_posit: x = m * 2^s, m in [1, 1.5) after one halving, 2*atanh series
// in t = (m-1)/(m+1), 8 terms with 1/(2k+1) quantized by from_float64.
static __device__ __noinline__ uint32_t p_log(const PositFmt& f, uint32_t x) {
    x &= code_mask(f);
    const uint32_t nar = nar_of(f);
    if (x == nar || x == 0 || (x & nar)) return nar;
    const uint32_t one = p_from_int64(f, 1), two = p_from_int64(f, 2);
    const uint32_t ln2 = p_from_float64(f, 0.6931471805599453);
    const uint32_t three_halves = p_from_float64(f, 1.5);
    const Unp u = unpack(f, x);
    int s = u.scale;
    uint32_t m = p_ldexp(f, x, -s);
    if (p_compare(f, m, three_halves) >= 0) {
        m = p_ldexp(f, m, -1);
        s += 1;
    }
    const uint32_t t = p_div(f, p_sub(f, m, one), p_add(f, m, one));
    const uint32_t uu = p_mul(f, t, t);
    uint32_t inner = p_from_float64(f, 1.0 / 15.0);
    for (int i = 6; i >= 0; --i) inner = p_add(f, p_mul(f, inner, uu), p_from_float64(f, 1.0 / (2 * i + 1)));
    const uint32_t logm = p_mul(f, two, p_mul(f, t, inner));
    return p_add(f, p_mul(f, p_from_int64(f, s), ln2), logm);
}

// tanh_posit, posit_math.cpp:109-118: r = (1 - e^(-2|x|)) / (1 + e^(-2|x|)), odd.
static __device__ __noinline__ uint32_t p_tanh(const PositFmt& f, uint32_t x) {
    x &= code_mask(f);
    if (x == nar_of(f) || x == 0) return x;
    const bool neg = (x & nar_of(f)) != 0;
    const uint32_t ax = neg ? p_negate(f, x) : x;
    const uint32_t one = p_from_int64(f, 1);
    const uint32_t t = p_exp(f, p_negate(f, p_ldexp(f, ax, 1)));
    const uint32_t r = p_div(f, p_sub(f, one, t), p_add(f, one, t));
    return neg ? p_negate(f, r) : r;
}

// sigmoid_posit, posit_math.cpp:120-130.
static __device__ __noinline__ uint32_t p_sigmoid(const PositFmt& f, uint32_t x) {
    x &= code_mask(f);
    if (x == nar_of(f)) return x;
    const uint32_t one = p_from_int64(f, 1);
    if (!(x & nar_of(f))) {
        const uint32_t t = p_exp(f, p_negate(f, x));
        return p_div(f, one, p_add(f, one, t));
    }
    const uint32_t t = p_exp(f, x);
    return p_div(f, t, p_add(f, one, t));
}

// sqrt_posit, posit_math.cpp:132-160: correctly rounded.  value = M * 2^(2q)
// with M = sig << j in [2^126, 2^128); the floor root r in [2^63, 2^64) and
// its remainder are unique, found here by the restoring (digit-by-digit)
// method; sticky = remainder != 0.
static __device__ __noinline__ uint32_t p_sqrt(const PositFmt& f, uint32_t x) {
    x &= code_mask(f);
    if (x == 0 || x == nar_of(f)) return x;
    if (x & nar_of(f)) return nar_of(f);
    const Unp u = unpack(f, x);
    const int j = (u.scale & 1) == 0 ? 63 : 64;
    const unsigned __int128 M = (unsigned __int128)u.sig << j;
    const int q = (u.scale - 63 - j) / 2;
    unsigned __int128 rem = 0, root = 0;
    for (int i = 63; i >= 0; --i) {
        rem = (rem << 2) | ((M >> (2 * i)) & 3);
        const unsigned __int128 t = (root << 2) | 1;
        root <<= 1;
        if (rem >= t) {
            rem -= t;
            root |= 1;
        }
    }
    return pack_round(f, false, q + 63, uint64_t(root), rem != 0);
}

}  // namespace pnn_b200
