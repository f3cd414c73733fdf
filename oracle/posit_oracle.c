/* Plain-C restatement of the reference's posit/quire hot path.
 *
 * TEST INFRASTRUCTURE ONLY -- see posit_oracle.h.  Written from the
 * reference's algorithm (file:line cited per function), not copied from it.
 * The key restatement: a posit x of format
 * (n,es) with R = max_scale is x = X * 2^-R for an exact integer X, and the
 * quire after any sequence of accumulate_product calls holds exactly
 * sum(X_a*X_b) mod 2^W, W = quire_bits, LSB weight 2^-2R (quire.hpp:53-60,
 * quire.cpp:26-53).  Reading it out is one rounding of that integer.
 */
#include "posit_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

#define WL 16 /* 1024-bit wide integers: enough for every nbits <= 32 quire */

int po_max_scale(int nbits, int es) { return (nbits - 2) << es; }
int po_quire_bits(int nbits, int es) { return 4 * po_max_scale(nbits, es) + nbits; }

static uint64_t pmask(int nbits) {
    return nbits >= 64 ? ~(uint64_t)0 : (((uint64_t)1 << nbits) - 1);
}
static uint64_t nar_of(int nbits) { return (uint64_t)1 << (nbits - 1); }

/* ---------------------------------------------------------------- decode */

/* posit.cpp:67-91: two's complement of negative patterns, then regime run,
 * terminator, up to es exponent bits (truncated low bits read as zero), and
 * the remaining fraction bits.  Walked bit by bit here. */
po_unpacked po_unpack(int nbits, int es, uint64_t code) {
    po_unpacked u;
    memset(&u, 0, sizeof u);
    uint64_t m = pmask(nbits);
    code &= m;
    if (code == 0) { u.cls = 0; return u; }
    if (code == nar_of(nbits)) { u.cls = 1; return u; }
    u.cls = 2;
    u.neg = (int)((code >> (nbits - 1)) & 1);
    uint64_t mag = u.neg ? ((~code + 1) & m) : code;
    int i = nbits - 2;
    int first = (int)((mag >> i) & 1);
    int run = 0;
    while (i >= 0 && (int)((mag >> i) & 1) == first) { ++run; --i; }
    int k = first ? run - 1 : -run;
    --i; /* skip the terminator (if any bit is left) */
    int rem = i + 1;
    if (rem < 0) rem = 0;
    int ebits = es < rem ? es : rem;
    unsigned e = 0;
    for (int b = 0; b < ebits; ++b) e = (e << 1) | (unsigned)((mag >> (rem - 1 - b)) & 1);
    e <<= (es - ebits);
    int fb = rem - ebits;
    uint64_t frac = fb > 0 ? (mag & ((((uint64_t)1) << fb) - 1)) : 0;
    u.scale = k * (1 << es) + (int)e;
    u.fbits = fb;
    u.frac = frac;
    u.sig = ((uint64_t)1 << 63) | (fb > 0 ? frac << (63 - fb) : 0);
    return u;
}

/* posit_tables.cpp:43-64 (Fixed form: x = (-1)^neg * sig * 2^lsb_scale). */
void po_decode_fixed(int nbits, int es, uint64_t code, int32_t* lsb_scale, uint32_t* sig,
                     uint8_t* neg, uint8_t* nar) {
    po_unpacked u = po_unpack(nbits, es, code);
    *lsb_scale = 0; *sig = 0; *neg = 0; *nar = 0;
    if (u.cls == 1) { *nar = 1; return; }
    if (u.cls == 0) return;
    *neg = (uint8_t)u.neg;
    *sig = (uint32_t)(((uint64_t)1 << u.fbits) | u.frac);
    *lsb_scale = u.scale - u.fbits;
}

/* ------------------------------------------------------------ pack/round */

/* posit.cpp:93-132.  Build the unbounded encoding bit string
 * [regime][es exponent bits][63 fraction bits], keep nbits-1 payload bits,
 * round to nearest with ties to the even pattern on guard/sticky,
 * saturate at maxpos (scale >= R), never underflow (scale < -R -> minpos). */
uint64_t po_pack_round(int nbits, int es, int neg, int scale, uint64_t sig, int sticky) {
    if (sig == 0) return 0;
    const int R = po_max_scale(nbits, es);
    uint64_t pat;
    if (scale >= R) {
        pat = nar_of(nbits) - 1;
    } else if (scale < -R) {
        pat = 1;
    } else {
        int useed = 1 << es;
        int k = scale >= 0 ? scale / useed : -((-scale + useed - 1) / useed);
        int e = scale - k * useed;
        unsigned char bits[64 + 8 + 64 + 8];
        int len = 0;
        if (k >= 0) {
            for (int i = 0; i < k + 1; ++i) bits[len++] = 1;
            bits[len++] = 0;
        } else {
            for (int i = 0; i < -k; ++i) bits[len++] = 0;
            bits[len++] = 1;
        }
        for (int b = es - 1; b >= 0; --b) bits[len++] = (unsigned char)((e >> b) & 1);
        for (int b = 62; b >= 0; --b) bits[len++] = (unsigned char)((sig >> b) & 1);
        int keep = nbits - 1;
        pat = 0;
        for (int i = 0; i < keep; ++i) pat = (pat << 1) | (i < len ? bits[i] : 0);
        int guard = keep < len ? bits[keep] : 0;
        int st = sticky;
        for (int i = keep + 1; i < len; ++i) st |= bits[i];
        if (guard && (st || (pat & 1))) ++pat;
    }
    return neg ? ((~pat + 1) & pmask(nbits)) : pat;
}

/* ------------------------------------------------------------ wide ints */

typedef struct { uint64_t w[WL]; } wide;

static void wide_zero(wide* a) { memset(a, 0, sizeof *a); }

/* a += (v << pos) or a -= (v << pos), v a 128-bit magnitude; mod 2^(64*WL). */
static void wide_addsub(wide* a, u128 v, int pos, int negate) {
    wide t;
    wide_zero(&t);
    int limb = pos >> 6, off = pos & 63;
    uint64_t lo = (uint64_t)v, hi = (uint64_t)(v >> 64);
    uint64_t parts[3];
    parts[0] = lo << off;
    parts[1] = off ? ((hi << off) | (lo >> (64 - off))) : hi;
    parts[2] = off ? (hi >> (64 - off)) : 0;
    for (int i = 0; i < 3; ++i)
        if (limb + i < WL) t.w[limb + i] = parts[i];
    if (!negate) {
        uint64_t c = 0;
        for (int i = 0; i < WL; ++i) {
            u128 s = (u128)a->w[i] + t.w[i] + c;
            a->w[i] = (uint64_t)s;
            c = (uint64_t)(s >> 64);
        }
    } else {
        uint64_t br = 0;
        for (int i = 0; i < WL; ++i) {
            u128 s = (u128)a->w[i] - t.w[i] - br;
            a->w[i] = (uint64_t)s;
            br = (uint64_t)(s >> 64) ? 1 : 0;
        }
    }
}

static void wide_mask(wide* a, int W) {
    for (int i = 0; i < WL; ++i) {
        int lo = i * 64;
        if (lo >= W) a->w[i] = 0;
        else if (lo + 64 > W) a->w[i] &= (((uint64_t)1) << (W - lo)) - 1;
    }
}

static int wide_bit(const wide* a, int b) { return (int)((a->w[b >> 6] >> (b & 63)) & 1); }

/* Round the W-bit two's complement integer q (LSB weight 2^lsb_exp) to a
 * posit -- Quire::to_posit, quire.cpp:105-146. */
static uint64_t wide_round(int nbits, int es, const wide* q, int W, int lsb_exp) {
    wide m = *q;
    wide_mask(&m, W);
    int neg = wide_bit(&m, W - 1);
    if (neg) { /* magnitude = 2^W - q */
        for (int i = 0; i < WL; ++i) m.w[i] = ~m.w[i];
        uint64_t c = 1;
        for (int i = 0; i < WL; ++i) {
            u128 s = (u128)m.w[i] + c;
            m.w[i] = (uint64_t)s;
            c = (uint64_t)(s >> 64);
        }
        wide_mask(&m, W);
    }
    int top = -1;
    for (int b = W - 1; b >= 0; --b)
        if (wide_bit(&m, b)) { top = b; break; }
    if (top < 0) return 0;
    uint64_t sig = 0;
    for (int i = 0; i < 64; ++i) {
        int b = top - i;
        sig = (sig << 1) | (uint64_t)(b >= 0 ? wide_bit(&m, b) : 0);
    }
    int sticky = 0;
    for (int b = top - 64; b >= 0 && !sticky; --b) sticky = wide_bit(&m, b);
    return po_pack_round(nbits, es, neg, top + lsb_exp, sig, sticky);
}

/* ----------------------------------------------------------------- quire */

struct po_quire {
    int nbits, es, R, W, nar;
    wide acc;
};

po_quire* po_quire_new(int nbits, int es) {
    po_quire* q = (po_quire*)calloc(1, sizeof(po_quire));
    q->nbits = nbits;
    q->es = es;
    q->R = po_max_scale(nbits, es);
    q->W = po_quire_bits(nbits, es);
    return q;
}
void po_quire_free(po_quire* q) { free(q); }
void po_quire_clear(po_quire* q) { wide_zero(&q->acc); q->nar = 0; }

/* quire.hpp:62-67 accumulate_value / quire.cpp:61-66 add_posit. */
void po_quire_add_posit(po_quire* q, uint64_t a) {
    po_unpacked u = po_unpack(q->nbits, q->es, a);
    if (u.cls == 1) { q->nar = 1; return; }
    if (u.cls == 0) return;
    uint64_t sig = ((uint64_t)1 << u.fbits) | u.frac;
    wide_addsub(&q->acc, sig, (u.scale - u.fbits) + 2 * q->R, u.neg);
    wide_mask(&q->acc, q->W);
}

/* quire.cpp:68-103: NaR operand makes the quire NaR (checked before zero). */
static void quire_prod(po_quire* q, uint64_t a, uint64_t b, int negate) {
    po_unpacked ua = po_unpack(q->nbits, q->es, a), ub = po_unpack(q->nbits, q->es, b);
    if (ua.cls == 1 || ub.cls == 1) { q->nar = 1; return; }
    if (ua.cls == 0 || ub.cls == 0) return;
    u128 sa = ((u128)1 << ua.fbits) | ua.frac, sb = ((u128)1 << ub.fbits) | ub.frac;
    int pos = (ua.scale - ua.fbits) + (ub.scale - ub.fbits) + 2 * q->R;
    wide_addsub(&q->acc, sa * sb, pos, (ua.neg ^ ub.neg ^ negate) != 0);
    wide_mask(&q->acc, q->W);
}
void po_quire_add_product(po_quire* q, uint64_t a, uint64_t b) { quire_prod(q, a, b, 0); }
void po_quire_sub_product(po_quire* q, uint64_t a, uint64_t b) { quire_prod(q, a, b, 1); }

uint64_t po_quire_to_posit(const po_quire* q) {
    if (q->nar) return nar_of(q->nbits);
    return wide_round(q->nbits, q->es, &q->acc, q->W, -2 * q->R);
}

int po_quire_words(const po_quire* q, uint64_t* out, int max_words, int* nar) {
    int n = (q->W + 63) / 64;
    if (n > max_words) return -1;
    memcpy(out, q->acc.w, (size_t)n * 8);
    *nar = q->nar;
    return n;
}

/* ------------------------------------------------------------ scalar ops */

/* Exact add/sub/mul through a scratch quire: the exact sum |a|+|b| <= 2^(R+1)
 * and product <= 2^2R both fit the W-bit quire, so one rounding of the exact
 * value equals the reference's exact kernels (posit.cpp:172-208, 393-416). */
uint64_t po_scalar_op(int nbits, int es, int op, uint64_t a, uint64_t b) {
    uint64_t m = pmask(nbits), nar = nar_of(nbits);
    a &= m;
    b &= m;
    if (a == nar || b == nar) return nar;
    if (op == 3) { /* div_exact, posit.cpp:210-228 */
        if (b == 0) return nar;
        if (a == 0) return 0;
        po_unpacked ua = po_unpack(nbits, es, a), ub = po_unpack(nbits, es, b);
        u128 num = (u128)ua.sig << 64;
        u128 qt = num / ub.sig, rem = num % ub.sig;
        int scale = ua.scale - ub.scale;
        uint64_t sig;
        int sticky;
        if (qt >> 64) {
            sig = (uint64_t)(qt >> 1);
            sticky = (int)(qt & 1) || rem != 0;
        } else {
            sig = (uint64_t)qt;
            sticky = rem != 0;
            scale -= 1;
        }
        return po_pack_round(nbits, es, ua.neg != ub.neg, scale, sig, sticky);
    }
    po_quire q;
    memset(&q, 0, sizeof q);
    q.nbits = nbits;
    q.es = es;
    q.R = po_max_scale(nbits, es);
    q.W = po_quire_bits(nbits, es);
    if (op == 2) {
        po_quire_add_product(&q, a, b);
    } else {
        po_quire_add_posit(&q, a);
        po_quire_add_posit(&q, op == 1 ? ((~b + 1) & m) : b);
    }
    return po_quire_to_posit(&q);
}

uint64_t po_convert(int sn, int se, int dn, int de, uint64_t code) {
    po_unpacked u = po_unpack(sn, se, code);
    if (u.cls == 0) return 0;
    if (u.cls == 1) return nar_of(dn);
    return po_pack_round(dn, de, u.neg, u.scale, u.sig, 0);
}

int po_compare(int nbits, int es, uint64_t a, uint64_t b) {
    (void)es;
    int sh = 64 - nbits;
    int64_t ia = (int64_t)(a << sh) >> sh, ib = (int64_t)(b << sh) >> sh;
    return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

/* posit.cpp:243-260 + 502-508. */
uint64_t po_from_float64(int nbits, int es, double x) {
    if (x == 0.0) return 0;
    if (!isfinite(x)) return nar_of(nbits);
    uint64_t b;
    memcpy(&b, &x, 8);
    int neg = (int)(b >> 63);
    int be = (int)((b >> 52) & 0x7FF);
    uint64_t mant = b & ((((uint64_t)1) << 52) - 1);
    uint64_t sig;
    int scale;
    if (be == 0) {
        int lead = __builtin_clzll(mant);
        sig = mant << lead;
        scale = -1023 - (lead - 11);
    } else {
        sig = ((((uint64_t)1) << 52) | mant) << 11;
        scale = be - 1023;
    }
    return po_pack_round(nbits, es, neg, scale, sig, 0);
}

double po_to_float64(int nbits, int es, uint64_t code) {
    po_unpacked u = po_unpack(nbits, es, code);
    if (u.cls == 0) return 0.0;
    if (u.cls == 1) return NAN;
    double v = ldexp((double)(u.sig >> 11), u.scale - 52) +
               ldexp((double)(u.sig & 2047), u.scale - 63);
    return u.neg ? -v : v;
}

uint64_t po_ldexp(int nbits, int es, uint64_t code, int k) {
    po_unpacked u = po_unpack(nbits, es, code);
    if (u.cls != 2) return code;
    long s = (long)u.scale + k;
    int R = po_max_scale(nbits, es);
    if (s > R) s = R;
    if (s < -R - 1) s = -R - 1;
    return po_pack_round(nbits, es, u.neg, (int)s, u.sig, 0);
}

uint64_t po_round_to_int(int nbits, int es, uint64_t code) {
    po_unpacked u = po_unpack(nbits, es, code);
    if (u.cls != 2) return code;
    if (u.scale >= 63) return code;
    if (u.scale < -1) return 0;
    if (u.scale == -1) { /* |v| in [1/2, 1): exactly 1/2 ties to 0 */
        if (u.sig == ((uint64_t)1 << 63)) return 0;
        return po_pack_round(nbits, es, u.neg, 0, (uint64_t)1 << 63, 0);
    }
    int fb = 63 - u.scale;
    uint64_t ip = fb >= 64 ? 0 : u.sig >> fb;
    uint64_t rem = u.sig & ((((uint64_t)1) << fb) - 1);
    uint64_t half = ((uint64_t)1) << (fb - 1);
    if (rem > half || (rem == half && (ip & 1))) ++ip;
    int lead = __builtin_clzll(ip);
    return po_pack_round(nbits, es, u.neg, 63 - lead, ip << lead, 0);
}

int64_t po_to_int64(int nbits, int es, uint64_t code) {
    po_unpacked u = po_unpack(nbits, es, code);
    if (u.cls != 2 || u.scale < 0) return 0;
    if (u.scale >= 62) return u.neg ? INT64_MIN : INT64_MAX;
    int64_t mag = (int64_t)(u.sig >> (63 - u.scale));
    return u.neg ? -mag : mag;
}

uint64_t po_from_int64(int nbits, int es, int64_t v) {
    if (v == 0) return 0;
    int neg = v < 0;
    uint64_t mag = neg ? (~(uint64_t)v + 1) : (uint64_t)v;
    int lead = __builtin_clzll(mag);
    return po_pack_round(nbits, es, neg, 63 - lead, mag << lead, 0);
}

#define OP_ADD(a, b) po_scalar_op(nbits, es, 0, (a), (b))
#define OP_SUB(a, b) po_scalar_op(nbits, es, 1, (a), (b))
#define OP_MUL(a, b) po_scalar_op(nbits, es, 2, (a), (b))
#define OP_DIV(a, b) po_scalar_op(nbits, es, 3, (a), (b))

/* posit_math.cpp:67-85: k = round(x*log2e); r = x - k*ln2; degree-10 Horner
 * in posit ops with coefficients from_float64(1/k!); ldexp by k. */
uint64_t po_exp(int nbits, int es, uint64_t x) {
    uint64_t nar = nar_of(nbits);
    x &= pmask(nbits);
    if (x == nar) return x;
    if (x == 0) return po_from_int64(nbits, es, 1);
    const int R = po_max_scale(nbits, es);
    uint64_t log2e = po_from_float64(nbits, es, 1.4426950408889634);
    uint64_t ln2 = po_from_float64(nbits, es, 0.6931471805599453);
    uint64_t coeff[11];
    double fact = 1.0;
    for (int k = 0; k <= 10; ++k) {
        if (k > 0) fact *= k;
        coeff[k] = po_from_float64(nbits, es, 1.0 / fact);
    }
    uint64_t kp = po_round_to_int(nbits, es, OP_MUL(x, log2e));
    int64_t k = po_to_int64(nbits, es, kp);
    if (k > R) return nar - 1;
    if (k < -R - 1) return 1;
    uint64_t r = OP_SUB(x, OP_MUL(kp, ln2));
    uint64_t p = coeff[10];
    for (int i = 9; i >= 0; --i) p = OP_ADD(OP_MUL(p, r), coeff[i]);
    return po_ldexp(nbits, es, p, (int)k);
}

/* posit_math.cpp:87-107: m = x*2^-s in [1,2) (halved once if >= 1.5),
 * log m = 2 atanh(t), t = (m-1)/(m+1), 8-term odd series in posit ops. */
uint64_t po_log(int nbits, int es, uint64_t x) {
    uint64_t nar = nar_of(nbits), m = pmask(nbits);
    x &= m;
    if (x == nar || x == 0 || ((x >> (nbits - 1)) & 1)) return nar;
    uint64_t one = po_from_int64(nbits, es, 1), two = po_from_int64(nbits, es, 2);
    uint64_t ln2 = po_from_float64(nbits, es, 0.6931471805599453);
    uint64_t three_halves = po_from_float64(nbits, es, 1.5);
    uint64_t lc[8];
    for (int k = 0; k < 8; ++k) lc[k] = po_from_float64(nbits, es, 1.0 / (2 * k + 1));
    po_unpacked u = po_unpack(nbits, es, x);
    int s = u.scale;
    uint64_t mm = po_ldexp(nbits, es, x, -s);
    if (po_compare(nbits, es, mm, three_halves) >= 0) {
        mm = po_ldexp(nbits, es, mm, -1);
        s += 1;
    }
    uint64_t t = OP_DIV(OP_SUB(mm, one), OP_ADD(mm, one));
    uint64_t uu = OP_MUL(t, t);
    uint64_t inner = lc[7];
    for (int i = 6; i >= 0; --i) inner = OP_ADD(OP_MUL(inner, uu), lc[i]);
    uint64_t logm = OP_MUL(two, OP_MUL(t, inner));
    return OP_ADD(OP_MUL(po_from_int64(nbits, es, s), ln2), logm);
}

/* ------------------------------------------------------- tensor kernels */

/* Decoded operand in integer-image form X = x * 2^R (exact integer). */
typedef struct {
    uint64_t sig;  /* fraction-bit integer significand (0 for zero) */
    int pos;       /* X = sig << pos */
    int neg, nar;
} xform;

typedef struct {
    int nbits, es, R, W;
    int fast; /* X fits int64 and products/sums fit 128-bit wrapping */
} fmtinfo;

static fmtinfo finfo(int nbits, int es) {
    fmtinfo f;
    f.nbits = nbits;
    f.es = es;
    f.R = po_max_scale(nbits, es);
    f.W = po_quire_bits(nbits, es);
    f.fast = (2 * f.R <= 62) && f.W <= 128;
    return f;
}

static xform xdecode(const fmtinfo* f, uint64_t code) {
    xform x = {0, 0, 0, 0};
    po_unpacked u = po_unpack(f->nbits, f->es, code);
    if (u.cls == 1) { x.nar = 1; return x; }
    if (u.cls == 0) return x;
    x.neg = u.neg;
    x.sig = ((uint64_t)1 << u.fbits) | u.frac;
    x.pos = (u.scale - u.fbits) + f->R;
    return x;
}

static xform* xdecode_all(const fmtinfo* f, const uint64_t* codes, int64_t n) {
    xform* v = (xform*)malloc(sizeof(xform) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) v[i] = xdecode(f, codes[i]);
    return v;
}

typedef struct {
    int nar;
    u128 a;  /* fast path: the quire mod 2^128 (masked to W at read-out) */
    wide w;  /* generic path */
} acc_t;

static void acc_clear(acc_t* q) { q->nar = 0; q->a = 0; wide_zero(&q->w); }

static void acc_prod(const fmtinfo* f, acc_t* q, const xform* a, const xform* b) {
    if (a->nar | b->nar) { q->nar = 1; return; }
    if (a->sig == 0 || b->sig == 0) return;
    int neg = a->neg ^ b->neg;
    if (f->fast) {
        i128 xa = (i128)(int64_t)(a->sig << a->pos), xb = (i128)(int64_t)(b->sig << b->pos);
        u128 p = (u128)(xa * xb);
        q->a = neg ? q->a - p : q->a + p;
    } else {
        wide_addsub(&q->w, (u128)a->sig * b->sig, a->pos + b->pos, neg);
    }
}

/* accumulate_value: X * 2^R in LSB-2^-2R units. */
static void acc_value(const fmtinfo* f, acc_t* q, const xform* a) {
    if (a->nar) { q->nar = 1; return; }
    if (a->sig == 0) return;
    if (f->fast) {
        u128 p = (u128)a->sig << (a->pos + f->R);
        q->a = a->neg ? q->a - p : q->a + p;
    } else {
        wide_addsub(&q->w, (u128)a->sig, a->pos + f->R, a->neg);
    }
}

static uint64_t acc_round(const fmtinfo* f, const acc_t* q) {
    if (q->nar) return nar_of(f->nbits);
    if (f->fast) {
        wide w;
        wide_zero(&w);
        w.w[0] = (uint64_t)q->a;
        w.w[1] = (uint64_t)(q->a >> 64);
        return wide_round(f->nbits, f->es, &w, f->W, -2 * f->R);
    }
    return wide_round(f->nbits, f->es, &q->w, f->W, -2 * f->R);
}

static int fmt_ok(int nbits, int es) { return nbits >= 2 && nbits <= 32 && es >= 0 && es <= 4; }

/* matmul_quire, tensor_ops.cpp:166-185. */
int po_matmul(int nbits, int es, const uint64_t* A, const uint64_t* B, uint64_t* C,
              int64_t m, int64_t k, int64_t n) {
    if (!fmt_ok(nbits, es)) return 1;
    fmtinfo f = finfo(nbits, es);
    if (k == 0) { memset(C, 0, sizeof(uint64_t) * (size_t)(m * n)); return 0; }
    xform* a = xdecode_all(&f, A, m * k);
    xform* b = xdecode_all(&f, B, k * n);
    acc_t q;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            acc_clear(&q);
            for (int64_t t = 0; t < k; ++t) acc_prod(&f, &q, &a[i * k + t], &b[t * n + j]);
            C[i * n + j] = acc_round(&f, &q);
        }
    free(a);
    free(b);
    return 0;
}

/* conv_quire + pad_nchw, tensor_ops.cpp:189-297: zero padding contributes
 * nothing, so out-of-range taps are skipped; bias goes inside the quire. */
int po_conv2d(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H,
              int64_t W, const uint64_t* w, int64_t F, int64_t KH, int64_t KW,
              const uint64_t* bias, int stride, int pad, uint64_t* y) {
    if (!fmt_ok(nbits, es) || stride < 1 || pad < 0) return 1;
    int64_t PH = H + 2 * pad, PW = W + 2 * pad;
    if (PH < KH || PW < KW) return 1;
    int64_t OH = (PH - KH) / stride + 1, OW = (PW - KW) / stride + 1;
    fmtinfo f = finfo(nbits, es);
    xform* xv = xdecode_all(&f, x, N * C * H * W);
    xform* wv = xdecode_all(&f, w, F * C * KH * KW);
    xform* bv = bias ? xdecode_all(&f, bias, F) : NULL;
    acc_t q;
    for (int64_t nn = 0; nn < N; ++nn)
        for (int64_t ff = 0; ff < F; ++ff)
            for (int64_t oy = 0; oy < OH; ++oy)
                for (int64_t ox = 0; ox < OW; ++ox) {
                    acc_clear(&q);
                    for (int64_t c = 0; c < C; ++c)
                        for (int64_t ky = 0; ky < KH; ++ky)
                            for (int64_t kx = 0; kx < KW; ++kx) {
                                int64_t iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
                                const xform* wt = &wv[((ff * C + c) * KH + ky) * KW + kx];
                                if (iy < 0 || iy >= H || ix < 0 || ix >= W) {
                                    /* padded zero: NaR weight still poisons (quire.hpp:55) */
                                    if (wt->nar) q.nar = 1;
                                    continue;
                                }
                                acc_prod(&f, &q, &xv[((nn * C + c) * H + iy) * W + ix], wt);
                            }
                    if (bv) acc_value(&f, &q, &bv[ff]);
                    y[((nn * F + ff) * OH + oy) * OW + ox] = acc_round(&f, &q);
                }
    free(xv);
    free(wv);
    free(bv);
    return 0;
}

/* conv2d_input_grad, tensor_ops.cpp:527-574 (padded positions computed then
 * cropped == computing the interior positions directly). */
int po_conv2d_input_grad(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                         int64_t OH, int64_t OW, const uint64_t* w, int64_t C, int64_t KH,
                         int64_t KW, int64_t H, int64_t W, int stride, int pad,
                         uint64_t* dx) {
    if (!fmt_ok(nbits, es) || stride < 1 || pad < 0) return 1;
    fmtinfo f = finfo(nbits, es);
    xform* dv = xdecode_all(&f, dy, N * F * OH * OW);
    xform* wv = xdecode_all(&f, w, F * C * KH * KW);
    acc_t q;
    for (int64_t nn = 0; nn < N; ++nn)
        for (int64_t c = 0; c < C; ++c)
            for (int64_t y0 = 0; y0 < H; ++y0)
                for (int64_t x0 = 0; x0 < W; ++x0) {
                    int64_t iy = y0 + pad, ix = x0 + pad;
                    acc_clear(&q);
                    for (int64_t ff = 0; ff < F; ++ff)
                        for (int64_t ky = 0; ky < KH; ++ky) {
                            int64_t ty = iy - ky;
                            if (ty < 0 || ty % stride) continue;
                            int64_t oy = ty / stride;
                            if (oy >= OH) continue;
                            for (int64_t kx = 0; kx < KW; ++kx) {
                                int64_t tx = ix - kx;
                                if (tx < 0 || tx % stride) continue;
                                int64_t ox = tx / stride;
                                if (ox >= OW) continue;
                                acc_prod(&f, &q, &dv[((nn * F + ff) * OH + oy) * OW + ox],
                                         &wv[((ff * C + c) * KH + ky) * KW + kx]);
                            }
                        }
                    dx[((nn * C + c) * H + y0) * W + x0] = acc_round(&f, &q);
                }
    free(dv);
    free(wv);
    return 0;
}

/* conv2d_weight_grad, tensor_ops.cpp:576-603: a batch reduction. */
int po_conv2d_weight_grad(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                          int64_t OH, int64_t OW, const uint64_t* x, int64_t C, int64_t H,
                          int64_t W, int64_t KH, int64_t KW, int stride, int pad,
                          uint64_t* dw) {
    if (!fmt_ok(nbits, es) || stride < 1 || pad < 0) return 1;
    fmtinfo f = finfo(nbits, es);
    xform* dv = xdecode_all(&f, dy, N * F * OH * OW);
    xform* xv = xdecode_all(&f, x, N * C * H * W);
    acc_t q;
    for (int64_t ff = 0; ff < F; ++ff)
        for (int64_t c = 0; c < C; ++c)
            for (int64_t ky = 0; ky < KH; ++ky)
                for (int64_t kx = 0; kx < KW; ++kx) {
                    acc_clear(&q);
                    for (int64_t nn = 0; nn < N; ++nn)
                        for (int64_t oy = 0; oy < OH; ++oy)
                            for (int64_t ox = 0; ox < OW; ++ox) {
                                int64_t iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
                                const xform* d = &dv[((nn * F + ff) * OH + oy) * OW + ox];
                                if (iy < 0 || iy >= H || ix < 0 || ix >= W) {
                                    /* padded zero: a NaR dy still poisons */
                                    if (d->nar) q.nar = 1;
                                    continue;
                                }
                                acc_prod(&f, &q, d, &xv[((nn * C + c) * H + iy) * W + ix]);
                            }
                    dw[((ff * C + c) * KH + ky) * KW + kx] = acc_round(&f, &q);
                }
    free(dv);
    free(xv);
    return 0;
}

/* conv2d_bias_grad, tensor_ops.cpp:605-618 (gather_quire_sum :353-365). */
int po_conv2d_bias_grad(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                        int64_t OH, int64_t OW, uint64_t* db) {
    if (!fmt_ok(nbits, es)) return 1;
    fmtinfo f = finfo(nbits, es);
    acc_t q;
    for (int64_t ff = 0; ff < F; ++ff) {
        acc_clear(&q);
        for (int64_t nn = 0; nn < N; ++nn)
            for (int64_t o = 0; o < OH * OW; ++o) {
                xform d = xdecode(&f, dy[(nn * F + ff) * OH * OW + o]);
                acc_value(&f, &q, &d);
            }
        db[ff] = acc_round(&f, &q);
    }
    return 0;
}

/* column_sum, tensor_ops.cpp:722-731. */
int po_column_sum(int nbits, int es, const uint64_t* x, int64_t B, int64_t N, uint64_t* out) {
    if (!fmt_ok(nbits, es)) return 1;
    fmtinfo f = finfo(nbits, es);
    acc_t q;
    for (int64_t j = 0; j < N; ++j) {
        acc_clear(&q);
        for (int64_t i = 0; i < B; ++i) {
            xform d = xdecode(&f, x[i * N + j]);
            acc_value(&f, &q, &d);
        }
        out[j] = acc_round(&f, &q);
    }
    return 0;
}

/* maxpool2d, tensor_ops.cpp:620-656: first strictly-greater element in
 * (ky,kx) scan order wins; argmax is the flat input index. */
int po_maxpool2d(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H,
                 int64_t W, int k, int stride, uint64_t* y, int64_t* argmax) {
    if (H < k || W < k) return 1;
    int64_t OH = (H - k) / stride + 1, OW = (W - k) / stride + 1;
    for (int64_t nc = 0; nc < N * C; ++nc)
        for (int64_t oy = 0; oy < OH; ++oy)
            for (int64_t ox = 0; ox < OW; ++ox) {
                int64_t base = nc * H * W;
                int64_t best = base + oy * stride * W + ox * stride;
                for (int ky = 0; ky < k; ++ky)
                    for (int kx = 0; kx < k; ++kx) {
                        int64_t idx = base + (oy * stride + ky) * W + ox * stride + kx;
                        if (po_compare(nbits, es, x[idx], x[best]) > 0) best = idx;
                    }
                y[(nc * OH + oy) * OW + ox] = x[best];
                argmax[(nc * OH + oy) * OW + ox] = best;
            }
    return 0;
}

/* maxpool2d_backward, tensor_ops.cpp:658-670: dx[argmax] = add(dx, dy). */
int po_maxpool2d_backward(int nbits, int es, const uint64_t* dy, int64_t ny,
                          const int64_t* argmax, int64_t nx, uint64_t* dx) {
    memset(dx, 0, sizeof(uint64_t) * (size_t)nx);
    for (int64_t i = 0; i < ny; ++i) {
        int64_t t = argmax[i];
        if (t < 0 || t >= nx) return 1;
        dx[t] = po_scalar_op(nbits, es, 0, dx[t], dy[i]);
    }
    return 0;
}

int po_convert_tensor(int sn, int se, int dn, int de, const uint64_t* x, int64_t n,
                      uint64_t* y) {
    for (int64_t i = 0; i < n; ++i)
        y[i] = (sn == dn && se == de) ? x[i] : po_convert(sn, se, dn, de, x[i]);
    return 0;
}

/* ------------------------------------------------ training-step semantics */

void po_ew(int nbits, int es, int op, const uint64_t* a, const uint64_t* b, uint64_t* out,
           int64_t n) {
    for (int64_t i = 0; i < n; ++i) out[i] = po_scalar_op(nbits, es, op, a[i], b[i]);
}

void po_relu_fwd(int nbits, int es, const uint64_t* x, uint64_t* y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] = po_compare(nbits, es, x[i], 0) > 0 ? x[i] : 0;
}

void po_relu_bwd(int x_nbits, int x_es, const uint64_t* x, const uint64_t* dy, uint64_t* dx,
                 int64_t n) {
    for (int64_t i = 0; i < n; ++i) dx[i] = po_compare(x_nbits, x_es, x[i], 0) > 0 ? dy[i] : 0;
}

/* m = max z (signed-pattern compare); e_j =
 * exp(sub(z_j, m)); S = quire sum of e_j rounded once; p_j = div(e_j, S);
 * loss_i = sub(log(S), sub(z_y, m)); batch loss = quire sum of loss_i rounded
 * once then ldexp by -log2(B); dlogits = ldexp(sub(p_j, [j==y]), -log2(B)). */
uint64_t po_softmax_xent(int nbits, int es, const uint64_t* logits, const int32_t* labels,
                         int64_t B, int64_t C, int log2_batch, uint64_t* dlogits,
                         uint64_t* loss_rows) {
    return po_softmax_xent_scaled(nbits, es, logits, labels, B, C, log2_batch, 0, dlogits,
                                  loss_rows);
}

/* Loss scaling (SPEC "scale_gradients"): the logit
 * gradient carries an extra 2^s, dlogits = ldexp(p - [j==y], s - log2 B); the
 * loss itself is not scaled. */
uint64_t po_softmax_xent_scaled(int nbits, int es, const uint64_t* logits, const int32_t* labels,
                                int64_t B, int64_t C, int log2_batch, int grad_scale_log2,
                                uint64_t* dlogits, uint64_t* loss_rows) {
    const uint64_t one = po_from_int64(nbits, es, 1);
    po_quire* tot = po_quire_new(nbits, es);
    po_quire* q = po_quire_new(nbits, es);
    for (int64_t i = 0; i < B; ++i) {
        const uint64_t* z = logits + i * C;
        uint64_t m = z[0];
        for (int64_t j = 1; j < C; ++j)
            if (po_compare(nbits, es, z[j], m) > 0) m = z[j];
        po_quire_clear(q);
        for (int64_t j = 0; j < C; ++j) po_quire_add_posit(q, po_exp(nbits, es, OP_SUB(z[j], m)));
        const uint64_t S = po_quire_to_posit(q);
        const int32_t y = labels[i];
        for (int64_t j = 0; j < C; ++j) {
            const uint64_t p = OP_DIV(po_exp(nbits, es, OP_SUB(z[j], m)), S);
            dlogits[i * C + j] =
                po_ldexp(nbits, es, OP_SUB(p, j == y ? one : 0), grad_scale_log2 - log2_batch);
        }
        loss_rows[i] = OP_SUB(po_log(nbits, es, S), OP_SUB(z[y], m));
        po_quire_add_posit(tot, loss_rows[i]);
    }
    const uint64_t loss = po_ldexp(nbits, es, po_quire_to_posit(tot), -log2_batch);
    po_quire_free(q);
    po_quire_free(tot);
    return loss;
}

void po_sgd(int opt_nbits, int opt_es, uint64_t* w, int g_nbits, int g_es, const uint64_t* g,
            int64_t n, uint64_t lr) {
    po_sgd_scaled(opt_nbits, opt_es, w, g_nbits, g_es, g, n, lr, 0);
}

/* Loss-scaled SGD: the gradient is unscaled in the optimizer format,
 * g_opt = ldexp(convert(g), -s), then w = sub(w, mul(lr, g_opt)). */
void po_sgd_scaled(int opt_nbits, int opt_es, uint64_t* w, int g_nbits, int g_es,
                   const uint64_t* g, int64_t n, uint64_t lr, int grad_scale_log2) {
    for (int64_t i = 0; i < n; ++i) {
        uint64_t gg = po_convert(g_nbits, g_es, opt_nbits, opt_es, g[i]);
        if (grad_scale_log2 != 0) gg = po_ldexp(opt_nbits, opt_es, gg, -grad_scale_log2);
        w[i] = po_scalar_op(opt_nbits, opt_es, 1, w[i],
                            po_scalar_op(opt_nbits, opt_es, 2, lr, gg));
    }
}

/* Round W-bit quire words (little-endian limbs, two's complement) once --
 * Quire::to_posit on an externally summed quire (data-parallel reduction). */
uint64_t po_round_words(int nbits, int es, const uint64_t* words, int nwords) {
    wide w;
    wide_zero(&w);
    for (int i = 0; i < nwords && i < WL; ++i) w.w[i] = words[i];
    return wide_round(nbits, es, &w, po_quire_bits(nbits, es), -2 * po_max_scale(nbits, es));
}

/* ------------------------------------------- non-quire sequential kernels */
/* matmul_seq / conv_seq / gather_seq(_sum), tensor_ops.cpp:145-164, 232-264,
 * 302-335: one correctly rounded multiply and add per term, in order. */

#define SEQ_ACC(acc, first, p) do { acc = first ? (p) : OP_ADD(acc, (p)); first = 0; } while (0)

int po_matmul_seq(int nbits, int es, const uint64_t* A, const uint64_t* B, uint64_t* C,
                  int64_t m, int64_t k, int64_t n) {
    if (!fmt_ok(nbits, es)) return 1;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            if (k == 0) { C[i * n + j] = 0; continue; }
            uint64_t acc = OP_MUL(A[i * k], B[j]);
            for (int64_t t = 1; t < k; ++t) acc = OP_ADD(acc, OP_MUL(A[i * k + t], B[t * n + j]));
            C[i * n + j] = acc;
        }
    return 0;
}

int po_conv2d_seq(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H, int64_t W,
                  const uint64_t* w, int64_t F, int64_t KH, int64_t KW, const uint64_t* bias,
                  int stride, int pad, uint64_t* y) {
    if (!fmt_ok(nbits, es) || stride < 1 || pad < 0) return 1;
    int64_t OH = (H + 2 * pad - KH) / stride + 1, OW = (W + 2 * pad - KW) / stride + 1;
    for (int64_t nn = 0; nn < N; ++nn)
        for (int64_t ff = 0; ff < F; ++ff)
            for (int64_t oy = 0; oy < OH; ++oy)
                for (int64_t ox = 0; ox < OW; ++ox) {
                    uint64_t acc = 0;
                    int first = 1;
                    for (int64_t c = 0; c < C; ++c)
                        for (int64_t ky = 0; ky < KH; ++ky)
                            for (int64_t kx = 0; kx < KW; ++kx) {
                                int64_t iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
                                uint64_t xv = (iy < 0 || iy >= H || ix < 0 || ix >= W)
                                                  ? 0 : x[((nn * C + c) * H + iy) * W + ix];
                                uint64_t p = OP_MUL(xv, w[((ff * C + c) * KH + ky) * KW + kx]);
                                SEQ_ACC(acc, first, p);
                            }
                    if (bias) acc = OP_ADD(acc, bias[ff]);
                    y[((nn * F + ff) * OH + oy) * OW + ox] = acc;
                }
    return 0;
}

int po_conv2d_input_grad_seq(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                             int64_t OH, int64_t OW, const uint64_t* w, int64_t C, int64_t KH,
                             int64_t KW, int64_t H, int64_t W, int stride, int pad, uint64_t* dx) {
    if (!fmt_ok(nbits, es) || stride < 1 || pad < 0) return 1;
    for (int64_t nn = 0; nn < N; ++nn)
        for (int64_t c = 0; c < C; ++c)
            for (int64_t y0 = 0; y0 < H; ++y0)
                for (int64_t x0 = 0; x0 < W; ++x0) {
                    int64_t iy = y0 + pad, ix = x0 + pad;
                    uint64_t acc = 0;
                    int first = 1;
                    for (int64_t ff = 0; ff < F; ++ff)
                        for (int64_t ky = 0; ky < KH; ++ky) {
                            int64_t ty = iy - ky;
                            if (ty < 0 || ty % stride) continue;
                            int64_t oy = ty / stride;
                            if (oy >= OH) continue;
                            for (int64_t kx = 0; kx < KW; ++kx) {
                                int64_t tx = ix - kx;
                                if (tx < 0 || tx % stride) continue;
                                int64_t ox = tx / stride;
                                if (ox >= OW) continue;
                                uint64_t p = OP_MUL(dy[((nn * F + ff) * OH + oy) * OW + ox],
                                                    w[((ff * C + c) * KH + ky) * KW + kx]);
                                SEQ_ACC(acc, first, p);
                            }
                        }
                    dx[((nn * C + c) * H + y0) * W + x0] = acc;
                }
    return 0;
}

int po_conv2d_weight_grad_seq(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                              int64_t OH, int64_t OW, const uint64_t* x, int64_t C, int64_t H,
                              int64_t W, int64_t KH, int64_t KW, int stride, int pad, uint64_t* dw) {
    if (!fmt_ok(nbits, es) || stride < 1 || pad < 0) return 1;
    for (int64_t ff = 0; ff < F; ++ff)
        for (int64_t c = 0; c < C; ++c)
            for (int64_t ky = 0; ky < KH; ++ky)
                for (int64_t kx = 0; kx < KW; ++kx) {
                    uint64_t acc = 0;
                    int first = 1;
                    for (int64_t nn = 0; nn < N; ++nn)
                        for (int64_t oy = 0; oy < OH; ++oy)
                            for (int64_t ox = 0; ox < OW; ++ox) {
                                int64_t iy = oy * stride + ky - pad, ix = ox * stride + kx - pad;
                                uint64_t xv = (iy < 0 || iy >= H || ix < 0 || ix >= W)
                                                  ? 0 : x[((nn * C + c) * H + iy) * W + ix];
                                uint64_t p = OP_MUL(dy[((nn * F + ff) * OH + oy) * OW + ox], xv);
                                SEQ_ACC(acc, first, p);
                            }
                    dw[((ff * C + c) * KH + ky) * KW + kx] = acc;
                }
    return 0;
}

int po_bias_grad_seq(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F, int64_t P,
                     uint64_t* db) {
    if (!fmt_ok(nbits, es)) return 1;
    for (int64_t ff = 0; ff < F; ++ff) {
        uint64_t acc = 0;
        int first = 1;
        for (int64_t nn = 0; nn < N; ++nn)
            for (int64_t p = 0; p < P; ++p) SEQ_ACC(acc, first, dy[(nn * F + ff) * P + p]);
        db[ff] = acc;
    }
    return 0;
}

/* tanh_posit / sigmoid_posit, posit_math.cpp:109-130 (posit-op sequences). */
uint64_t po_tanh(int nbits, int es, uint64_t x) {
    uint64_t m = pmask(nbits), nar = nar_of(nbits);
    x &= m;
    if (x == nar || x == 0) return x;
    int neg = (int)((x >> (nbits - 1)) & 1);
    uint64_t ax = neg ? ((~x + 1) & m) : x;
    uint64_t one = po_from_int64(nbits, es, 1);
    uint64_t t2 = po_ldexp(nbits, es, ax, 1);
    uint64_t t = po_exp(nbits, es, (~t2 + 1) & m);
    uint64_t r = OP_DIV(OP_SUB(one, t), OP_ADD(one, t));
    return neg ? ((~r + 1) & m) : r;
}

uint64_t po_sigmoid(int nbits, int es, uint64_t x) {
    uint64_t m = pmask(nbits), nar = nar_of(nbits);
    x &= m;
    if (x == nar) return x;
    uint64_t one = po_from_int64(nbits, es, 1);
    if (!((x >> (nbits - 1)) & 1)) {
        uint64_t t = po_exp(nbits, es, (~x + 1) & m);
        return OP_DIV(one, OP_ADD(one, t));
    }
    uint64_t t = po_exp(nbits, es, x);
    return OP_DIV(t, OP_ADD(one, t));
}

/* avgpool2d / avgpool2d_backward, tensor_ops.cpp:672-720. */
int po_avgpool2d(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H, int64_t W,
                 int k, int stride, int use_quire, uint64_t recip, uint64_t* y) {
    if (H < k || W < k) return 1;
    int64_t OH = (H - k) / stride + 1, OW = (W - k) / stride + 1;
    for (int64_t nc = 0; nc < N * C; ++nc)
        for (int64_t oy = 0; oy < OH; ++oy)
            for (int64_t ox = 0; ox < OW; ++ox) {
                uint64_t sum = 0;
                if (use_quire) {
                    po_quire* q = po_quire_new(nbits, es);
                    for (int ky = 0; ky < k; ++ky)
                        for (int kx = 0; kx < k; ++kx)
                            po_quire_add_posit(q, x[nc * H * W + (oy * stride + ky) * W + ox * stride + kx]);
                    sum = po_quire_to_posit(q);
                    po_quire_free(q);
                } else {
                    int first = 1;
                    for (int ky = 0; ky < k; ++ky)
                        for (int kx = 0; kx < k; ++kx) {
                            uint64_t v = x[nc * H * W + (oy * stride + ky) * W + ox * stride + kx];
                            SEQ_ACC(sum, first, v);
                        }
                }
                y[(nc * OH + oy) * OW + ox] = OP_MUL(sum, recip);
            }
    return 0;
}

int po_avgpool2d_backward(int nbits, int es, const uint64_t* dy, int64_t N, int64_t C, int64_t H,
                          int64_t W, int k, int stride, uint64_t recip, uint64_t* dx) {
    int64_t OH = (H - k) / stride + 1, OW = (W - k) / stride + 1;
    memset(dx, 0, sizeof(uint64_t) * (size_t)(N * C * H * W));
    for (int64_t nc = 0; nc < N * C; ++nc)
        for (int64_t oy = 0; oy < OH; ++oy)
            for (int64_t ox = 0; ox < OW; ++ox) {
                uint64_t g = OP_MUL(dy[(nc * OH + oy) * OW + ox], recip);
                for (int ky = 0; ky < k; ++ky)
                    for (int kx = 0; kx < k; ++kx) {
                        int64_t t = nc * H * W + (oy * stride + ky) * W + ox * stride + kx;
                        dx[t] = OP_ADD(dx[t], g);
                    }
            }
    return 0;
}
