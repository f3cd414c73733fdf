/* Plain-C oracle for the remaining SPEC layers:
 * sqrt, tanh / sigmoid layers (forward + backward), dropout, MSE loss,
 * batch normalisation, SGD with momentum.
 *
 * TEST INFRASTRUCTURE ONLY (see posit_oracle.h): the product path never links
 * or calls this file.
 *
 * The reference has no layer code for these (proj/src/layers.cpp etc. are
 * placeholders); SPEC.md:326-332 / 342-344 / 351-353 say
 * what they compute, not how a posit implementation rounds.  The rounding
 * sequence chosen here is written out per function and mirrored op for op by
 * the device kernels (paper_2105_00053_b200/csrc/layers.cu).  Every scalar
 * step is one reference scalar op (posit.cpp:393-416, each exactly rounded);
 * every reduction is one quire (quire.hpp:18-81: exact, one rounding).
 * sqrt is the reference's sqrt_posit (posit_math.cpp:132-160), pinned to
 * the compiled reference by tests/test_layers_ext.py.
 */
#include <stdlib.h>
#include <string.h>

#include "posit_oracle.h"

typedef unsigned __int128 u128;

static uint64_t pmask_(int n) { return n >= 64 ? ~(uint64_t)0 : (((uint64_t)1 << n) - 1); }
static uint64_t nar_(int n) { return (uint64_t)1 << (n - 1); }

#define ADD(f, a, b) po_scalar_op((f)[0], (f)[1], 0, (a), (b))
#define SUB(f, a, b) po_scalar_op((f)[0], (f)[1], 1, (a), (b))
#define MUL(f, a, b) po_scalar_op((f)[0], (f)[1], 2, (a), (b))
#define DIV(f, a, b) po_scalar_op((f)[0], (f)[1], 3, (a), (b))
#define CVT(s, d, c) po_convert((s)[0], (s)[1], (d)[0], (d)[1], (c))

/* sqrt_posit, posit_math.cpp:132-160: correctly rounded square root.  The
 * value is sig * 2^(scale-63) = M * 2^(2q) with M = sig << j in [2^126,
 * 2^128); r = floor(sqrt(M)) in [2^63, 2^64) is found here bit by bit
 * (restoring method) rather than by the reference's Newton iteration -- the
 * floor root and the remainder are unique, so the rounding is the same. */
uint64_t po_sqrt(int nbits, int es, uint64_t x) {
    x &= pmask_(nbits);
    if (x == 0 || x == nar_(nbits)) return x;
    if ((x >> (nbits - 1)) & 1) return nar_(nbits);
    po_unpacked u = po_unpack(nbits, es, x);
    int j = (u.scale & 1) == 0 ? 63 : 64;
    u128 M = (u128)u.sig << j;
    int q = (u.scale - 63 - j) / 2;
    u128 rem = 0, root = 0;
    for (int i = 63; i >= 0; --i) { /* two bits of M per root bit */
        rem = (rem << 2) | (u128)((M >> (2 * i)) & 3);
        u128 t = (root << 2) | 1;
        root <<= 1;
        if (rem >= t) {
            rem -= t;
            root |= 1;
        }
    }
    return po_pack_round(nbits, es, 0, q + 63, (uint64_t)root, rem != 0);
}

/* ---- activation layers ("sigmoid_f/b; tanh_f/b") ------------
 * kind 1 tanh, 2 sigmoid.  Forward: y = tanh_posit / sigmoid_posit (x) in the
 * forward format.  Backward in the backward format b, from the forward
 * OUTPUT y (converted f -> b once):
 *   tanh:    dx = mul(dy, sub(1, mul(yb, yb)))
 *   sigmoid: dx = mul(dy, mul(yb, sub(1, yb)))                              */
void po_act_fwd(int kind, int nbits, int es, const uint64_t* x, uint64_t* y, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        y[i] = kind == 1 ? po_tanh(nbits, es, x[i]) : po_sigmoid(nbits, es, x[i]);
}

void po_act_bwd(int kind, int fn, int fe, const uint64_t* y, int bn, int be, const uint64_t* dy,
                uint64_t* dx, int64_t n) {
    const int f[2] = {fn, fe}, b[2] = {bn, be};
    const uint64_t one = po_from_int64(bn, be, 1);
    for (int64_t i = 0; i < n; ++i) {
        uint64_t yb = CVT(f, b, y[i]);
        uint64_t t = kind == 1 ? SUB(b, one, MUL(b, yb, yb)) : MUL(b, yb, SUB(b, one, yb));
        dx[i] = MUL(b, dy[i], t);
    }
}

/* ---- dropout ("seeded mask, scale 1/(1-p) at train time") ---
 * Counter-based mask: u = mix64(seed ^ (i * 0xD1B54A32D192ED03)) (the
 * splitmix64 finaliser), keep element i iff (u >> 32) >= thresh, thresh =
 * floor(p * 2^32).  y = keep ? mul(x, scale) : 0 with scale =
 * from_float64(1/(1-p)) in the tensor's format.  The backward is the same
 * function on dy with the scale quantised in the backward format (the mask
 * is recomputed from the seed, never stored). */
uint64_t po_dropout_bits(uint64_t seed, int64_t i) {
    uint64_t z = seed ^ ((uint64_t)i * 0xD1B54A32D192ED03ull);
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void po_dropout(int nbits, int es, const uint64_t* x, uint64_t* y, int64_t n, uint64_t seed,
                uint32_t thresh, uint64_t scale) {
    const int f[2] = {nbits, es};
    for (int64_t i = 0; i < n; ++i) {
        int keep = (uint32_t)(po_dropout_bits(seed, i) >> 32) >= thresh;
        y[i] = keep ? MUL(f, x[i], scale) : 0;
    }
}

/* ---- MSE loss (mean (y - t)^2, gradient 2(y - t)/N) -----
 * In the loss format, with G = the GLOBAL element count (from_int64(G)):
 *   d_i    = sub(y_i, t_i)
 *   loss   = div(round(quire sum d_i * d_i), G)
 *   grad_i = ldexp(mul(d_i, div(2, G)), grad_scale_log2)                    */
uint64_t po_mse(int nbits, int es, const uint64_t* y, const uint64_t* t, int64_t n, int64_t G,
                int grad_scale_log2, uint64_t* grad) {
    const int f[2] = {nbits, es};
    const uint64_t g = po_from_int64(nbits, es, G);
    const uint64_t c = DIV(f, po_from_int64(nbits, es, 2), g);
    po_quire* q = po_quire_new(nbits, es);
    for (int64_t i = 0; i < n; ++i) {
        uint64_t d = SUB(f, y[i], t[i]);
        po_quire_add_product(q, d, d);
        uint64_t gi = MUL(f, d, c);
        grad[i] = grad_scale_log2 ? po_ldexp(nbits, es, gi, grad_scale_log2) : gi;
    }
    uint64_t s = po_quire_to_posit(q);
    po_quire_free(q);
    return DIV(f, s, g);
}

/* ---- batch normalisation (per channel, running stats in the
 * optimizer format).  x [N,C,H,W] in the forward format f, M = N*H*W,
 * Mc = from_int64(M), eps = the caller's code in f.  Per channel c:
 *   mean   = div(round(quire sum x), Mc)
 *   d_i    = sub(x_i, mean)
 *   var    = div(round(quire sum d_i * d_i), Mc)        (biased)
 *   inv    = div(1, sqrt(add(var, eps)))
 *   xhat_i = mul(d_i, inv)
 *   y_i    = add(mul(gamma, xhat_i), beta)
 * Running statistics, optimizer format o, momentum code mom in o:
 *   rm = add(rm, mul(mom, sub(convert(mean), rm)))   (same for rv with var)
 * Eval mode (training = 0): mean / var are convert(rm / rv, o -> f) and the
 * running statistics are left alone.
 * Outputs: y, xhat (for the backward), inv[C]. */
void po_batchnorm_fwd(int fn, int fe, const uint64_t* x, int64_t N, int64_t C, int64_t HW,
                      const uint64_t* gamma, const uint64_t* beta, uint64_t eps, int training,
                      int on, int oe, uint64_t* run_mean, uint64_t* run_var, uint64_t mom,
                      uint64_t* y, uint64_t* xhat, uint64_t* inv_out) {
    const int f[2] = {fn, fe}, o[2] = {on, oe};
    const int64_t M = N * HW;
    const uint64_t Mc = po_from_int64(fn, fe, M), one = po_from_int64(fn, fe, 1);
    po_quire* q = po_quire_new(fn, fe);
    for (int64_t c = 0; c < C; ++c) {
        uint64_t mean, var;
        if (training) {
            po_quire_clear(q);
            for (int64_t n = 0; n < N; ++n)
                for (int64_t p = 0; p < HW; ++p) po_quire_add_posit(q, x[(n * C + c) * HW + p]);
            mean = DIV(f, po_quire_to_posit(q), Mc);
            po_quire_clear(q);
            for (int64_t n = 0; n < N; ++n)
                for (int64_t p = 0; p < HW; ++p) {
                    uint64_t d = SUB(f, x[(n * C + c) * HW + p], mean);
                    po_quire_add_product(q, d, d);
                }
            var = DIV(f, po_quire_to_posit(q), Mc);
            run_mean[c] = ADD(o, run_mean[c], MUL(o, mom, SUB(o, CVT(f, o, mean), run_mean[c])));
            run_var[c] = ADD(o, run_var[c], MUL(o, mom, SUB(o, CVT(f, o, var), run_var[c])));
        } else {
            mean = CVT(o, f, run_mean[c]);
            var = CVT(o, f, run_var[c]);
        }
        uint64_t inv = DIV(f, one, po_sqrt(fn, fe, ADD(f, var, eps)));
        inv_out[c] = inv;
        for (int64_t n = 0; n < N; ++n)
            for (int64_t p = 0; p < HW; ++p) {
                int64_t i = (n * C + c) * HW + p;
                uint64_t xh = MUL(f, SUB(f, x[i], mean), inv);
                xhat[i] = xh;
                y[i] = ADD(f, MUL(f, gamma[c], xh), beta[c]);
            }
    }
    po_quire_free(q);
}

/* Backward, backward format b, gradient format g; gamma_b = gamma in b.
 *   dgamma_c = round_g(quire sum convert(dy -> g) * convert(xhat -> g))
 *   dbeta_c  = round_g(quire sum convert(dy -> g))
 *   dxh_i    = mul(dy_i, gamma_b);   xh_i = convert(xhat_i, f -> b)
 *   s1 = div(round_b(quire sum dxh_i), Mb);  s2 = div(round_b(quire sum dxh_i * xh_i), Mb)
 *   dx_i     = mul(convert(inv, f -> b), sub(sub(dxh_i, s1), mul(xh_i, s2)))   */
void po_batchnorm_bwd(int fn, int fe, const uint64_t* xhat, const uint64_t* inv, int bn, int be,
                      const uint64_t* dy, int64_t N, int64_t C, int64_t HW,
                      const uint64_t* gamma_b, int gn, int ge, uint64_t* dx, uint64_t* dgamma,
                      uint64_t* dbeta) {
    const int f[2] = {fn, fe}, b[2] = {bn, be}, g[2] = {gn, ge};
    const int64_t M = N * HW;
    const uint64_t Mb = po_from_int64(bn, be, M);
    po_quire *qg = po_quire_new(gn, ge), *qb = po_quire_new(gn, ge);
    po_quire *q1 = po_quire_new(bn, be), *q2 = po_quire_new(bn, be);
    for (int64_t c = 0; c < C; ++c) {
        po_quire_clear(qg);
        po_quire_clear(qb);
        po_quire_clear(q1);
        po_quire_clear(q2);
        for (int64_t n = 0; n < N; ++n)
            for (int64_t p = 0; p < HW; ++p) {
                int64_t i = (n * C + c) * HW + p;
                uint64_t dyg = CVT(b, g, dy[i]);
                po_quire_add_product(qg, dyg, CVT(f, g, xhat[i]));
                po_quire_add_posit(qb, dyg);
                uint64_t dxh = MUL(b, dy[i], gamma_b[c]);
                po_quire_add_posit(q1, dxh);
                po_quire_add_product(q2, dxh, CVT(f, b, xhat[i]));
            }
        dgamma[c] = po_quire_to_posit(qg);
        dbeta[c] = po_quire_to_posit(qb);
        uint64_t s1 = DIV(b, po_quire_to_posit(q1), Mb), s2 = DIV(b, po_quire_to_posit(q2), Mb);
        uint64_t ib = CVT(f, b, inv[c]);
        for (int64_t n = 0; n < N; ++n)
            for (int64_t p = 0; p < HW; ++p) {
                int64_t i = (n * C + c) * HW + p;
                uint64_t xh = CVT(f, b, xhat[i]);
                uint64_t dxh = MUL(b, dy[i], gamma_b[c]);
                dx[i] = MUL(b, ib, SUB(b, SUB(b, dxh, s1), MUL(b, xh, s2)));
            }
    }
    po_quire_free(qg);
    po_quire_free(qb);
    po_quire_free(q1);
    po_quire_free(q2);
}

/* ---- SGD with momentum ("optional momentum buffer in
 * p_optimizer config"), optimizer format o:
 *   g = ldexp(convert(grad -> o), -grad_scale_log2)
 *   v = add(mul(mu, v), g)
 *   w = sub(w, mul(lr, v))
 * mu = 0 is not special-cased here: callers use po_sgd_scaled for it. */
void po_sgd_momentum(int on, int oe, uint64_t* w, uint64_t* v, int gn, int ge, const uint64_t* grad,
                     int64_t n, uint64_t lr, uint64_t mu, int grad_scale_log2) {
    const int o[2] = {on, oe}, g[2] = {gn, ge};
    for (int64_t i = 0; i < n; ++i) {
        uint64_t gi = CVT(g, o, grad[i]);
        if (grad_scale_log2) gi = po_ldexp(on, oe, gi, -grad_scale_log2);
        v[i] = ADD(o, MUL(o, mu, v[i]), gi);
        w[i] = SUB(o, w[i], MUL(o, lr, v[i]));
    }
}
