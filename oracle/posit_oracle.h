/* Plain-C restatement of the reference's posit/quire hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as the checker
 * -- never as the thing measured or shipped.  The product path
 * (paper_2105_00053_b200/) never links or calls it.
 *
 * Parity pinning: tests/test_oracle_pin.py checks every function here
 * against (a) the reference's own known-answer tests (proj/tests/
 * test_quire.cpp, test_tensor.cpp, test_posit.cpp), (b) committed golden
 * fixtures generated from the unmodified reference (tests/golden/,
 * tests/golden/make_golden.py), and (c) the reference library itself built
 * from its sources (oracle/_ref/libpnn_ref.so) on random inputs.
 *
 * Codes are right-aligned posit bit patterns in uint64 (reference
 * tensor.hpp:10-14).  Tensor functions implement the quire (use_quire=true)
 * semantics of proj/src/tensor_ops.cpp for nbits <= 32.
 */
#ifndef POSIT_ORACLE_H
#define POSIT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Format descriptor: posit.hpp:17-42. */
int po_max_scale(int nbits, int es);  /* R = (nbits-2) << es */
int po_quire_bits(int nbits, int es); /* W = 4R + nbits      */

/* detail::unpack, posit.cpp:67-91.  cls: 0 zero, 1 NaR, 2 finite. */
typedef struct {
    int cls, neg, scale, fbits;
    uint64_t sig;  /* normalized: bit 63 set */
    uint64_t frac; /* fbits-bit fraction field */
} po_unpacked;
po_unpacked po_unpack(int nbits, int es, uint64_t code);

/* DecodeTables::Fixed, posit_tables.cpp:43-64. */
void po_decode_fixed(int nbits, int es, uint64_t code, int32_t* lsb_scale, uint32_t* sig,
                     uint8_t* neg, uint8_t* nar);

/* detail::pack_round, posit.cpp:93-132. */
uint64_t po_pack_round(int nbits, int es, int neg, int scale, uint64_t sig, int sticky);

/* Scalar ops: posit.cpp:437-485 (op 0 add, 1 sub, 2 mul, 3 div). */
uint64_t po_scalar_op(int nbits, int es, int op, uint64_t a, uint64_t b);
uint64_t po_convert(int sn, int se, int dn, int de, uint64_t code); /* posit.cpp:487-495 */
int po_compare(int nbits, int es, uint64_t a, uint64_t b);          /* posit.cpp:514-520 */
uint64_t po_from_float64(int nbits, int es, double x);              /* posit.cpp:502-508 */
double po_to_float64(int nbits, int es, uint64_t code);             /* posit.cpp:228-236 */
uint64_t po_ldexp(int nbits, int es, uint64_t code, int k);         /* posit.cpp:522-532 */
uint64_t po_round_to_int(int nbits, int es, uint64_t code);         /* posit.cpp:534-555 */
int64_t po_to_int64(int nbits, int es, uint64_t code);              /* posit.cpp:557-563 */
uint64_t po_from_int64(int nbits, int es, int64_t v);               /* posit_math.cpp:51-57 */
uint64_t po_exp(int nbits, int es, uint64_t code);                  /* posit_math.cpp:67-85 */
uint64_t po_log(int nbits, int es, uint64_t code);                  /* posit_math.cpp:87-107 */

/* Quire as an opaque accumulator: quire.hpp:18-86, quire.cpp. */
typedef struct po_quire po_quire;
po_quire* po_quire_new(int nbits, int es);
void po_quire_free(po_quire* q);
void po_quire_clear(po_quire* q);
void po_quire_add_posit(po_quire* q, uint64_t a);
void po_quire_add_product(po_quire* q, uint64_t a, uint64_t b);
void po_quire_sub_product(po_quire* q, uint64_t a, uint64_t b);
uint64_t po_quire_to_posit(const po_quire* q);
/* Raw quire words (little-endian uint64 limbs, W bits, two's complement). */
int po_quire_words(const po_quire* q, uint64_t* out, int max_words, int* nar);

/* Non-quire sequential kernels (use_quire=false): tensor_ops.cpp:145-164,
 * 232-264, 302-335 -- one rounding per multiply and per add, in order. */
int po_matmul_seq(int nbits, int es, const uint64_t* A, const uint64_t* B, uint64_t* C,
                  int64_t m, int64_t k, int64_t n);
int po_conv2d_seq(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H, int64_t W,
                  const uint64_t* w, int64_t F, int64_t KH, int64_t KW, const uint64_t* bias,
                  int stride, int pad, uint64_t* y);
int po_conv2d_input_grad_seq(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                             int64_t OH, int64_t OW, const uint64_t* w, int64_t C, int64_t KH,
                             int64_t KW, int64_t H, int64_t W, int stride, int pad, uint64_t* dx);
int po_conv2d_weight_grad_seq(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                              int64_t OH, int64_t OW, const uint64_t* x, int64_t C, int64_t H,
                              int64_t W, int64_t KH, int64_t KW, int stride, int pad, uint64_t* dw);
int po_bias_grad_seq(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F, int64_t P,
                     uint64_t* db);

/* tanh_posit / sigmoid_posit (posit_math.cpp:109-130) and avg-pool
 * (tensor_ops.cpp:672-720) -- SURVEY.md §8f item 2. */
uint64_t po_tanh(int nbits, int es, uint64_t x);
uint64_t po_sigmoid(int nbits, int es, uint64_t x);
int po_avgpool2d(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H, int64_t W,
                 int k, int stride, int use_quire, uint64_t recip, uint64_t* y);
int po_avgpool2d_backward(int nbits, int es, const uint64_t* dy, int64_t N, int64_t C, int64_t H,
                          int64_t W, int k, int stride, uint64_t recip, uint64_t* dx);

/* Round externally summed W-bit quire words once (data-parallel reduction). */
uint64_t po_round_words(int nbits, int es, const uint64_t* words, int nwords);

/* Tensor kernels, quire mode (tensor_ops.cpp).  Return 0 on success. */
int po_matmul(int nbits, int es, const uint64_t* A, const uint64_t* B, uint64_t* C,
              int64_t m, int64_t k, int64_t n);
int po_conv2d(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H,
              int64_t W, const uint64_t* w, int64_t F, int64_t KH, int64_t KW,
              const uint64_t* bias, int stride, int pad, uint64_t* y);
int po_conv2d_input_grad(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                         int64_t OH, int64_t OW, const uint64_t* w, int64_t C, int64_t KH,
                         int64_t KW, int64_t H, int64_t W, int stride, int pad,
                         uint64_t* dx);
int po_conv2d_weight_grad(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                          int64_t OH, int64_t OW, const uint64_t* x, int64_t C, int64_t H,
                          int64_t W, int64_t KH, int64_t KW, int stride, int pad,
                          uint64_t* dw);
int po_conv2d_bias_grad(int nbits, int es, const uint64_t* dy, int64_t N, int64_t F,
                        int64_t OH, int64_t OW, uint64_t* db);
int po_column_sum(int nbits, int es, const uint64_t* x, int64_t B, int64_t N, uint64_t* out);
int po_maxpool2d(int nbits, int es, const uint64_t* x, int64_t N, int64_t C, int64_t H,
                 int64_t W, int k, int stride, uint64_t* y, int64_t* argmax);
int po_maxpool2d_backward(int nbits, int es, const uint64_t* dy, int64_t ny,
                          const int64_t* argmax, int64_t nx, uint64_t* dx);
int po_convert_tensor(int sn, int se, int dn, int de, const uint64_t* x, int64_t n,
                      uint64_t* y);

/* ---- training-step semantics the reference leaves open (placeholders in
 * layers.cpp / losses.cpp / optimizer.cpp), pinned per SURVEY.md Appendix A
 * and restated here as the single CPU definition the GPU step must match. */
/* Vector scalar op over n elements (op 0 add 1 sub 2 mul 3 div). */
void po_ew(int nbits, int es, int op, const uint64_t* a, const uint64_t* b, uint64_t* out,
           int64_t n);
/* A.2 ReLU: x > 0 ? x : 0 by signed-pattern compare (NaR sorts lowest -> 0). */
void po_relu_fwd(int nbits, int es, const uint64_t* x, uint64_t* y, int64_t n);
/* dx = x > 0 ? dy : 0 (x in the forward format, dy in the backward format). */
void po_relu_bwd(int x_nbits, int x_es, const uint64_t* x, const uint64_t* dy, uint64_t* dx,
                 int64_t n);
/* A.5 softmax cross-entropy in the loss format; returns the batch loss code. */
uint64_t po_softmax_xent(int nbits, int es, const uint64_t* logits, const int32_t* labels,
                         int64_t B, int64_t C, int log2_batch, uint64_t* dlogits,
                         uint64_t* loss_rows);
/* A.7 SGD: w = sub(w, mul(lr, convert(g -> opt))) in the optimizer format. */
void po_sgd(int opt_nbits, int opt_es, uint64_t* w, int g_nbits, int g_es, const uint64_t* g,
            int64_t n, uint64_t lr);
/* Loss scaling by 2^s: dlogits carry 2^s; the SGD
 * update unscales in the optimizer format, g = ldexp(convert(g), -s). */
uint64_t po_softmax_xent_scaled(int nbits, int es, const uint64_t* logits, const int32_t* labels,
                                int64_t B, int64_t C, int log2_batch, int grad_scale_log2,
                                uint64_t* dlogits, uint64_t* loss_rows);
void po_sgd_scaled(int opt_nbits, int opt_es, uint64_t* w, int g_nbits, int g_es,
                   const uint64_t* g, int64_t n, uint64_t lr, int grad_scale_log2);

/* ---- remaining SPEC layers (layers_oracle.c; semantics written there) ---- */
uint64_t po_sqrt(int nbits, int es, uint64_t x); /* posit_math.cpp:132-160 */
void po_act_fwd(int kind, int nbits, int es, const uint64_t* x, uint64_t* y, int64_t n);
void po_act_bwd(int kind, int fn, int fe, const uint64_t* y, int bn, int be, const uint64_t* dy,
                uint64_t* dx, int64_t n);
uint64_t po_dropout_bits(uint64_t seed, int64_t i);
void po_dropout(int nbits, int es, const uint64_t* x, uint64_t* y, int64_t n, uint64_t seed,
                uint32_t thresh, uint64_t scale);
uint64_t po_mse(int nbits, int es, const uint64_t* y, const uint64_t* t, int64_t n, int64_t G,
                int grad_scale_log2, uint64_t* grad);
void po_batchnorm_fwd(int fn, int fe, const uint64_t* x, int64_t N, int64_t C, int64_t HW,
                      const uint64_t* gamma, const uint64_t* beta, uint64_t eps, int training,
                      int on, int oe, uint64_t* run_mean, uint64_t* run_var, uint64_t mom,
                      uint64_t* y, uint64_t* xhat, uint64_t* inv_out);
void po_batchnorm_bwd(int fn, int fe, const uint64_t* xhat, const uint64_t* inv, int bn, int be,
                      const uint64_t* dy, int64_t N, int64_t C, int64_t HW,
                      const uint64_t* gamma_b, int gn, int ge, uint64_t* dx, uint64_t* dgamma,
                      uint64_t* dbeta);
void po_sgd_momentum(int on, int oe, uint64_t* w, uint64_t* v, int gn, int ge, const uint64_t* grad,
                     int64_t n, uint64_t lr, uint64_t mu, int grad_scale_log2);

#ifdef __cplusplus
}
#endif

#endif
