/* pnn_b200 -- C-ABI of the B200-native posit/quire kernels.
 *
 * Drop-in boundary for the reference's operator API
 * (/root/reference/proj/include/pnn/tensor_ops.hpp:17-61, quire.hpp:18-86).
 * Plain pointers, sizes and int status codes only; no C++ or torch types.
 *
 * Conventions (mirroring the reference):
 *   - A posit format is (nbits, es); every kernel implements the reference's
 *     use_quire=true path: one exact quire accumulation per output element,
 *     rounded once (tensor_ops.cpp header comment, lines 10-14).
 *   - Device entry points (suffix-free) take DEVICE pointers to PACKED codes:
 *     uint8_t per element for nbits <= 8, uint16_t for 9..16, row-major
 *     (NCHW activations, FCKK weights), plus a cudaStream_t passed as void*.
 *     They are asynchronous on that stream.
 *   - Host entry points (suffix _host) take HOST uint64_t code arrays -- the
 *     reference Tensor storage (tensor.hpp:10-14, one code per 64-bit slot) --
 *     and are synchronous, like the reference functions they replace.
 *   - Status: 0 = ok; nonzero = error, message via pnn_last_error().  The C++
 *     wrapper (include/pnn_b200/tensor_ops.hpp) rethrows nonzero status as
 *     std::invalid_argument, the reference's error type (tensor_ops.cpp:17-27).
 *   - Supported device formats: nbits in [2,16] with 2*max_scale <= 56
 *     (all of posit(8,0), (8,1), (8,2), (12,1), (16,1)).
 */
#ifndef PNN_B200_H
#define PNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PNN_OK 0
#define PNN_EINVAL 1         /* bad shape / argument (reference: std::invalid_argument) */
#define PNN_EUNSUPPORTED 2   /* format not supported on device */
#define PNN_EWORKSPACE 3     /* workspace too small */
#define PNN_ECUDA 4          /* CUDA runtime error */

const char* pnn_last_error(void);
int pnn_abi_version(void);
/* 1 if (nbits, es) runs on the device kernels. */
int pnn_format_supported(int nbits, int es);
/* Bytes per packed code on device for nbits (1 or 2). */
int pnn_code_bytes(int nbits);

/* ---- quire GEMM ---------------------------------------------------------
 * Replaces matmul(a, b, use_quire=true) -> matmul_quire
 * (tensor_ops.cpp:461-487, 166-185): C[M,N] = round(A[M,K] . B[K,N]). */
int pnn_quire_gemm_workspace(int nbits, int es, int64_t M, int64_t N, int64_t K, size_t* bytes);
int pnn_quire_gemm(int nbits, int es, const void* A, const void* B, void* C, int64_t M, int64_t N,
                   int64_t K, void* workspace, size_t workspace_bytes, void* stream);
/* Same, forcing split-K with at most max_kblocks k-blocks per split (tests). */
int pnn_quire_gemm_splitk(int nbits, int es, const void* A, const void* B, void* C, int64_t M,
                          int64_t N, int64_t K, int64_t max_kblocks, void* workspace,
                          size_t workspace_bytes, void* stream);
/* Same as pnn_quire_gemm, then synchronizes the stream and reports the
 * device time (CUDA events on that stream) of each phase in milliseconds:
 * ms[0] operand decode/pack, ms[1] tcgen05 MMA kernel, ms[2] split-K finalize.
 * For benchmarking / roofline accounting only. */
int pnn_quire_gemm_profiled(int nbits, int es, const void* A, const void* B, void* C, int64_t M,
                            int64_t N, int64_t K, void* workspace, size_t workspace_bytes,
                            void* stream, float* ms);
/* Host Tensor-storage entry: matmul(a, b, true) on uint64 code arrays. */
int pnn_matmul_host(int nbits, int es, const uint64_t* A, const uint64_t* B, uint64_t* C,
                    int64_t M, int64_t K, int64_t N);

/* ---- Conv2d / Linear passes (implicit GEMMs on the same tcgen05 core) -----
 * Shapes follow the reference: x [N,C,H,W], w [F,C,KH,KW], bias [F] or NULL,
 * y/dy [N,F,OH,OW] with OH = (H+2pad-KH)/stride+1.  A Linear layer is the
 * 1x1 convolution of x [B,in,1,1] with w [out,in,1,1].
 * pass: 0 forward (conv2d, tensor_ops.cpp:494-525 -- bias inside the quire),
 *       1 input grad (conv2d_input_grad, :527-574),
 *       2 weight grad (conv2d_weight_grad, :576-603).
 * Two implementations, same results bit for bit: the explicit path packs the
 * im2col digit image in HBM; the implicit path (stride 1, contracted channels
 * a multiple of 32, pixel rows tiling 128-row tiles) digitises each operand
 * once and lets TMA tile loads do the gather.  pnn_conv_algo selects:
 * 0 auto (implicit where eligible; default), 1 explicit only, 2 implicit only
 * (ineligible shapes fail with PNN_EUNSUPPORTED).  Returns the previous
 * setting, or -1 for an invalid value.  Query the workspace after setting. */
int pnn_conv_algo(int algo);
/* Reduced-digit GEMM variants (flag-selected 3/4-digit kernels) are
 * launched for passes of at least `macs` posit MACs (default 2^27); returns the
 * previous threshold (macs < 0: query only).  Results never depend on it. */
int64_t pnn_variant_min_work(int64_t macs);
int pnn_conv2d_workspace(int pass, int nbits, int es, int64_t N, int64_t C, int64_t H, int64_t W,
                         int64_t F, int64_t KH, int64_t KW, int stride, int pad, int has_bias,
                         size_t* bytes);
int pnn_conv2d_fwd(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H, int64_t W,
                   const void* w, int64_t F, int64_t KH, int64_t KW, const void* bias, int stride,
                   int pad, void* y, void* workspace, size_t workspace_bytes, void* stream);
int pnn_conv2d_dgrad(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t OH,
                     int64_t OW, const void* w, int64_t C, int64_t KH, int64_t KW, int64_t H,
                     int64_t W, int stride, int pad, void* dx, void* workspace,
                     size_t workspace_bytes, void* stream);
/* dw codes [F,C,KH,KW] (may be NULL) and/or the exact unrounded quire words
 * (16 bytes each, W-bit two's complement, same layout) + NaR mask -- the
 * data-parallel reduction input. */
int pnn_conv2d_wgrad(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t OH,
                     int64_t OW, const void* x, int64_t C, int64_t H, int64_t W, int64_t KH,
                     int64_t KW, int stride, int pad, void* dw, void* raw_words, void* raw_nar,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Layer-level Conv2d pair (the nn layer's forward / backward, SPEC.md §3.3 and
 * SURVEY.md Appendix A.6; the reference's layers are placeholders, layers.cpp:1).
 * Results are bit-identical to the per-pass calls above; what changes is the
 * data flow:
 *  - pnn_conv2d_fwd_save = pnn_conv2d_fwd that also leaves x's int8 digit
 *    planes (+ NaR map) in `saved` (pnn_conv2d_saved_bytes; 0 = geometry has no
 *    implicit forward/weight-gradient pair), the layer's saved tensor;
 *  - pnn_conv2d_backward = in one call
 *        dw = conv2d_weight_grad(p_g, convert(dy, p_b -> p_g), convert(x, p_f -> p_g))
 *        dx = conv2d_input_grad(p_b, dy, w_bwd)           (dx may be NULL)
 *    with the weight gradient reading the saved forward digits (same format, or
 *    an exact widening p_f -> p_g by whole digits), stage conversions folded
 *    into the digitisers, and dy digitised once for both passes when p_b == p_g.
 *    dw codes and/or raw quire words + NaR mask as in pnn_conv2d_wgrad.
 *    PNN_EUNSUPPORTED from the workspace query = use the per-pass calls. */
int pnn_conv2d_saved_bytes(int nbits, int es, int64_t N, int64_t C, int64_t H, int64_t W, int64_t F,
                           int64_t KH, int64_t KW, int stride, int pad, size_t* bytes);
int pnn_conv2d_fwd_save(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H, int64_t W,
                        const void* w, int64_t F, int64_t KH, int64_t KW, const void* bias, int stride,
                        int pad, void* y, void* saved, size_t saved_bytes, void* workspace,
                        size_t workspace_bytes, void* stream);
/* pnn_conv2d_fwd_save with the following ReLU layer fused (relu != 0: y =
 * relu(conv), SURVEY.md Appendix A.2 -- relu(NaR) = 0 -- and, if y_pre is
 * non-NULL, the pre-activation conv output there too).  saved may be NULL.
 * Implicit-path geometries only (else PNN_EUNSUPPORTED). */
int pnn_conv2d_fwd_layer(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H, int64_t W,
                         const void* w, int64_t F, int64_t KH, int64_t KW, const void* bias, int stride,
                         int pad, int relu, void* y, void* y_pre, void* saved, size_t saved_bytes,
                         void* workspace, size_t workspace_bytes, void* stream);
int pnn_conv2d_backward_workspace(int f_nbits, int f_es, int b_nbits, int b_es, int g_nbits, int g_es,
                                  int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int64_t KH,
                                  int64_t KW, int stride, int pad, int raw, int has_dx, int has_saved,
                                  size_t* bytes);
int pnn_conv2d_backward(int f_nbits, int f_es, int b_nbits, int b_es, int g_nbits, int g_es,
                        const void* dy, const void* x, const void* saved, size_t saved_bytes,
                        const void* w_bwd, int64_t N, int64_t C, int64_t H, int64_t W, int64_t F,
                        int64_t KH, int64_t KW, int stride, int pad, void* dx, void* dw,
                        void* raw_words, void* raw_nar, void* workspace, size_t workspace_bytes,
                        void* stream);
/* pnn_conv2d_backward for a Conv2d followed by a ReLU layer: dy is the ReLU's
 * output gradient and gate its saved forward values (format p_f, layout of
 * dy); the ReLU backward (dy where gate > 0, else 0, Appendix A.2) is applied
 * inside the digitisers; dy_gated (may be NULL) receives the gated dy itself
 * (p_b codes) when a caller wants it (pnn_bias_grad_gated does not need it). */
int pnn_conv2d_backward_gated(int f_nbits, int f_es, int b_nbits, int b_es, int g_nbits, int g_es,
                              const void* dy, const void* gate, void* dy_gated, const void* x,
                              const void* saved, size_t saved_bytes, const void* w_bwd, int64_t N,
                              int64_t C, int64_t H, int64_t W, int64_t F, int64_t KH, int64_t KW,
                              int stride, int pad, void* dx, void* dw, void* raw_words, void* raw_nar,
                              void* workspace, size_t workspace_bytes, void* stream);
/* conv2d_bias_grad (tensor_ops.cpp:605-618) for dy [N,F,P] with P = OH*OW,
 * and column_sum (:722-731) with P = 1: db[f] = round(quire sum of dy[:,f,:]). */
int pnn_bias_grad_workspace(int64_t F, size_t* bytes);
int pnn_bias_grad(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t P, void* db,
                  void* raw_words, void* raw_nar, void* workspace, size_t workspace_bytes,
                  void* stream);
/* conv2d_bias_grad of a ReLU's input gradient: db[f] = round(quire sum of
 * (gate > 0 ? dy : 0)) with gate = the ReLU's forward values ((gate_nbits)
 * codes, layout of dy) -- the gated tensor is never materialised.  Table
 * formats (nbits <= 12) with 16-byte rows only (else PNN_EUNSUPPORTED). */
int pnn_bias_grad_gated(int nbits, int es, const void* dy, int gate_nbits, const void* gate, int64_t N,
                        int64_t F, int64_t P, void* db, void* raw_words, void* raw_nar, void* workspace,
                        size_t workspace_bytes, void* stream);

/* ---- elementwise kernels of the training step -----------------------------
 * Semantics: convert = convert_tensor (tensor_ops.cpp:807-821); maxpool =
 * maxpool2d / maxpool2d_backward (:620-670, argmax = flat input index, int64);
 * ReLU, softmax cross-entropy and SGD have no reference code (placeholders,
 * SURVEY.md §0.3) and follow SURVEY.md Appendix A.2 / A.5 / A.7 exactly as the
 * CPU oracle step (oracle/step.py) does. */
int pnn_convert(int src_nbits, int src_es, int dst_nbits, int dst_es, const void* src, void* dst,
                int64_t n, void* stream);
int pnn_relu_fwd(int nbits, int es, const void* x, void* y, int64_t n, void* stream);
/* dx = x > 0 ? dy : 0 with x in (x_nbits, x_es) and dy/dx in (g_nbits, g_es). */
int pnn_relu_bwd(int x_nbits, int x_es, const void* x, int g_nbits, int g_es, const void* dy,
                 void* dx, int64_t n, void* stream);
/* argmax may be NULL for 2x2 / stride-2 tiled pooling (the layer then
 * recomputes it in pnn_maxpool2d_bwd_x instead of storing 8 bytes per output). */
int pnn_maxpool2d_fwd(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H,
                      int64_t W, int k, int stride, void* y, int64_t* argmax, void* stream);
/* Window-specialised backward: dy and argmax MUST be the (N, C, OH, OW) output
 * of pnn_maxpool2d_fwd with the same k / stride (each argmax inside its own
 * window); any other argmax: pnn_maxpool2d_bwd_scatter. */
int pnn_maxpool2d_bwd(int nbits, int es, const void* dy, const int64_t* argmax, int64_t N,
                      int64_t C, int64_t H, int64_t W, int k, int stride, void* dx, void* stream);
/* maxpool2d_backward(dy, argmax, x_shape) exactly as tensor_ops.cpp:658-670:
 * dx = 0, then for i = 0..n_out-1 in order dx[argmax[i]] = add(dx[argmax[i]], dy[i]),
 * for ANY argmax (no window assumed; n_in = numel(x_shape)).  Indices outside
 * [0, n_in) are dropped (the reference's behaviour there is undefined; the host
 * mirrors reject them).  n_out, n_in < 2^31.  Replaces maxpool2d_backward
 * (tensor_ops.hpp:50-51). */
int pnn_maxpool2d_bwd_scatter_workspace(int64_t n_out, int64_t n_in, size_t* bytes);
int pnn_maxpool2d_bwd_scatter(int nbits, int es, const void* dy, const int64_t* argmax, int64_t n_out,
                              void* dx, int64_t n_in, void* workspace, size_t workspace_bytes,
                              void* stream);
/* maxpool2d_backward(dy, argmax of maxpool2d(x)) with the argmax recomputed
 * from the pooled input x (x in (x_nbits, x_es), dy/dx in (g_nbits, g_es));
 * 2x2 / stride-2 tiled windows (else PNN_EUNSUPPORTED: use the argmax pair). */
int pnn_maxpool2d_bwd_x(int x_nbits, int x_es, const void* x, int g_nbits, int g_es, const void* dy,
                        int64_t N, int64_t C, int64_t H, int64_t W, int k, int stride, void* dx,
                        void* stream);
/* Same, for a MaxPool2d fed by a ReLU (x = the ReLU's output): relu_gate != 0
 * also applies the ReLU backward (zero unless the window max is > 0), i.e.
 * relu_bwd(maxpool2d_backward(dy)) in one pass. */
int pnn_maxpool2d_relu_bwd_x(int x_nbits, int x_es, const void* x, int g_nbits, int g_es, const void* dy,
                             int64_t N, int64_t C, int64_t H, int64_t W, int k, int stride, int relu_gate,
                             void* dx, void* stream);
/* logits [B, classes] in the loss format; labels int32 [B]; outputs dlogits
 * [B, classes] (already scaled by 2^-log2_batch), per-row losses [B], the
 * batch loss (1 code, may be NULL) and/or the raw quire word (16 bytes) + NaR
 * byte of sum(loss_i) for the data-parallel reduction (may be NULL). */
int pnn_softmax_xent(int nbits, int es, const void* logits, const int32_t* labels, int64_t B,
                     int64_t classes, int log2_batch, void* dlogits, void* loss_rows,
                     void* loss_out, void* raw_word, void* raw_nar, void* stream);
/* master = sub(master, mul(lr, convert(grad -> opt))) in the optimizer
 * format; copy1/copy2 (may be NULL) receive convert(master -> their format). */
int pnn_sgd_step(int opt_nbits, int opt_es, void* master, int g_nbits, int g_es, const void* grad,
                 int64_t n, uint32_t lr_code, int c1_nbits, int c1_es, void* copy1, int c2_nbits,
                 int c2_es, void* copy2, void* stream);
/* Loss scaling by 2^s (SPEC "scale_gradients"): the
 * logit gradient leaves the loss as ldexp(p - onehot, s - log2_batch) (the
 * loss value is not scaled); the SGD step unscales in the optimizer format,
 * g = ldexp(convert(grad), -s), before master = sub(master, mul(lr, g)).
 * s = 0 is the unscaled entry above. */
int pnn_softmax_xent_scaled(int nbits, int es, const void* logits, const int32_t* labels,
                            int64_t B, int64_t classes, int log2_batch, int grad_scale_log2,
                            void* dlogits, void* loss_rows, void* loss_out, void* raw_word,
                            void* raw_nar, void* stream);
/* The same step split in two so the loss can run beside the backward pass:
 * _grad writes dlogits and the rounded row sums S (loss format, [B]); _loss
 * turns them into the per-row losses log(S) - (z_y - m) and the batch loss /
 * raw word exactly as pnn_softmax_xent_scaled does. */
int pnn_softmax_xent_grad(int nbits, int es, const void* logits, const int32_t* labels, int64_t B,
                          int64_t classes, int log2_batch, int grad_scale_log2, void* dlogits,
                          void* s_rows, void* stream);
int pnn_softmax_xent_loss(int nbits, int es, const void* logits, const int32_t* labels,
                          const void* s_rows, int64_t B, int64_t classes, int log2_batch,
                          void* loss_rows, void* loss_out, void* raw_word, void* raw_nar, void* stream);
/* The batch-loss half of pnn_softmax_xent on its own: loss_out[0] =
 * ldexp(round(quire sum of loss_rows[0..B)), -log2_batch).  Data-parallel
 * training gathers the ranks' loss rows through it when the loss format's
 * quire is wider than the 128-bit raw word (posit(10,2): W = 138). */
int pnn_loss_reduce(int nbits, int es, const void* loss_rows, int64_t B, int log2_batch,
                    void* loss_out, void* stream);
int pnn_sgd_step_scaled(int opt_nbits, int opt_es, void* master, int g_nbits, int g_es,
                        const void* grad, int64_t n, uint32_t lr_code, int c1_nbits, int c1_es,
                        void* copy1, int c2_nbits, int c2_es, void* copy2, int grad_scale_log2,
                        void* stream);
/* The optimizer step of several parameter tensors (same formats) in one
 * launch: tensor i is pnn_sgd_step_scaled on (masters[i], grads[i], ns[i],
 * copy1s[i], copy2s[i]); copy1s / copy2s may be NULL (no such stage copy). */
int pnn_sgd_step_multi(int opt_nbits, int opt_es, int g_nbits, int g_es, uint32_t lr_code, int c1_nbits,
                       int c1_es, int c2_nbits, int c2_es, int grad_scale_log2, int count,
                       void* const* masters, const void* const* grads, void* const* copy1s,
                       void* const* copy2s, const int64_t* ns, void* stream);
/* avgpool2d / avgpool2d_backward (tensor_ops.cpp:672-720): window sum (quire
 * when use_quire, else an add chain) times the caller-quantized reciprocal. */
int pnn_avgpool2d_fwd(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H,
                      int64_t W, int k, int stride, int use_quire, uint32_t recip_code, void* y,
                      void* stream);
int pnn_avgpool2d_bwd(int nbits, int es, const void* dy, int64_t N, int64_t C, int64_t H,
                      int64_t W, int k, int stride, uint32_t recip_code, void* dx, void* stream);

/* ---- remaining SPEC layers ---------
 * No reference code exists for these (placeholders); the rounding sequence of
 * each is fixed in oracle/layers_oracle.c and reproduced bit for bit.
 * Reductions are exact quires, so the formats they run in need W <= 128
 * (PNN_EUNSUPPORTED otherwise); elementwise steps take formats up to 2R <= 96.
 *
 * Activation layers, kind 1 tanh / 2 sigmoid (posit_math.cpp:109-130):
 * y = act(x); backward from the forward OUTPUT y (converted to dy's format b):
 * tanh dx = dy*(1 - y*y), sigmoid dx = dy*(y*(1 - y)), each op rounded in b. */
int pnn_act_fwd(int kind, int nbits, int es, const void* x, void* y, int64_t n, void* stream);
int pnn_act_bwd(int kind, int f_nbits, int f_es, const void* y, int b_nbits, int b_es,
                const void* dy, void* dx, int64_t n, void* stream);
/* Dropout (seeded mask, scale 1/(1-p)): with s = seed + (*seed_offset if
 * seed_offset, a DEVICE uint64, is not NULL -- a per-step counter that a
 * captured CUDA graph advances on replay), keep element i iff
 * (splitmix64(s ^ i*0xD1B54A32D192ED03) >> 32) >= thresh (thresh =
 * floor(p*2^32)); y = keep ? x*scale : 0.  The backward is the same call on
 * dy with the backward format's scale code and the same seed. */
int pnn_dropout(int nbits, int es, const void* x, void* y, int64_t n, uint64_t seed,
                const void* seed_offset, uint32_t thresh, uint32_t scale_code, void* stream);
/* MSE: d = y - t; loss = round(quire sum d*d) / G;
 * grad = ldexp(d * (2 / G), grad_scale_log2); G = global element count. */
int pnn_mse(int nbits, int es, const void* y, const void* t, int64_t n, int64_t global_count,
            int grad_scale_log2, void* grad, void* loss_out, void* stream);
/* Batch normalisation over [N, C, HW] per channel (training: batch mean /
 * biased variance by quire sums, running stats updated in the optimizer
 * format with momentum code mom; eval: the running stats).  y = gamma*xhat +
 * beta, xhat and inv = 1/sqrt(var + eps) saved for the backward. */
int pnn_batchnorm_workspace(int64_t C, size_t* bytes);
int pnn_batchnorm_fwd(int f_nbits, int f_es, const void* x, int64_t N, int64_t C, int64_t HW,
                      const void* gamma, const void* beta, uint32_t eps_code, int training,
                      int o_nbits, int o_es, void* run_mean, void* run_var, uint32_t mom_code,
                      void* y, void* xhat, void* inv, void* workspace, size_t workspace_bytes,
                      void* stream);
/* dgamma / dbeta (gradient format, may be NULL) and/or their raw quire words
 * (16 bytes + NaR byte per channel) for the data-parallel reduction. */
int pnn_batchnorm_bwd(int f_nbits, int f_es, const void* xhat, const void* inv, int b_nbits,
                      int b_es, const void* dy, int64_t N, int64_t C, int64_t HW,
                      const void* gamma_b, int g_nbits, int g_es, void* dx, void* dgamma,
                      void* dbeta, void* dgamma_raw, void* dgamma_nar, void* dbeta_raw,
                      void* dbeta_nar, void* workspace, size_t workspace_bytes, void* stream);
/* SGD with momentum in the optimizer format:
 * g = ldexp(convert(grad), -s); v = mu*v + g; master = master - lr*v. */
int pnn_sgd_step_momentum(int opt_nbits, int opt_es, void* master, void* velocity, int g_nbits,
                          int g_es, const void* grad, int64_t n, uint32_t lr_code,
                          uint32_t mu_code, int c1_nbits, int c1_es, void* copy1, int c2_nbits,
                          int c2_es, void* copy2, int grad_scale_log2, void* stream);
/* Data ingestion: from_float64 (posit.cpp:502-508) of device doubles into
 * packed codes -- inputs, labels-free data and initial weights. */
int pnn_from_float64(int nbits, int es, const double* x, void* codes, int64_t n, void* stream);
/* Scalar ALU on device (parity): op 0 add 1 sub 2 mul 3 div 4 exp 5 log
 * 6 round_to_int 7 ldexp(a, (int)b) 8 compare 9 to_int64 (low 32 bits) 10 tanh
 * 11 sigmoid (posit_math.cpp:109-130) 12 sqrt (posit_math.cpp:132-160). */
int pnn_scalar_eval(int nbits, int es, int op, const uint32_t* a, const uint32_t* b,
                    uint32_t* out, int64_t n, void* stream);

/* ---- device posit core (parity / diagnostics) ----------------------------
 * pnn_decode_x: code -> exact integer image X = value * 2^max_scale and NaR
 *   flag (detail::unpack posit.cpp:67-91 / DecodeTables::Fixed).
 * pnn_quire_round: raw W-bit quire words (lo, hi pairs, two's complement,
 *   LSB 2^-2R) -> posit code (Quire::to_posit, quire.cpp:105-146).
 * pnn_pack_round: (neg, scale, sig, sticky) -> code (detail::pack_round,
 *   posit.cpp:93-132). */
int pnn_decode_x(int nbits, int es, const uint32_t* codes, int64_t n, int64_t* X, uint8_t* nar,
                 void* stream);
int pnn_quire_round(int nbits, int es, const uint64_t* q, int64_t n, uint32_t* codes,
                    void* stream);
int pnn_pack_round(int nbits, int es, const int32_t* neg, const int32_t* scale,
                   const uint64_t* sig, const int32_t* sticky, int64_t n, uint32_t* codes,
                   void* stream);

/* ---- non-quire posit path (use_quire = false) -----------------------------
 * One correctly rounded posit multiply and add per term in the reference's
 * term order: matmul_seq / conv_seq / gather_seq(_sum), tensor_ops.cpp:145-164,
 * 232-264, 302-335.  Device pointers to packed codes; one thread per output. */
int pnn_matmul_seq(int nbits, int es, const void* A, const void* B, void* C, int64_t M, int64_t N,
                   int64_t K, void* stream);
int pnn_conv2d_fwd_seq(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H, int64_t W,
                       const void* w, int64_t F, int64_t KH, int64_t KW, const void* bias,
                       int stride, int pad, void* y, void* stream);
int pnn_conv2d_dgrad_seq(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t OH,
                         int64_t OW, const void* w, int64_t C, int64_t KH, int64_t KW, int64_t H,
                         int64_t W, int stride, int pad, void* dx, void* stream);
int pnn_conv2d_wgrad_seq(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t OH,
                         int64_t OW, const void* x, int64_t C, int64_t H, int64_t W, int64_t KH,
                         int64_t KW, int stride, int pad, void* dw, void* stream);
int pnn_bias_grad_seq(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t P, void* db,
                      void* stream);

/* ---- data-parallel quire-word reduction --------------
 * Raw W-bit quire words (16 bytes each) + NaR bytes -> int64 lanes
 * [n][L+1] of 60-bit digits (L = pnn_quire_lanes) plus a NaR lane, ready for
 * an integer SUM all-reduce (NCCL int64; 8 ranks * (2^60-1) < 2^63: no overflow); then
 * lanes -> carry-propagated W-bit quire -> one rounding (codes) and/or the
 * reduced raw words. */
int pnn_quire_lanes(int nbits, int es);
int pnn_quire_to_lanes(int nbits, int es, const void* words, const uint8_t* nar, int64_t n,
                       uint64_t* lanes, void* stream);
int pnn_lanes_to_posit(int nbits, int es, const uint64_t* lanes, int64_t n, void* codes,
                       void* words_out, void* stream);

/* ---- measurement ---------------------------------------------------------
 * Tensor-pipe ceiling for the kind::i8 MMA shape the quire GEMM issues
 * (M=128, N=256, K=32 from shared memory), one CTA per SM, `iters` MMAs each;
 * returns int8 TOPS (2 ops per MAC) and the launch time.  Roofline
 * denominator for bench.py. */
int pnn_probe_int8_peak(int iters, double* tops, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* PNN_B200_H */
