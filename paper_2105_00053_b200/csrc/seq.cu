// Non-quire (use_quire = false) posit kernels: one correctly rounded posit
// multiply and add per term, in the reference's term order (SURVEY.md §8f
// item 1).  Inherently sequential along K, so one thread owns one output.
//
//   matmul_seq          proj/src/tensor_ops.cpp:145-164   acc = mul(a0,b0); acc = add(acc, mul(ak,bk))
//   conv_seq            tensor_ops.cpp:232-264            taps (c,ky,kx) over the zero-padded input, then + bias
//   gather_seq          tensor_ops.cpp:302-318            input grad (f,ky,kx valid taps), weight grad (n,oy,ox)
//   gather_seq_sum      tensor_ops.cpp:320-335            bias grad / column sum
// Empty term sets give 0 (tensor_ops.cpp:315).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/pnn_b200.h"
#include "posit_scalar.cuh"
#include "status.h"

namespace pnn_b200 {

__device__ __forceinline__ uint32_t ldc(const void* p, int64_t i, int b) {
    return b == 1 ? uint32_t(static_cast<const uint8_t*>(p)[i])
                  : uint32_t(static_cast<const uint16_t*>(p)[i]);
}
__device__ __forceinline__ void stc(void* p, int64_t i, int b, uint32_t c) {
    if (b == 1) static_cast<uint8_t*>(p)[i] = uint8_t(c);
    else static_cast<uint16_t*>(p)[i] = uint16_t(c);
}

#define SEQ_LOOP(i, n)                                                           \
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < (n); \
         i += int64_t(gridDim.x) * blockDim.x)

__global__ void matmul_seq_kernel(PositFmt f, int b, const void* A, const void* B, void* C,
                                  int64_t M, int64_t N, int64_t K) {
    SEQ_LOOP(o, M * N) {
        const int64_t i = o / N, j = o % N;
        uint32_t acc = p_mul(f, ldc(A, i * K, b), ldc(B, j, b));
        for (int64_t k = 1; k < K; ++k)
            acc = p_add(f, acc, p_mul(f, ldc(A, i * K + k, b), ldc(B, k * N + j, b)));
        stc(C, o, b, acc);
    }
}

struct SeqConv {
    int64_t N, C, H, W, F, KH, KW, OH, OW;
    int stride, pad;
};

__global__ void conv_fwd_seq_kernel(PositFmt f, int b, const void* x, const void* w,
                                    const void* bias, SeqConv g, void* y) {
    SEQ_LOOP(o, g.N * g.F * g.OH * g.OW) {
        const int64_t ox = o % g.OW, oy = (o / g.OW) % g.OH, ff = (o / (g.OW * g.OH)) % g.F,
                      n = o / (g.OW * g.OH * g.F);
        uint32_t acc = 0;
        bool first = true;
        for (int64_t c = 0; c < g.C; ++c)
            for (int64_t ky = 0; ky < g.KH; ++ky)
                for (int64_t kx = 0; kx < g.KW; ++kx) {
                    const int64_t iy = oy * g.stride + ky - g.pad, ix = ox * g.stride + kx - g.pad;
                    const uint32_t xv = (iy < 0 || iy >= g.H || ix < 0 || ix >= g.W)
                                            ? 0u  // pad_nchw zero (tensor_ops.cpp:189-203)
                                            : ldc(x, ((n * g.C + c) * g.H + iy) * g.W + ix, b);
                    const uint32_t p = p_mul(f, xv, ldc(w, ((ff * g.C + c) * g.KH + ky) * g.KW + kx, b));
                    acc = first ? p : p_add(f, acc, p);
                    first = false;
                }
        if (bias) acc = p_add(f, acc, ldc(bias, ff, b));
        stc(y, o, b, acc);
    }
}

__global__ void conv_dgrad_seq_kernel(PositFmt f, int b, const void* dy, const void* w, SeqConv g,
                                      void* dx) {
    SEQ_LOOP(o, g.N * g.C * g.H * g.W) {
        const int64_t ix = o % g.W + g.pad, iy = (o / g.W) % g.H + g.pad,
                      c = (o / (g.W * g.H)) % g.C, n = o / (g.W * g.H * g.C);
        uint32_t acc = 0;
        bool first = true;
        for (int64_t ff = 0; ff < g.F; ++ff)
            for (int64_t ky = 0; ky < g.KH; ++ky) {
                const int64_t ty = iy - ky;
                if (ty < 0 || ty % g.stride) continue;
                const int64_t oy = ty / g.stride;
                if (oy >= g.OH) continue;
                for (int64_t kx = 0; kx < g.KW; ++kx) {
                    const int64_t tx = ix - kx;
                    if (tx < 0 || tx % g.stride) continue;
                    const int64_t ox = tx / g.stride;
                    if (ox >= g.OW) continue;
                    const uint32_t p = p_mul(f, ldc(dy, ((n * g.F + ff) * g.OH + oy) * g.OW + ox, b),
                                             ldc(w, ((ff * g.C + c) * g.KH + ky) * g.KW + kx, b));
                    acc = first ? p : p_add(f, acc, p);
                    first = false;
                }
            }
        stc(dx, o, b, acc);
    }
}

__global__ void conv_wgrad_seq_kernel(PositFmt f, int b, const void* dy, const void* x, SeqConv g,
                                      void* dw) {
    SEQ_LOOP(o, g.F * g.C * g.KH * g.KW) {
        const int64_t kx = o % g.KW, ky = (o / g.KW) % g.KH, c = (o / (g.KW * g.KH)) % g.C,
                      ff = o / (g.KW * g.KH * g.C);
        uint32_t acc = 0;
        bool first = true;
        for (int64_t n = 0; n < g.N; ++n)
            for (int64_t oy = 0; oy < g.OH; ++oy)
                for (int64_t ox = 0; ox < g.OW; ++ox) {
                    const int64_t iy = oy * g.stride + ky - g.pad, ix = ox * g.stride + kx - g.pad;
                    const uint32_t xv = (iy < 0 || iy >= g.H || ix < 0 || ix >= g.W)
                                            ? 0u
                                            : ldc(x, ((n * g.C + c) * g.H + iy) * g.W + ix, b);
                    const uint32_t p = p_mul(f, ldc(dy, ((n * g.F + ff) * g.OH + oy) * g.OW + ox, b), xv);
                    acc = first ? p : p_add(f, acc, p);
                    first = false;
                }
        stc(dw, o, b, acc);
    }
}

// dy [N][F][P] -> out[f] = add-chain over (n, p) in order (gather_seq_sum).
__global__ void bias_grad_seq_kernel(PositFmt f, int b, const void* dy, int64_t N, int64_t F,
                                     int64_t P, void* out) {
    SEQ_LOOP(ch, F) {
        uint32_t acc = 0;
        bool first = true;
        for (int64_t n = 0; n < N; ++n)
            for (int64_t p = 0; p < P; ++p) {
                const uint32_t v = ldc(dy, (n * F + ch) * P + p, b);
                acc = first ? v : p_add(f, acc, v);
                first = false;
            }
        stc(out, ch, b, acc);
    }
}

}  // namespace pnn_b200

using namespace pnn_b200;

namespace {

bool seq_fmt_ok(int nbits, int es) {
    if (nbits < 2 || nbits > 16 || es < 0 || es > 4) return false;
    return 2 * make_fmt(nbits, es).R <= 56;
}
int seq_grid(int64_t n) {
    int64_t b = (n + 127) / 128;
    if (b > 148 * 32) b = 148 * 32;
    return int(b < 1 ? 1 : b);
}
int done(const char* what) {
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PNN_OK : set_status(PNN_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
bool geom(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int64_t KH, int64_t KW, int s,
          int p, SeqConv* g) {
    if (N < 0 || C < 1 || H < 1 || W < 1 || F < 1 || KH < 1 || KW < 1 || s < 1 || p < 0) return false;
    if (H + 2 * p < KH || W + 2 * p < KW) return false;
    *g = SeqConv{N, C, H, W, F, KH, KW, (H + 2 * p - KH) / s + 1, (W + 2 * p - KW) / s + 1, s, p};
    return true;
}

}  // namespace

extern "C" {

int pnn_matmul_seq(int nbits, int es, const void* A, const void* B, void* C, int64_t M, int64_t N,
                   int64_t K, void* stream) {
    if (!seq_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "matmul_seq: format");
    if (M < 0 || N < 0 || K < 0) return set_status(PNN_EINVAL, "matmul: negative dimension");
    if (M == 0 || N == 0) return PNN_OK;
    const int b = nbits <= 8 ? 1 : 2;
    if (K == 0) {
        cudaMemsetAsync(C, 0, size_t(M * N) * b, (cudaStream_t)stream);
        return done("matmul_seq");
    }
    matmul_seq_kernel<<<seq_grid(M * N), 128, 0, (cudaStream_t)stream>>>(make_fmt(nbits, es), b, A,
                                                                          B, C, M, N, K);
    return done("matmul_seq");
}

int pnn_conv2d_fwd_seq(int nbits, int es, const void* x, int64_t N, int64_t C, int64_t H, int64_t W,
                       const void* w, int64_t F, int64_t KH, int64_t KW, const void* bias,
                       int stride, int pad, void* y, void* stream) {
    SeqConv g;
    if (!seq_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "conv_seq: format");
    if (!geom(N, C, H, W, F, KH, KW, stride, pad, &g)) return set_status(PNN_EINVAL, "conv2d: bad shape");
    if (N == 0) return PNN_OK;
    conv_fwd_seq_kernel<<<seq_grid(N * F * g.OH * g.OW), 128, 0, (cudaStream_t)stream>>>(
        make_fmt(nbits, es), nbits <= 8 ? 1 : 2, x, w, bias, g, y);
    return done("conv2d_fwd_seq");
}

int pnn_conv2d_dgrad_seq(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t OH,
                         int64_t OW, const void* w, int64_t C, int64_t KH, int64_t KW, int64_t H,
                         int64_t W, int stride, int pad, void* dx, void* stream) {
    SeqConv g;
    if (!seq_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "conv_seq: format");
    if (!geom(N, C, H, W, F, KH, KW, stride, pad, &g) || g.OH != OH || g.OW != OW)
        return set_status(PNN_EINVAL, "conv2d_input_grad: bad shape");
    if (N == 0) return PNN_OK;
    conv_dgrad_seq_kernel<<<seq_grid(N * C * H * W), 128, 0, (cudaStream_t)stream>>>(
        make_fmt(nbits, es), nbits <= 8 ? 1 : 2, dy, w, g, dx);
    return done("conv2d_dgrad_seq");
}

int pnn_conv2d_wgrad_seq(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t OH,
                         int64_t OW, const void* x, int64_t C, int64_t H, int64_t W, int64_t KH,
                         int64_t KW, int stride, int pad, void* dw, void* stream) {
    SeqConv g;
    if (!seq_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "conv_seq: format");
    if (!geom(N, C, H, W, F, KH, KW, stride, pad, &g) || g.OH != OH || g.OW != OW)
        return set_status(PNN_EINVAL, "conv2d_weight_grad: bad shape");
    conv_wgrad_seq_kernel<<<seq_grid(F * C * KH * KW), 128, 0, (cudaStream_t)stream>>>(
        make_fmt(nbits, es), nbits <= 8 ? 1 : 2, dy, x, g, dw);
    return done("conv2d_wgrad_seq");
}

int pnn_bias_grad_seq(int nbits, int es, const void* dy, int64_t N, int64_t F, int64_t P, void* db,
                      void* stream) {
    if (!seq_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "bias_grad_seq: format");
    if (N < 0 || F < 1 || P < 1) return set_status(PNN_EINVAL, "bias_grad: bad shape");
    bias_grad_seq_kernel<<<seq_grid(F), 128, 0, (cudaStream_t)stream>>>(make_fmt(nbits, es),
                                                                        nbits <= 8 ? 1 : 2, dy, N,
                                                                        F, P, db);
    return done("bias_grad_seq");
}

}  // extern "C"
