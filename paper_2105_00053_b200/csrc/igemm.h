// Internal interface of the implicit-GEMM convolution path (igemm.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "posit_device.cuh"

namespace pnn_b200 {

struct ConvGeom {
    int64_t N, C, H, W, F, KH, KW, OH, OW;
    int stride, pad;
};

// Conv algorithm selection (pnn_conv_algo): 0 auto (implicit where eligible),
// 1 always the explicit pack path, 2 implicit only (ineligible -> error).
int conv_algo();
int64_t variant_min_work();
int64_t set_variant_min_work(int64_t v);

// Whether pass (0 fwd, 1 input grad, 2 weight grad) runs implicitly for this
// geometry / format under the current algorithm setting; *bytes = workspace.
bool igemm_eligible(int pass, const PositFmt& f, const ConvGeom& g, bool raw, size_t* bytes);

// 0 ok, 3 workspace too small, 4 CUDA error, 5 tensor-map encoding failed.
// saved != null: x's digits (+ NaR map) are written there and kept for the
// weight gradient (igemm_conv_backward); igemm_saved_bytes = its size (0: the
// geometry has no implicit forward + weight-gradient pair).
int igemm_conv_fwd(const PositFmt& f, const ConvGeom& g, const void* x, const void* w,
                   const void* bias, void* y, void* ws, size_t ws_bytes, cudaStream_t st,
                   void* saved = nullptr, size_t saved_bytes = 0, int relu = 0,
                   void* pre = nullptr);
size_t igemm_saved_bytes(const PositFmt& f, const ConvGeom& g);
int igemm_conv_dgrad(const PositFmt& f, const ConvGeom& g, const void* dy, const void* w, void* dx,
                     void* ws, size_t ws_bytes, cudaStream_t st);
int igemm_conv_wgrad(const PositFmt& f, const ConvGeom& g, const void* dy, const void* x, void* dw,
                     unsigned __int128* raw_words, uint8_t* raw_nar, void* ws, size_t ws_bytes,
                     cudaStream_t st);

// Fused layer backward (weight gradient in fg from dy of format fb and x of
// format ff -- or the forward's saved digits --, then the input gradient in fb
// reusing dy's digits when fb == fg).  Eligibility / workspace first.
bool igemm_backward_eligible(const PositFmt& ff, const PositFmt& fb, const PositFmt& fg,
                             const ConvGeom& g, bool raw, bool has_dx, bool saved, size_t* bytes);
int igemm_conv_backward(const PositFmt& ff, const PositFmt& fb, const PositFmt& fg, const ConvGeom& g,
                        const void* dy, const void* x, const void* saved, size_t saved_bytes,
                        const void* w_bwd, void* dx, void* dw, unsigned __int128* raw_words,
                        uint8_t* raw_nar, void* ws, size_t ws_bytes, cudaStream_t st,
                        const void* gate = nullptr, int gate_nbits = 0, void* dy_gated = nullptr);

}  // namespace pnn_b200
