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

// Whether pass (0 fwd, 1 input grad, 2 weight grad) runs implicitly for this
// geometry / format under the current algorithm setting; *bytes = workspace.
bool igemm_eligible(int pass, const PositFmt& f, const ConvGeom& g, bool raw, size_t* bytes);

// 0 ok, 3 workspace too small, 4 CUDA error, 5 tensor-map encoding failed.
int igemm_conv_fwd(const PositFmt& f, const ConvGeom& g, const void* x, const void* w,
                   const void* bias, void* y, void* ws, size_t ws_bytes, cudaStream_t st);
int igemm_conv_dgrad(const PositFmt& f, const ConvGeom& g, const void* dy, const void* w, void* dx,
                     void* ws, size_t ws_bytes, cudaStream_t st);
int igemm_conv_wgrad(const PositFmt& f, const ConvGeom& g, const void* dy, const void* x, void* dw,
                     unsigned __int128* raw_words, uint8_t* raw_nar, void* ws, size_t ws_bytes,
                     cudaStream_t st);

}  // namespace pnn_b200
