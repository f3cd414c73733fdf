// Shared helpers of the elementwise kernels (eltwise.cu, layers.cu): packed
// code load/store for 1- or 2-byte codes and a grid-stride loop.
#pragma once

#include <cstdint>

namespace pnn_b200 {

template <typename T>
__device__ __forceinline__ uint32_t ld_code(const void* p, int64_t i) {
    return uint32_t(static_cast<const T*>(p)[i]);
}

__device__ __forceinline__ uint32_t load_any(const void* p, int64_t i, int bytes) {
    return bytes == 1 ? uint32_t(static_cast<const uint8_t*>(p)[i])
                      : uint32_t(static_cast<const uint16_t*>(p)[i]);
}
__device__ __forceinline__ void store_any(void* p, int64_t i, int bytes, uint32_t c) {
    if (bytes == 1) static_cast<uint8_t*>(p)[i] = uint8_t(c);
    else static_cast<uint16_t*>(p)[i] = uint16_t(c);
}

}  // namespace pnn_b200

#define GRID_STRIDE(i, n)                                                        \
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < (n); \
         i += int64_t(gridDim.x) * blockDim.x)
