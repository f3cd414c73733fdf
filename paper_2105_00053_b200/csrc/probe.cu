// Tensor-pipe peak probe: the roofline denominator for the kind::i8 kernels.
//
// One CTA per SM issues back-to-back tcgen05.mma.kind::i8 (M=128, N=256,
// K=32, operands in shared memory, two alternating TMEM accumulators) from a
// single thread -- the same instruction shape the quire GEMM issues -- and the
// host times the launch with CUDA events.  Nothing is loaded from HBM, so the
// result is the int8 tensor-core issue ceiling on this GPU at its current
// clocks, measured the same way the GEMM is.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/pnn_b200.h"
#include "sm100_ptx.cuh"

namespace pnn_b200 {

__global__ void __launch_bounds__(128, 1) tc_int8_probe_kernel(int iters) {
    constexpr int kN = 256;
    __shared__ __align__(1024) int8_t sa[128 * 32];
    __shared__ __align__(1024) int8_t sb[kN * 32];
    __shared__ uint64_t done;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 128 * 32 / 16; i += blockDim.x)
        reinterpret_cast<int4*>(sa)[i] = make_int4(0x01010101, 0x01010101, 0x01010101, 0x01010101);
    for (int i = threadIdx.x; i < kN * 32 / 16; i += blockDim.x)
        reinterpret_cast<int4*>(sb)[i] = make_int4(0x01010101, 0x01010101, 0x01010101, 0x01010101);
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&done, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 0) ptx::tmem_alloc<512>(&slot);
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = ptx::idesc_i8(128, kN);
        const uint64_t ad = ptx::smem_desc_kmajor(ptx::smem_u32(sa), 128, 256);
        const uint64_t bd = ptx::smem_desc_kmajor(ptx::smem_u32(sb), 128, 256);
        for (int i = 0; i < iters; ++i)
            ptx::mma_i8(tmem + (i & 1) * kN, ad, bd, idesc, i >= 2 ? 1u : 0u);
        ptx::mma_commit(&done);
        ptx::mbar_wait(&done, 0);
    }
    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

}  // namespace pnn_b200

extern "C" int pnn_probe_int8_peak(int iters, double* tops, double* ms) {
    if (iters < 4 || !tops || !ms) return PNN_EINVAL;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    pnn_b200::tc_int8_probe_kernel<<<sms, 128>>>(iters);  // warm-up
    cudaEventRecord(a);
    pnn_b200::tc_int8_probe_kernel<<<sms, 128>>>(iters);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float t = 0;
    cudaEventElapsedTime(&t, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) return PNN_ECUDA;
    *ms = t;
    *tops = 2.0 * 128 * 256 * 32 * double(iters) * sms / (t / 1e3) / 1e12;
    return PNN_OK;
}
