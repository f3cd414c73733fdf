// Programmatic dependent launch (PDL) for the kernels of the training step.
//
// A kernel launched by launch_pdl() may start while its predecessor on the
// stream is still running: its CTAs do their prologue (shared-memory tables,
// mbarrier init, descriptor prefetch) in the predecessor's tail, then block in
// pdl_wait() until the predecessor grid has completed and its memory is
// visible.  Rules for every kernel launched this way:
//   * pdl_wait() on EVERY path, before the first read of global memory a
//     predecessor writes and before the first global write (no early exit
//     ahead of it: a kernel that completes without waiting would let its own
//     successors start before the predecessor finished);
//   * pdl_trigger() early (all CTAs of the grid resident -> the next kernel
//     may launch);
//   * nothing before pdl_wait() but registers, shared memory, TMEM and kernel
//     parameters.
// Both instructions are no-ops for a kernel launched without the attribute.
// PNN_PDL=0 turns the attribute off (A/B experiments).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace pnn_b200 {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* v = getenv("PNN_PDL");
        return v == nullptr || v[0] != '0';
    }();
    return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace pnn_b200
