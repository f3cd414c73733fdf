// Process-lifetime device tables (code -> digits, code -> integer image,
// code -> code): built once per key on the caller's stream, outside stream
// capture, then reused by every later launch -- a CUDA-graph replay finds them
// resident and runs no table-building kernel.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <functional>

namespace pnn_b200 {

// Table for `key` (bytes long), built by build(ptr, st) the first time.
// Returns nullptr while `st` is capturing and the table does not exist yet, or
// on an allocation / launch error; callers then fall back to their per-call
// table in the workspace.
void* persistent_table(uint64_t key, size_t bytes, cudaStream_t st,
                       const std::function<void(void*, cudaStream_t)>& build);

// kind and five small parameters (formats, digit counts) plus a 16-bit code
inline uint64_t table_key(int kind, int a, int b, int c, int d, int e, uint32_t x = 0) {
    return (uint64_t(kind & 0xFF) << 56) | (uint64_t(a & 0xFF) << 48) | (uint64_t(b & 0xFF) << 40) |
           (uint64_t(c & 0xFF) << 32) | (uint64_t(d & 0xFF) << 24) | (uint64_t(e & 0xFF) << 16) |
           uint64_t(x & 0xFFFFu);
}

}  // namespace pnn_b200
