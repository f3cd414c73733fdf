// maxpool2d_backward(dy, argmax, x_shape) with the reference's exact,
// window-independent semantics (proj/src/tensor_ops.cpp:658-670):
//
//     dx = 0;  for i in 0..n_out-1 (ascending):  dx[argmax[i]] = add(dx[argmax[i]], dy[i])
//
// The argmax may point anywhere in dx (any window, overlapping windows, or an
// argmax not produced by maxpool2d at all).  Posit addition is not associative,
// so a target hit by several outputs must add them in increasing output order.
// Device plan (no atomics on the values, deterministic):
//   1. key[i] = argmax[i] (int32; out-of-range -> n_in, which sorts last and is
//      dropped), val[i] = i;
//   2. stable LSD radix sort of (key, val) over ceil(log2(n_in + 1)) key bits
//      (cub::DeviceRadixSort -- stability keeps every target's outputs in
//      ascending i);
//   3. dx = 0; the first position of each key run sums its run sequentially
//      with p_add (add(0, v) == v, NaR sticky) and stores dx[key].
// Out-of-range indices are undefined behaviour in the reference; the host
// mirrors (ops.py, host_ops.cpp) reject them with invalid_argument before the
// call, and the kernel ignores them.
#include <cuda_runtime.h>

#include <cstdint>
#include <cub/device/device_radix_sort.cuh>

#include "../../include/pnn_b200.h"
#include "eltwise_common.cuh"
#include "posit_scalar.cuh"
#include "status.h"

namespace pnn_b200 {

__global__ void scatter_keys_kernel(const int64_t* __restrict__ argmax, int64_t n_out, int32_t n_in,
                                    int32_t* __restrict__ key, int32_t* __restrict__ val) {
    GRID_STRIDE(i, n_out) {
        const int64_t t = argmax[i];
        key[i] = (t >= 0 && t < n_in) ? int32_t(t) : n_in;
        val[i] = int32_t(i);
    }
}

__global__ void scatter_runs_kernel(PositFmt f, int b, const void* __restrict__ dy,
                                    const int32_t* __restrict__ key, const int32_t* __restrict__ val,
                                    int64_t n_out, int32_t n_in, void* __restrict__ dx) {
    GRID_STRIDE(j, n_out) {
        const int32_t t = key[j];
        if (t == n_in || (j > 0 && key[j - 1] == t)) continue;  // dropped, or not a run head
        uint32_t acc = load_any(dy, val[j], b);                 // add(0, v) == v
        for (int64_t k = j + 1; k < n_out && key[k] == t; ++k)
            acc = p_add(f, acc, load_any(dy, val[k], b));
        store_any(dx, t, b, acc);
    }
}

}  // namespace pnn_b200

using namespace pnn_b200;

namespace {

struct ScatterLayout {
    size_t key_in, val_in, key_out, val_out, temp, temp_bytes, total;
};

int key_bits(int64_t n_in) {
    int bits = 1;
    while (bits < 32 && (int64_t(1) << bits) <= n_in) ++bits;  // n_in itself must fit (sentinel)
    return bits;
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

int scatter_layout(int64_t n_out, int64_t n_in, ScatterLayout* L) {
    const size_t a = align256(size_t(n_out) * 4);
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, (const int32_t*)nullptr, (int32_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, int(n_out), 0,
                                    key_bits(n_in));
    L->key_in = 0;
    L->val_in = a;
    L->key_out = 2 * a;
    L->val_out = 3 * a;
    L->temp = 4 * a;
    L->temp_bytes = temp;
    L->total = 4 * a + align256(temp);
    return PNN_OK;
}

bool scatter_fmt_ok(int nbits, int es) {
    if (nbits < 2 || nbits > 16 || es < 0 || es > 4) return false;
    return 2 * make_fmt(nbits, es).R <= 96;
}

}  // namespace

extern "C" {

int pnn_maxpool2d_bwd_scatter_workspace(int64_t n_out, int64_t n_in, size_t* bytes) {
    if (!bytes || n_out < 0 || n_in < 0) return set_status(PNN_EINVAL, "maxpool2d_backward: bad sizes");
    if (n_out >= (int64_t(1) << 31) || n_in >= (int64_t(1) << 31) - 1)
        return set_status(PNN_EUNSUPPORTED, "maxpool2d_backward scatter: sizes >= 2^31");
    ScatterLayout L;
    scatter_layout(n_out, n_in, &L);
    *bytes = L.total;
    return PNN_OK;
}

int pnn_maxpool2d_bwd_scatter(int nbits, int es, const void* dy, const int64_t* argmax, int64_t n_out,
                              void* dx, int64_t n_in, void* workspace, size_t workspace_bytes,
                              void* stream) {
    if (!scatter_fmt_ok(nbits, es)) return set_status(PNN_EUNSUPPORTED, "format not supported");
    size_t need = 0;
    if (int rc = pnn_maxpool2d_bwd_scatter_workspace(n_out, n_in, &need)) return rc;
    if ((n_out && (!dy || !argmax)) || (n_in && !dx))
        return set_status(PNN_EINVAL, "maxpool2d_backward: null buffer");
    if (workspace_bytes < need || (need && !workspace))
        return set_status(PNN_EWORKSPACE, "maxpool2d_backward: workspace too small");
    auto st = static_cast<cudaStream_t>(stream);
    const int b = nbits <= 8 ? 1 : 2;
    if (n_in == 0) return PNN_OK;
    cudaError_t e = cudaMemsetAsync(dx, 0, size_t(n_in) * b, st);
    if (e != cudaSuccess) return set_status(PNN_ECUDA, std::string("maxpool2d_backward: ") + cudaGetErrorString(e));
    if (n_out == 0) return PNN_OK;
    ScatterLayout L;
    scatter_layout(n_out, n_in, &L);
    auto* w = static_cast<uint8_t*>(workspace);
    auto* key_in = reinterpret_cast<int32_t*>(w + L.key_in);
    auto* val_in = reinterpret_cast<int32_t*>(w + L.val_in);
    auto* key_out = reinterpret_cast<int32_t*>(w + L.key_out);
    auto* val_out = reinterpret_cast<int32_t*>(w + L.val_out);
    int64_t blocks = (n_out + 255) / 256;
    const int grid = int(blocks > 148 * 16 ? 148 * 16 : blocks);
    scatter_keys_kernel<<<grid, 256, 0, st>>>(argmax, n_out, int32_t(n_in), key_in, val_in);
    size_t temp = L.temp_bytes;
    e = cub::DeviceRadixSort::SortPairs(w + L.temp, temp, key_in, key_out, val_in, val_out, int(n_out), 0,
                                        key_bits(n_in), st);
    if (e != cudaSuccess) return set_status(PNN_ECUDA, std::string("maxpool2d_backward sort: ") + cudaGetErrorString(e));
    scatter_runs_kernel<<<grid, 256, 0, st>>>(make_fmt(nbits, es), b, dy, key_out, val_out, n_out,
                                              int32_t(n_in), dx);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_status(PNN_ECUDA, std::string("maxpool2d_backward: ") + cudaGetErrorString(e));
    return PNN_OK;
}

}  // extern "C"
