// Data-parallel gradient reduction on exact quire words.
//
// Each rank emits, per parameter, the UNROUNDED W-bit quire of its batch
// shard (conv2d_weight_grad / conv2d_bias_grad / the loss sum in raw mode).
// The quire is exact and addition mod 2^W is associative, so summing the
// ranks' quires and rounding once is bit-identical to the single-process
// reference for any rank count and order.  Integer all-reduce (NCCL int64
// SUM) does not carry between words, so a W-bit value v is split into
// L = ceil(W/60) 60-bit digits in int64 lanes: <= 8 ranks * (2^60 - 1) < 2^63
// never wraps.  One extra lane carries the NaR flag (summed, > 0 == NaR).
//   lanes layout: [n][L + 1] int64, lane L = NaR count.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/pnn_b200.h"
#include "posit_device.cuh"
#include "status.h"

namespace pnn_b200 {

__global__ void quire_to_lanes_kernel(const unsigned __int128* __restrict__ words,
                                      const uint8_t* __restrict__ nar, int64_t n, int L, int W,
                                      uint64_t* __restrict__ lanes) {
    const unsigned __int128 one = 1;
    const unsigned __int128 wmask = W >= 128 ? ~(unsigned __int128)0 : ((one << W) - 1);
    const uint64_t dmask = (uint64_t(1) << 60) - 1;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const unsigned __int128 v = words[i] & wmask;
        uint64_t* out = lanes + i * (L + 1);
        for (int l = 0; l < L; ++l) out[l] = uint64_t(v >> (60 * l)) & dmask;
        out[L] = nar[i] ? 1 : 0;
    }
}

template <typename CodeT>
__global__ void lanes_to_posit_kernel(const uint64_t* __restrict__ lanes, int64_t n, int L,
                                      PositFmt f, CodeT* __restrict__ codes,
                                      unsigned __int128* __restrict__ words_out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t* in = lanes + i * (L + 1);
        unsigned __int128 v = 0;
        for (int l = 0; l < L; ++l) v += (unsigned __int128)in[l] << (60 * l);  // carries resolve here
        if (words_out) words_out[i] = v;
        if (codes) codes[i] = CodeT(in[L] ? (1u << (f.nbits - 1)) : quire_word_to_posit(f, v));
    }
}

}  // namespace pnn_b200

using namespace pnn_b200;

extern "C" {

int pnn_quire_lanes(int nbits, int es) {
    if (nbits < 2 || nbits > 16 || es < 0 || es > 4) return 0;
    const int W = make_fmt(nbits, es).W;
    return W > 128 ? 0 : (W + 59) / 60;
}

int pnn_quire_to_lanes(int nbits, int es, const void* words, const uint8_t* nar, int64_t n,
                       uint64_t* lanes, void* stream) {
    const int L = pnn_quire_lanes(nbits, es);
    if (L == 0) return set_status(PNN_EUNSUPPORTED, "quire_to_lanes: format not supported");
    if (n < 0 || (n > 0 && (!words || !nar || !lanes)))
        return set_status(PNN_EINVAL, "quire_to_lanes: bad arguments");
    if (n == 0) return PNN_OK;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    quire_to_lanes_kernel<<<int(blocks), 256, 0, (cudaStream_t)stream>>>(
        static_cast<const unsigned __int128*>(words), nar, n, L, make_fmt(nbits, es).W, lanes);
    return cudaGetLastError() == cudaSuccess ? PNN_OK : set_status(PNN_ECUDA, "quire_to_lanes");
}

int pnn_lanes_to_posit(int nbits, int es, const uint64_t* lanes, int64_t n, void* codes,
                       void* words_out, void* stream) {
    const int L = pnn_quire_lanes(nbits, es);
    if (L == 0) return set_status(PNN_EUNSUPPORTED, "lanes_to_posit: format not supported");
    if (n < 0 || (n > 0 && !lanes)) return set_status(PNN_EINVAL, "lanes_to_posit: bad arguments");
    if (n == 0) return PNN_OK;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    const PositFmt f = make_fmt(nbits, es);
    auto* w = static_cast<unsigned __int128*>(words_out);
    if (nbits <= 8)
        lanes_to_posit_kernel<uint8_t><<<int(blocks), 256, 0, (cudaStream_t)stream>>>(
            lanes, n, L, f, static_cast<uint8_t*>(codes), w);
    else
        lanes_to_posit_kernel<uint16_t><<<int(blocks), 256, 0, (cudaStream_t)stream>>>(
            lanes, n, L, f, static_cast<uint16_t*>(codes), w);
    return cudaGetLastError() == cudaSuccess ? PNN_OK : set_status(PNN_ECUDA, "lanes_to_posit");
}

}  // extern "C"
