// Host-side narrowing / widening between the reference's Tensor storage (one
// posit code per uint64_t, tensor.hpp:10-14) and packed 8/16-bit codes, for the
// host entry points (pnn_matmul_host).  These loops are host-memory bound:
// AVX-512 truncating moves (VPMOVQB / VPMOVQW) and zero-extending loads with
// non-temporal 64-byte stores for the wide output (no read-for-ownership of the
// uint64 destination), chosen at run time; a portable loop otherwise.
#include <immintrin.h>

#include <cstdint>

namespace pnn_b200 {

namespace {

__attribute__((target("avx512f,avx512bw"))) void narrow_avx512(const uint64_t* src, void* dst,
                                                                 int64_t n, int cb, uint64_t mask) {
    const __m512i m = _mm512_set1_epi64(int64_t(mask));
    int64_t i = 0;
    if (cb == 1) {
        auto* d = static_cast<uint8_t*>(dst);
        for (; i + 8 <= n; i += 8) {
            const __m512i v = _mm512_and_si512(_mm512_loadu_si512(src + i), m);
            _mm_storel_epi64(reinterpret_cast<__m128i*>(d + i), _mm512_cvtepi64_epi8(v));
        }
        for (; i < n; ++i) d[i] = uint8_t(src[i] & mask);
    } else {
        auto* d = static_cast<uint16_t*>(dst);
        for (; i + 8 <= n; i += 8) {
            const __m512i v = _mm512_and_si512(_mm512_loadu_si512(src + i), m);
            _mm_storeu_si128(reinterpret_cast<__m128i*>(d + i), _mm512_cvtepi64_epi16(v));
        }
        for (; i < n; ++i) d[i] = uint16_t(src[i] & mask);
    }
}

__attribute__((target("avx512f,avx512bw"))) void widen_avx512(const void* src, uint64_t* dst,
                                                                int64_t n, int cb) {
    int64_t i = 0;
    // scalar head until the destination is 64-byte aligned (streaming stores)
    while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 63)) {
        dst[i] = cb == 1 ? static_cast<const uint8_t*>(src)[i] : static_cast<const uint16_t*>(src)[i];
        ++i;
    }
    if (cb == 1) {
        const auto* s = static_cast<const uint8_t*>(src);
        for (; i + 8 <= n; i += 8)
            _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i),
                                _mm512_cvtepu8_epi64(_mm_loadl_epi64(reinterpret_cast<const __m128i*>(s + i))));
        for (; i < n; ++i) dst[i] = s[i];
    } else {
        const auto* s = static_cast<const uint16_t*>(src);
        for (; i + 8 <= n; i += 8)
            _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i),
                                _mm512_cvtepu16_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i))));
        for (; i < n; ++i) dst[i] = s[i];
    }
    _mm_sfence();
}

bool have_avx512() {
    static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
    return ok;
}

}  // namespace

// dst[i] = code bits of src[i] (1 or 2 bytes per code)
void host_narrow_codes(const uint64_t* src, void* dst, int64_t n, int code_bytes, uint64_t mask) {
    if (have_avx512()) return narrow_avx512(src, dst, n, code_bytes, mask);
    if (code_bytes == 1)
        for (int64_t i = 0; i < n; ++i) static_cast<uint8_t*>(dst)[i] = uint8_t(src[i] & mask);
    else
        for (int64_t i = 0; i < n; ++i) static_cast<uint16_t*>(dst)[i] = uint16_t(src[i] & mask);
}

// dst[i] = zero-extended code src[i]
void host_widen_codes(const void* src, uint64_t* dst, int64_t n, int code_bytes) {
    if (have_avx512()) return widen_avx512(src, dst, n, code_bytes);
    if (code_bytes == 1)
        for (int64_t i = 0; i < n; ++i) dst[i] = static_cast<const uint8_t*>(src)[i];
    else
        for (int64_t i = 0; i < n; ++i) dst[i] = static_cast<const uint16_t*>(src)[i];
}

}  // namespace pnn_b200
