// Division by a launch-constant divisor without the ~20-instruction integer
// division sequence: q = (umulhi(n, m) + n) >> l with l = ceil(log2 d) and
// m = floor(2^32 (2^l - d) / d) + 1 (Granlund-Montgomery), exact for every
// n < 2^31 (the planners keep indices below 2^31).
#pragma once

#include <cstdint>

namespace pnn_b200 {

struct FastDiv {
    uint32_t m = 1, l = 0, d = 1;
    FastDiv() = default;
    __host__ explicit FastDiv(uint32_t div) : d(div ? div : 1) {
        while ((uint64_t(1) << l) < d) ++l;
        m = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << l) - d)) / d + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> l; }
    __device__ __forceinline__ void divmod(uint32_t n, uint32_t& q, uint32_t& r) const {
        q = div(n);
        r = n - q * d;
    }
};

}  // namespace pnn_b200
