// Host memory bandwidth probe for the e2e host path: per thread count, the
// rate of (a) reading uint64 storage (sum), (b) narrowing uint64 -> uint16,
// (c) widening uint16 -> uint64 with streaming stores.  Build:
//   g++ -O3 -march=x86-64-v3 -mavx512f -mavx512bw -pthread hostbw.cpp -o hostbw
#include <immintrin.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char** argv) {
    const int64_t n = int64_t(1) << 25;  // 32 M codes = 256 MiB of uint64
    uint64_t* big = static_cast<uint64_t*>(aligned_alloc(64, n * 8));
    uint16_t* small = static_cast<uint16_t*>(aligned_alloc(64, n * 2));
    for (int64_t i = 0; i < n; ++i) big[i] = i & 0xFFFF;
    memset(small, 1, n * 2);
    const int maxT = std::thread::hardware_concurrency();
    printf("hardware_concurrency %d\n", maxT);
    std::vector<int> ts = {1, 2, 4, 8, 12, 16, 24, 32, 48, 64};
    for (int T : ts) {
        if (T > maxT) break;
        double best[3] = {1e9, 1e9, 1e9};
        volatile uint64_t sink = 0;
        for (int rep = 0; rep < 4; ++rep) {
            for (int kind = 0; kind < 3; ++kind) {
                std::vector<std::thread> th;
                std::vector<uint64_t> sums(T);
                double t0 = now();
                for (int t = 0; t < T; ++t)
                    th.emplace_back([&, t] {
                        int64_t lo = n * t / T, hi = n * (t + 1) / T;
                        lo &= ~int64_t(7);
                        hi = t == T - 1 ? n : hi & ~int64_t(7);
                        if (kind == 0) {
                            __m512i acc = _mm512_setzero_si512();
                            for (int64_t i = lo; i < hi; i += 8) acc = _mm512_add_epi64(acc, _mm512_load_si512(big + i));
                            sums[t] = _mm512_reduce_add_epi64(acc);
                        } else if (kind == 1) {
                            for (int64_t i = lo; i < hi; i += 8)
                                _mm_storeu_si128(reinterpret_cast<__m128i*>(small + i),
                                                 _mm512_cvtepi64_epi16(_mm512_load_si512(big + i)));
                        } else {
                            for (int64_t i = lo; i < hi; i += 8)
                                _mm512_stream_si512(reinterpret_cast<__m512i*>(big + i),
                                                    _mm512_cvtepu16_epi64(_mm_loadu_si128(
                                                        reinterpret_cast<const __m128i*>(small + i))));
                            _mm_sfence();
                        }
                    });
                for (auto& x : th) x.join();
                double dt = now() - t0;
                if (dt < best[kind]) best[kind] = dt;
                for (auto s : sums) sink += s;
            }
        }
        printf("T=%2d  read u64 %6.1f GB/s   narrow(u64->u16) %6.1f GB/s of u64   widen(u16->u64 NT) %6.1f GB/s of u64\n",
               T, n * 8 / best[0] / 1e9, n * 8 / best[1] / 1e9, n * 8 / best[2] / 1e9);
    }
    return 0;
}
