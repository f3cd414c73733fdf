// C-ABI entry points (include/pnn_b200.h).  Argument validation mirrors the
// reference's checks (tensor_ops.cpp:17-27, 461-466); every error is a status
// code plus a thread-local message.  There is no CPU fallback: if the device
// or a kernel fails, the call fails.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pnn_b200.h"
#include "posit_device.cuh"
#include "quire_gemm.h"
#include "status.h"

using namespace pnn_b200;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

}  // namespace

namespace pnn_b200 {
void set_last_error(const std::string& msg) { g_err = msg; }
int set_status(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
// host_copy.cpp (AVX-512 when the CPU has it)
void host_narrow_codes(const uint64_t* src, void* dst, int64_t n, int code_bytes, uint64_t mask);
void host_widen_codes(const void* src, uint64_t* dst, int64_t n, int code_bytes);
}  // namespace pnn_b200

namespace {

int cuda_fail(cudaError_t e, const char* where) {
    return fail(PNN_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool fmt_ok(int nbits, int es) {
    if (nbits < 2 || nbits > 16 || es < 0 || es > 4) return false;
    const PositFmt f = make_fmt(nbits, es);
    return 2 * f.R <= 56;
}

int check_fmt(int nbits, int es) {
    if (!fmt_ok(nbits, es))
        return fail(PNN_EUNSUPPORTED, "posit(" + std::to_string(nbits) + "," + std::to_string(es) +
                                          ") is not supported by the device kernels");
    return PNN_OK;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Grow-only device scratch for the synchronous host entry points.
constexpr int64_t kHostChunk = int64_t(1) << 22;  // codes per host narrow/widen chunk
constexpr int kEvents = 16;
constexpr int kPanels = 4;  // row panels of the host-entry GEMM (copy/compute pipeline)

// Persistent host worker pool for the synchronous host entry points (the
// reference's ThreadPool::parallel_for role, thread_pool.hpp:21-48: contiguous
// chunks, caller participates).
class HostPool {
public:
    HostPool() {
        unsigned n = std::thread::hardware_concurrency();
        nworkers_ = int(n < 2 ? 1 : (n > 32 ? 32 : n));
        for (int i = 1; i < nworkers_; ++i) threads_.emplace_back([this, i] { loop(i); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> l(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn) {
        if (n <= 0) return;
        if (nworkers_ == 1 || n < 65536) {
            fn(0, n);
            return;
        }
        {
            std::lock_guard<std::mutex> l(mu_);
            fn_ = &fn;
            n_ = n;
            pending_ = nworkers_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        fn(0, n / nworkers_);
        std::unique_lock<std::mutex> l(mu_);
        done_cv_.wait(l, [this] { return pending_ == 0; });
        fn_ = nullptr;
    }

private:
    void loop(int idx) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int64_t, int64_t)>* fn;
            int64_t n;
            {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                fn = fn_;
                n = n_;
            }
            (*fn)(n * idx / nworkers_, n * (idx + 1) / nworkers_);
            std::lock_guard<std::mutex> l(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    int nworkers_ = 1;
    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int64_t, int64_t)>* fn_ = nullptr;
    int64_t n_ = 0;
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

HostPool& host_pool() {
    static HostPool pool;
    return pool;
}

struct Scratch {
    std::mutex mu;
    void* ptr = nullptr;
    size_t bytes = 0;
    void* hptr = nullptr;
    size_t hbytes = 0;
    cudaStream_t stream = nullptr;   // GEMMs
    cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the host entry
    cudaEvent_t ev[kEvents] = {};
    cudaEvent_t evB = nullptr, evA[kPanels] = {}, evG[kPanels] = {};
    void* reserve_host(size_t n) {
        if (n <= hbytes) return hptr;
        if (hptr) cudaFreeHost(hptr);
        hptr = nullptr;
        hbytes = 0;
        if (cudaHostAlloc(&hptr, n, cudaHostAllocDefault) != cudaSuccess) return nullptr;
        hbytes = n;
        return hptr;
    }
    void* reserve(size_t n) {
        if (n <= bytes) return ptr;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        if (cudaMalloc(&ptr, n) != cudaSuccess) return nullptr;
        bytes = n;
        return ptr;
    }
};
Scratch g_scratch;

__global__ void narrow_codes_kernel(const uint64_t* __restrict__ src, void* __restrict__ dst,
                                    int64_t n, int code_bytes, uint64_t mask) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t c = src[i] & mask;
        if (code_bytes == 1) static_cast<uint8_t*>(dst)[i] = uint8_t(c);
        else static_cast<uint16_t*>(dst)[i] = uint16_t(c);
    }
}

__global__ void widen_codes_kernel(const void* __restrict__ src, uint64_t* __restrict__ dst,
                                   int64_t n, int code_bytes) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        dst[i] = code_bytes == 1 ? uint64_t(static_cast<const uint8_t*>(src)[i])
                                 : uint64_t(static_cast<const uint16_t*>(src)[i]);
    }
}

int blocks_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 32) b = 148 * 32;
    return int(b < 1 ? 1 : b);
}

__global__ void decode_x_kernel(const uint32_t* codes, int64_t n, PositFmt f, int64_t* X,
                                uint8_t* nar) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        int64_t x;
        nar[i] = decode_x(codes[i], f, x) ? 1 : 0;
        X[i] = x;
    }
}

__global__ void quire_round_kernel(const uint64_t* q, int64_t n, PositFmt f, uint32_t* codes) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const unsigned __int128 v = (unsigned __int128)q[2 * i] | ((unsigned __int128)q[2 * i + 1] << 64);
        codes[i] = f.nbits <= 16 ? quire_word_to_posit(f, v) : quire_to_posit(f, v);
    }
}

__global__ void pack_round_kernel(const int32_t* neg, const int32_t* scale, const uint64_t* sig,
                                  const int32_t* sticky, int64_t n, PositFmt f, uint32_t* codes) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (f.nbits <= 16)
            codes[i] = pack_round32(f, neg[i] != 0, scale[i], uint32_t(sig[i] >> 32),
                                    sticky[i] != 0 || uint32_t(sig[i]) != 0);
        else
            codes[i] = pack_round(f, neg[i] != 0, scale[i], sig[i], sticky[i] != 0);
    }
}

int gemm_common(int nbits, int es, const void* A, const void* B, void* C, int64_t M, int64_t N,
                int64_t K, int64_t max_kb, void* ws, size_t ws_bytes, void* stream) {
    if (int rc = check_fmt(nbits, es)) return rc;
    if (M < 0 || N < 0 || K < 0) return fail(PNN_EINVAL, "matmul: negative dimension");
    if (M == 0 || N == 0) return PNN_OK;
    const int cb = nbits <= 8 ? 1 : 2;
    if (K == 0) {  // reference returns an all-zero tensor (tensor_ops.cpp:467)
        cudaError_t e = cudaMemsetAsync(C, 0, size_t(M * N) * cb, as_stream(stream));
        return e == cudaSuccess ? PNN_OK : cuda_fail(e, "matmul memset");
    }
    if (!A || !B || !C) return fail(PNN_EINVAL, "matmul: null pointer");
    int rc = quire_gemm_launch(nbits, es, A, B, C, M, N, K, K, N, N, ws, ws_bytes, max_kb,
                               as_stream(stream), nullptr);
    if (rc == 3) return fail(PNN_EWORKSPACE, "matmul: workspace too small");
    if (rc == 2) return fail(PNN_EUNSUPPORTED, "matmul: format not supported");
    if (rc == 4) return cuda_fail(cudaGetLastError(), "matmul launch");
    return rc;
}

}  // namespace

extern "C" {

const char* pnn_last_error(void) { return g_err.c_str(); }

int pnn_abi_version(void) { return 1; }

int pnn_format_supported(int nbits, int es) { return fmt_ok(nbits, es) ? 1 : 0; }

int pnn_code_bytes(int nbits) { return nbits <= 8 ? 1 : 2; }

int pnn_quire_gemm_workspace(int nbits, int es, int64_t M, int64_t N, int64_t K, size_t* bytes) {
    if (int rc = check_fmt(nbits, es)) return rc;
    if (M < 0 || N < 0 || K < 0 || !bytes) return fail(PNN_EINVAL, "matmul: bad arguments");
    QuireGemmPlan p;
    if (M == 0 || N == 0 || K == 0) {
        *bytes = 0;
        return PNN_OK;
    }
    if (quire_gemm_plan(nbits, es, M, N, K, 0, &p)) return fail(PNN_EUNSUPPORTED, "format");
    *bytes = p.workspace_bytes;
    return PNN_OK;
}

int pnn_quire_gemm(int nbits, int es, const void* A, const void* B, void* C, int64_t M, int64_t N,
                   int64_t K, void* workspace, size_t workspace_bytes, void* stream) {
    return gemm_common(nbits, es, A, B, C, M, N, K, 0, workspace, workspace_bytes, stream);
}

int pnn_quire_gemm_splitk(int nbits, int es, const void* A, const void* B, void* C, int64_t M,
                          int64_t N, int64_t K, int64_t max_kblocks, void* workspace,
                          size_t workspace_bytes, void* stream) {
    if (max_kblocks < 1) return fail(PNN_EINVAL, "splitk: max_kblocks must be >= 1");
    return gemm_common(nbits, es, A, B, C, M, N, K, max_kblocks, workspace, workspace_bytes,
                       stream);
}

int pnn_quire_gemm_profiled(int nbits, int es, const void* A, const void* B, void* C, int64_t M,
                            int64_t N, int64_t K, void* workspace, size_t workspace_bytes,
                            void* stream, float* ms) {
    if (int rc = check_fmt(nbits, es)) return rc;
    if (M <= 0 || N <= 0 || K <= 0 || !A || !B || !C || !ms)
        return fail(PNN_EINVAL, "profiled gemm: bad arguments");
    QuireGemmStats stats;
    for (auto& e : stats.ev) cudaEventCreate(&e);
    cudaStream_t st = as_stream(stream);
    int rc = quire_gemm_launch(nbits, es, A, B, C, M, N, K, K, N, N, workspace, workspace_bytes, 0,
                               st, &stats);
    if (rc == 0) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = cuda_fail(e, "profiled gemm sync");
        else
            for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&ms[i], stats.ev[i], stats.ev[i + 1]);
    } else {
        rc = fail(rc, "profiled gemm launch failed");
    }
    for (auto& e : stats.ev) cudaEventDestroy(e);
    return rc;
}

int pnn_matmul_host(int nbits, int es, const uint64_t* A, const uint64_t* B, uint64_t* C,
                    int64_t M, int64_t K, int64_t N) {
    if (int rc = check_fmt(nbits, es)) return rc;
    if (M < 0 || N < 0 || K < 0) return fail(PNN_EINVAL, "matmul: negative dimension");
    if (M == 0 || N == 0) return PNN_OK;
    if (K == 0) {
        std::memset(C, 0, size_t(M * N) * 8);
        return PNN_OK;
    }
    std::lock_guard<std::mutex> lock(g_scratch.mu);
    if (!g_scratch.stream) {
        for (cudaStream_t* sp : {&g_scratch.stream, &g_scratch.h2d, &g_scratch.d2h})
            if (cudaError_t e = cudaStreamCreateWithFlags(sp, cudaStreamNonBlocking))
                return cuda_fail(e, "stream");
        for (auto& ev : g_scratch.ev)
            if (cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming))
                return cuda_fail(e, "event");
        for (int i = 0; i < kPanels; ++i)
            for (cudaEvent_t* ep : {&g_scratch.evA[i], &g_scratch.evG[i]})
                if (cudaError_t e = cudaEventCreateWithFlags(ep, cudaEventDisableTiming))
                    return cuda_fail(e, "event");
        if (cudaError_t e = cudaEventCreateWithFlags(&g_scratch.evB, cudaEventDisableTiming))
            return cuda_fail(e, "event");
    }
    cudaStream_t st = g_scratch.stream, sh = g_scratch.h2d, sd = g_scratch.d2h;
    QuireGemmPlan p;
    if (quire_gemm_plan(nbits, es, M, N, K, 0, &p)) return fail(PNN_EUNSUPPORTED, "format");
    const int cb = nbits <= 8 ? 1 : 2;
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t pa = al(size_t(M * K) * cb), pb = al(size_t(K * N) * cb), pc = al(size_t(M * N) * cb);
    uint8_t* base = static_cast<uint8_t*>(g_scratch.reserve(pa + pb + pc + p.workspace_bytes));
    uint8_t* hbase = static_cast<uint8_t*>(g_scratch.reserve_host(pa + pb + pc));
    if (!base || !hbase) return fail(PNN_ECUDA, "matmul_host: allocation failed");
    uint8_t *dA = base, *dB = base + pa, *dC = base + pa + pb, *ws = base + pa + pb + pc;
    uint8_t *hA = hbase, *hB = hbase + pa, *hC = hbase + pa + pb;
    const uint64_t mask = (uint64_t(1) << nbits) - 1;
    HostPool& pool = host_pool();
    cudaError_t e;
    // Host threads narrow the uint64 Tensor storage (tensor.hpp:10-14) to packed
    // codes chunk by chunk; each chunk's H2D copy (copy stream) overlaps the
    // next chunk's narrowing.
    auto upload = [&](const uint64_t* src, uint8_t* hdst, uint8_t* ddst, int64_t n) -> cudaError_t {
        for (int64_t c0 = 0; c0 < n; c0 += kHostChunk) {
            const int64_t c1 = std::min(n, c0 + kHostChunk);
            pool.parallel_for(c1 - c0, [&](int64_t lo, int64_t hi) {
                host_narrow_codes(src + c0 + lo, hdst + (c0 + lo) * cb, hi - lo, cb, mask);
            });
            if (cudaError_t err = cudaMemcpyAsync(ddst + c0 * cb, hdst + c0 * cb, size_t(c1 - c0) * cb,
                                                  cudaMemcpyHostToDevice, sh))
                return err;
        }
        return cudaSuccess;
    };
    static const bool prof = getenv("PNN_HOST_PROFILE") != nullptr;  // phase times to stderr
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t0 = now();
    // Row panels: GEMM of panel i runs while the host narrows panel i+1 of A,
    // and while it widens the results of earlier panels (three streams).
    const int P = M >= 1024 ? kPanels : 1;
    const int64_t rows = (M + P - 1) / P;
    if ((e = upload(B, hB, dB, K * N))) return cuda_fail(e, "H2D B");
    cudaEventRecord(g_scratch.evB, sh);
    cudaStreamWaitEvent(st, g_scratch.evB, 0);
    for (int i = 0; i < P; ++i) {
        const int64_t r0 = i * rows, r1 = std::min(M, r0 + rows);
        if (r0 >= r1) break;
        if ((e = upload(A + r0 * K, hA + r0 * K * cb, dA + r0 * K * cb, (r1 - r0) * K)))
            return cuda_fail(e, "H2D A");
        cudaEventRecord(g_scratch.evA[i], sh);
        cudaStreamWaitEvent(st, g_scratch.evA[i], 0);
        int rc = quire_gemm_launch(nbits, es, dA + r0 * K * cb, dB, dC + r0 * N * cb, r1 - r0, N, K, K, N, N,
                                   ws, p.workspace_bytes, 0, st, nullptr);
        if (rc) return rc == 4 ? cuda_fail(cudaGetLastError(), "matmul launch") : fail(rc, "matmul");
        cudaEventRecord(g_scratch.evG[i], st);
    }
    const auto t1 = now();
    // D2H per panel (after its GEMM) in chunks; widen chunk j on the host while
    // chunk j+1 is in flight.
    for (int i = 0; i < P; ++i) {
        const int64_t r0 = i * rows, r1 = std::min(M, r0 + rows);
        if (r0 >= r1) break;
        cudaStreamWaitEvent(sd, g_scratch.evG[i], 0);
        const int64_t off = r0 * N, n = (r1 - r0) * N;
        const int64_t nch = (n + kHostChunk - 1) / kHostChunk;
        for (int64_t c = 0; c < nch; c += kEvents) {
            const int64_t cend = std::min(nch, c + kEvents);
            for (int64_t k = c; k < cend; ++k) {
                const int64_t c0 = off + k * kHostChunk, c1 = std::min(off + n, c0 + kHostChunk);
                if ((e = cudaMemcpyAsync(hC + c0 * cb, dC + c0 * cb, size_t(c1 - c0) * cb,
                                         cudaMemcpyDeviceToHost, sd)))
                    return cuda_fail(e, "D2H C");
                cudaEventRecord(g_scratch.ev[k - c], sd);
            }
            for (int64_t k = c; k < cend; ++k) {
                if ((e = cudaEventSynchronize(g_scratch.ev[k - c]))) return cuda_fail(e, "D2H sync");
                const int64_t c0 = off + k * kHostChunk, c1 = std::min(off + n, c0 + kHostChunk);
                pool.parallel_for(c1 - c0, [&](int64_t lo, int64_t hi) {
                    host_widen_codes(hC + (c0 + lo) * cb, C + c0 + lo, hi - lo, cb);
                });
            }
        }
    }
    for (cudaStream_t s2 : {sh, st, sd})
        if ((e = cudaStreamSynchronize(s2))) return cuda_fail(e, "matmul_host sync");
    if (prof) {
        const auto t2 = now();
        fprintf(stderr, "[pnn_matmul_host] narrow+H2D+GEMM issue %.2f ms, D2H+widen %.2f ms\n",
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
    return PNN_OK;
}

int pnn_decode_x(int nbits, int es, const uint32_t* codes, int64_t n, int64_t* X, uint8_t* nar,
                 void* stream) {
    if (int rc = check_fmt(nbits, es)) return rc;
    if (n <= 0) return PNN_OK;
    decode_x_kernel<<<blocks_for(n), 256, 0, as_stream(stream)>>>(codes, n, make_fmt(nbits, es), X,
                                                                   nar);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PNN_OK : cuda_fail(e, "decode_x");
}

int pnn_quire_round(int nbits, int es, const uint64_t* q, int64_t n, uint32_t* codes,
                    void* stream) {
    if (int rc = check_fmt(nbits, es)) return rc;
    if (n <= 0) return PNN_OK;
    quire_round_kernel<<<blocks_for(n), 256, 0, as_stream(stream)>>>(q, n, make_fmt(nbits, es),
                                                                      codes);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PNN_OK : cuda_fail(e, "quire_round");
}

int pnn_pack_round(int nbits, int es, const int32_t* neg, const int32_t* scale,
                   const uint64_t* sig, const int32_t* sticky, int64_t n, uint32_t* codes,
                   void* stream) {
    if (nbits < 2 || nbits > 32 || es < 0 || es > 4)
        return fail(PNN_EUNSUPPORTED, "pack_round: bad format");
    if (n <= 0) return PNN_OK;
    pack_round_kernel<<<blocks_for(n), 256, 0, as_stream(stream)>>>(neg, scale, sig, sticky, n,
                                                                     make_fmt(nbits, es), codes);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PNN_OK : cuda_fail(e, "pack_round");
}

}  // extern "C"
