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
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pnn_b200.h"
#include "epilogue.cuh"
#include "posit_device.cuh"
#include "quire_gemm.h"
#include "status.h"
#include "tables.h"

using namespace pnn_b200;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

}  // namespace

namespace pnn_b200 {
void* persistent_table(uint64_t key, size_t bytes, cudaStream_t st,
                       const std::function<void(void*, cudaStream_t)>& build) {
    static std::mutex mu;
    static std::map<uint64_t, void*>* cache = new std::map<uint64_t, void*>();  // lives with the process
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache->find(key);
    if (it != cache->end()) return it->second;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (cs != cudaStreamCaptureStatusNone) return nullptr;
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    build(p, st);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) {
        cudaFree(p);
        return nullptr;
    }
    (*cache)[key] = p;
    return p;
}

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
constexpr int kPanels = 4;  // default row panels of the host-entry GEMM (copy/compute pipeline)
constexpr int kMaxPanels = 16;

// Persistent host worker pool for the synchronous host entry points (the
// reference's ThreadPool::parallel_for role, thread_pool.hpp:21-48: contiguous
// chunks, caller participates).
class HostPool {
public:
    HostPool() {
        unsigned n = std::thread::hardware_concurrency();
        if (const char* v = getenv("PNN_HOST_THREADS")) n = unsigned(atoi(v) > 0 ? atoi(v) : 1);
        nworkers_ = int(n < 2 ? 1 : (n > 64 ? 64 : n));
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

    int workers() const { return nworkers_; }

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
    cudaStream_t stream = nullptr;                  // GEMMs + narrow / widen kernels
    cudaStream_t h2d = nullptr, d2h = nullptr;      // packed-code copies (host-narrowed rows)
    cudaStream_t h2d_raw = nullptr, d2h_raw = nullptr;  // uint64 copies (device-narrowed rows)
    cudaEvent_t ev[kEvents] = {};
    cudaEvent_t evB = nullptr, evBr = nullptr, evA[kMaxPanels] = {}, evAr[kMaxPanels] = {},
                evG[kMaxPanels] = {};
    bool init() {
        if (stream) return true;
        for (cudaStream_t* sp : {&stream, &h2d, &d2h, &h2d_raw, &d2h_raw})
            if (cudaStreamCreateWithFlags(sp, cudaStreamNonBlocking) != cudaSuccess) return false;
        std::vector<cudaEvent_t*> evs = {&evB, &evBr};
        for (auto& e : ev) evs.push_back(&e);
        for (int i = 0; i < kMaxPanels; ++i)
            for (cudaEvent_t* ep : {&evA[i], &evAr[i], &evG[i]}) evs.push_back(ep);
        for (cudaEvent_t* ep : evs)
            if (cudaEventCreateWithFlags(ep, cudaEventDisableTiming) != cudaSuccess) return false;
        return true;
    }
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

// Device halves of the host-entry copies: rows whose uint64 Tensor storage is
// moved by the copy engine as is (pinned user buffers) are narrowed / widened
// here, so the DMA engines carry part of the host-memory traffic that the host
// threads would otherwise do alone.  n % 2 == 0 handled by the tail loop.
template <typename CodeT>
__global__ void narrow_codes_kernel(const uint64_t* __restrict__ src, CodeT* __restrict__ dst, int64_t n,
                                    uint64_t mask) {
    const int64_t n2 = n / 2;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2;
         i += int64_t(gridDim.x) * blockDim.x) {
        const ulonglong2 v = reinterpret_cast<const ulonglong2*>(src)[i];
        dst[2 * i] = CodeT(v.x & mask);
        dst[2 * i + 1] = CodeT(v.y & mask);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) dst[n - 1] = CodeT(src[n - 1] & mask);
}

template <typename CodeT>
__global__ void widen_codes_kernel(const CodeT* __restrict__ src, uint64_t* __restrict__ dst, int64_t n) {
    const int64_t n2 = n / 2;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2;
         i += int64_t(gridDim.x) * blockDim.x)
        reinterpret_cast<ulonglong2*>(dst)[i] = make_ulonglong2(src[2 * i], src[2 * i + 1]);
    if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) dst[n - 1] = src[n - 1];
}

void launch_narrow(const uint64_t* src, void* dst, int64_t n, int cb, uint64_t mask, cudaStream_t st) {
    if (n <= 0) return;
    const int grid = int(std::min<int64_t>(148 * 8, (n / 2 + 255) / 256 + 1));
    if (cb == 1) narrow_codes_kernel<uint8_t><<<grid, 256, 0, st>>>(src, static_cast<uint8_t*>(dst), n, mask);
    else narrow_codes_kernel<uint16_t><<<grid, 256, 0, st>>>(src, static_cast<uint16_t*>(dst), n, mask);
}

void launch_widen(const void* src, uint64_t* dst, int64_t n, int cb, cudaStream_t st) {
    if (n <= 0) return;
    const int grid = int(std::min<int64_t>(148 * 8, (n / 2 + 255) / 256 + 1));
    if (cb == 1) widen_codes_kernel<uint8_t><<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(src), dst, n);
    else widen_codes_kernel<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(src), dst, n);
}

bool host_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

double env_frac(const char* name, double dflt) {
    const char* v = getenv(name);
    if (!v) return dflt;
    const double x = atof(v);
    return x < 0 ? 0 : (x > 1 ? 1 : x);
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
        int64_t x, xb;
        const bool nr = decode_x(codes[i], f, x);
        // the digitisers' branch-free decode must agree code for code (a
        // mismatch shows as an impossible NaR flag and a poisoned image)
        const bool nb = decode_x_bf(codes[i], f, xb);
        const bool same = nb == nr && xb == x;
        nar[i] = same ? (nr ? 1 : 0) : 2;
        X[i] = same ? x : INT64_MIN;
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

// Reference-facing host entry (matmul over uint64 Tensor storage, tensor.hpp:10-14).
// The call is bound by host-memory traffic (8 bytes per code in, 8 out), so
// three resources share it, each on its own rows:
//   * host threads narrow rows to packed codes in pinned staging (packed H2D)
//     and widen packed results (packed D2H);
//   * when the user buffers are pinned, the copy engines move a fraction of the
//     rows as raw uint64 (H2D of inputs, D2H of results) and the GPU narrows /
//     widens them -- PCIe and the DMA engines add bandwidth the host cores
//     cannot reach on their own;
//   * the GEMM runs per row panel as soon as the panel's A rows (both halves)
//     and all of B are on the device.
// Fractions: PNN_HOST_DMA_IN / PNN_HOST_DMA_OUT (share of rows moved raw),
// PNN_HOST_PANELS; defaults measured on the B200 box.
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
    if (!g_scratch.init()) return cuda_fail(cudaGetLastError(), "matmul_host streams");
    cudaStream_t st = g_scratch.stream, sh = g_scratch.h2d, sd = g_scratch.d2h;
    cudaStream_t shr = g_scratch.h2d_raw, sdr = g_scratch.d2h_raw;
    QuireGemmPlan p;
    if (quire_gemm_plan(nbits, es, M, N, K, 0, &p)) return fail(PNN_EUNSUPPORTED, "format");
    const int cb = nbits <= 8 ? 1 : 2;
    const uint64_t mask = (uint64_t(1) << nbits) - 1;
    // raw (DMA) shares: only for pinned user buffers and large operands
    const bool big = M * K + K * N >= (int64_t(1) << 21);
    // defaults balance PCIe (raw: 8 B per code, packed: cb) against the host
    // threads (8 B per code): f = (8 Rp - cb Rc) / (8 Rp + (8 - cb) Rc) with the
    // box's measured Rp ~ 51 GB/s (pinned H2D) and Rc ~ 100 GB/s (narrowing)
    const double f_in_env = env_frac("PNN_HOST_DMA_IN", cb == 1 ? 0.28 : 0.20);
    const double f_out_env = env_frac("PNN_HOST_DMA_OUT", cb == 1 ? 0.30 : 0.20);
    const double f_in = big && host_pinned(A) && host_pinned(B) ? f_in_env : 0.0;
    const double f_out = big && host_pinned(C) ? f_out_env : 0.0;
    static const int panels_env = [] {
        const char* v = getenv("PNN_HOST_PANELS");
        const int x = v ? atoi(v) : kPanels;
        return x < 1 ? 1 : (x > kMaxPanels ? kMaxPanels : x);
    }();
    const int P = M >= 256 * panels_env ? panels_env : 1;
    const int64_t rows = (M + P - 1) / P;
    const int64_t kc = K - int64_t(double(K) * f_in);  // B rows [0, kc) host-narrowed, [kc, K) raw
    auto split_in = [&](int64_t r0, int64_t r1) { return r1 - int64_t(double(r1 - r0) * f_in); };
    auto split_out = [&](int64_t r0, int64_t r1) { return r1 - int64_t(double(r1 - r0) * f_out); };
    // raw staging: each segment starts 256-byte aligned (vector loads / stores)
    auto seg = [](int64_t n) { return (n + 31) & ~int64_t(31); };
    int64_t raw_in = seg((K - kc) * N), raw_out = 0;
    for (int i = 0; i < P; ++i) {
        const int64_t r0 = i * rows, r1 = std::min(M, r0 + rows);
        if (r0 >= r1) break;
        raw_in += seg((r1 - split_in(r0, r1)) * K);
        raw_out += seg((r1 - split_out(r0, r1)) * N);
    }
    // GEMM workspace: the largest panel plan (a short panel may split K to fill the SMs)
    size_t ws_bytes = 0;
    for (int i = 0; i < P; ++i) {
        const int64_t r0 = i * rows, r1 = std::min(M, r0 + rows);
        if (r0 >= r1) break;
        QuireGemmPlan pp;
        quire_gemm_plan(nbits, es, r1 - r0, N, K, 0, &pp);
        ws_bytes = std::max(ws_bytes, pp.workspace_bytes);
    }
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t pa = al(size_t(M * K) * cb), pb = al(size_t(K * N) * cb), pc = al(size_t(M * N) * cb);
    const size_t pri = al(size_t(raw_in) * 8), pro = al(size_t(raw_out) * 8);
    uint8_t* base = static_cast<uint8_t*>(g_scratch.reserve(pa + pb + pc + pri + pro + ws_bytes));
    uint8_t* hbase = static_cast<uint8_t*>(g_scratch.reserve_host(pa + pb + pc));
    if (!base || !hbase) return fail(PNN_ECUDA, "matmul_host: allocation failed");
    uint8_t *dA = base, *dB = base + pa, *dC = base + pa + pb;
    uint64_t* rin = reinterpret_cast<uint64_t*>(base + pa + pb + pc);
    uint64_t* rout = reinterpret_cast<uint64_t*>(base + pa + pb + pc + pri);
    uint8_t* ws = base + pa + pb + pc + pri + pro;
    uint8_t *hA = hbase, *hB = hbase + pa, *hC = hbase + pa + pb;
    HostPool& pool = host_pool();
    cudaError_t e;
    static const bool prof = getenv("PNN_HOST_PROFILE") != nullptr;  // phase times to stderr
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t0 = now();
    cudaEvent_t tev[2 * kMaxPanels + 1] = {};
    if (prof) {
        for (int i = 0; i <= 2 * P; ++i) cudaEventCreate(&tev[i]);
        cudaEventRecord(tev[0], st);
    }

    // 1. every raw input share goes to the copy engine first (own stream: the
    //    host-narrowed chunks do not queue behind it); the GPU narrows each.
    uint64_t* rcur = rin;
    auto raw_upload = [&](const uint64_t* src, uint8_t* ddst, int64_t n, cudaEvent_t ev) -> cudaError_t {
        if (n > 0) {
            if (cudaError_t err = cudaMemcpyAsync(rcur, src, size_t(n) * 8, cudaMemcpyHostToDevice, shr))
                return err;
        }
        cudaEventRecord(ev, shr);
        cudaStreamWaitEvent(st, ev, 0);
        launch_narrow(rcur, ddst, n, cb, mask, st);
        rcur += seg(n);
        return cudaSuccess;
    };
    if ((e = raw_upload(B + kc * N, dB + kc * N * cb, (K - kc) * N, g_scratch.evBr)))
        return cuda_fail(e, "H2D B raw");
    // (the A raw shares follow B's packed chunks, below)
    // 2. host-narrowed chunks: packed H2D overlaps the next chunk's narrowing
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
    if ((e = upload(B, hB, dB, kc * N))) return cuda_fail(e, "H2D B");
    cudaEventRecord(g_scratch.evB, sh);
    cudaStreamWaitEvent(st, g_scratch.evB, 0);
    // B gates every panel: the A raw shares start once B's packed chunks are
    // queued, so they do not take PCIe bandwidth from B
    cudaStreamWaitEvent(shr, g_scratch.evB, 0);
    // queue all A raw shares now (the copy engine runs ahead of the host threads)
    for (int i = 0; i < P; ++i) {
        const int64_t r0 = i * rows, r1 = std::min(M, r0 + rows);
        if (r0 >= r1) break;
        const int64_t s = split_in(r0, r1);
        if (r1 > s) {
            if ((e = cudaMemcpyAsync(rcur, A + s * K, size_t((r1 - s) * K) * 8, cudaMemcpyHostToDevice, shr)))
                return cuda_fail(e, "H2D A raw");
        }
        cudaEventRecord(g_scratch.evAr[i], shr);
        rcur += seg((r1 - s) * K);
    }
    uint64_t* acur = rin + seg((K - kc) * N);
    QuireGemmPlan p0{};
    uint64_t* ocur = rout;
    for (int i = 0; i < P; ++i) {
        const int64_t r0 = i * rows, r1 = std::min(M, r0 + rows);
        if (r0 >= r1) break;
        const int64_t s = split_in(r0, r1);
        if ((e = upload(A + r0 * K, hA + r0 * K * cb, dA + r0 * K * cb, (s - r0) * K)))
            return cuda_fail(e, "H2D A");
        cudaEventRecord(g_scratch.evA[i], sh);
        cudaStreamWaitEvent(st, g_scratch.evA[i], 0);
        cudaStreamWaitEvent(st, g_scratch.evAr[i], 0);
        launch_narrow(acur, dA + s * K * cb, (r1 - s) * K, cb, mask, st);
        acur += seg((r1 - s) * K);
        if (prof) cudaEventRecord(tev[2 * i + 1], st);
        // B's digit image is packed by the first panel and reused while the
        // panel plans share the workspace layout
        QuireGemmPlan pp;
        quire_gemm_plan(nbits, es, r1 - r0, N, K, 0, &pp);
        const bool same = i > 0 && pp.off_b == p0.off_b && pp.b_img_bytes == p0.b_img_bytes &&
                          pp.off_col_nar == p0.off_col_nar && pp.off_flags == p0.off_flags &&
                          pp.D == p0.D && pp.kbt == p0.kbt && pp.ntiles == p0.ntiles;
        if (i == 0) p0 = pp;
        int rc = quire_gemm_launch(nbits, es, dA + r0 * K * cb, dB, dC + r0 * N * cb, r1 - r0, N, K, K, N, N,
                                   ws, ws_bytes, 0, st, nullptr, /*pack_b=*/!same);
        if (rc) return rc == 4 ? cuda_fail(cudaGetLastError(), "matmul launch") : fail(rc, "matmul");
        // raw output share of this panel: widened on the GPU, DMA'd into C
        const int64_t so = split_out(r0, r1);
        launch_widen(dC + so * N * cb, ocur, (r1 - so) * N, cb, st);
        cudaEventRecord(g_scratch.evG[i], st);
        if (r1 > so) {
            cudaStreamWaitEvent(sdr, g_scratch.evG[i], 0);
            if ((e = cudaMemcpyAsync(C + so * N, ocur, size_t((r1 - so) * N) * 8, cudaMemcpyDeviceToHost, sdr)))
                return cuda_fail(e, "D2H C raw");
        }
        ocur += seg((r1 - so) * N);
        if (prof) cudaEventRecord(tev[2 * i + 2], st);
    }
    const auto t1 = now();
    // 3. host-widened share of each panel: chunked packed D2H, widen chunk j
    //    while chunk j+1 is in flight
    for (int i = 0; i < P; ++i) {
        const int64_t r0 = i * rows, r1 = std::min(M, r0 + rows);
        if (r0 >= r1) break;
        cudaStreamWaitEvent(sd, g_scratch.evG[i], 0);
        const int64_t off = r0 * N, n = (split_out(r0, r1) - r0) * N;
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
    const auto t2 = now();
    for (cudaStream_t s2 : {sh, shr, st, sd, sdr})
        if ((e = cudaStreamSynchronize(s2))) return cuda_fail(e, "matmul_host sync");
    if (prof) {
        const auto t3 = now();
        fprintf(stderr,
                "[pnn_matmul_host] posit(%d,%d) P=%d f_in=%.2f f_out=%.2f threads=%d: narrow+issue %.2f ms, "
                "widen %.2f ms, final sync %.2f ms\n",
                nbits, es, P, f_in, f_out, pool.workers(),
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(t2 - t1).count(),
                std::chrono::duration<double, std::milli>(t3 - t2).count());
        // device timeline: panel i's GEMM starts after its inputs (tev[2i+1]), ends at tev[2i+2]
        std::string tl;
        for (int i = 0; i < P; ++i) {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, tev[0], tev[2 * i + 1]);
            cudaEventElapsedTime(&b, tev[0], tev[2 * i + 2]);
            char buf[64];
            snprintf(buf, sizeof buf, " [%.2f..%.2f]", a, b);
            tl += buf;
        }
        fprintf(stderr, "[pnn_matmul_host]   gemm panels (ms from issue start):%s\n", tl.c_str());
        for (int i = 0; i <= 2 * P; ++i) cudaEventDestroy(tev[i]);
    }
    return PNN_OK;
}

// Internal test hook (not part of include/pnn_b200.h): the epilogue's two
// 64-bit quire-word roundings (integer leading-one search vs the FP64
// converter) on the same words, for tests/test_epilogue_gpu.py.
__global__ void round64_check_kernel(PositFmt f, const uint64_t* q, int64_t n, uint32_t* a, uint32_t* b) {
    __shared__ uint4 s_lut[kPackLutEntries];
    build_pack_lut(f, s_lut, threadIdx.x, blockDim.x);
    __syncthreads();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        a[i] = q_to_posit_lut(f, q[i], s_lut);
        b[i] = q_to_posit_lut_f64(f, q[i], s_lut);
    }
}

int pnn_internal_round64_check(int nbits, int es, const uint64_t* q, int64_t n, uint32_t* a, uint32_t* b,
                               void* stream) {
    if (int rc = check_fmt(nbits, es)) return rc;
    const PositFmt f = make_fmt(nbits, es);
    if (n <= 0) return PNN_OK;  // (W > 64: the word is the exact value as int64, no wrap)
    round64_check_kernel<<<148 * 4, 256, 0, as_stream(stream)>>>(f, q, n, a, b);
    return cudaGetLastError() == cudaSuccess ? PNN_OK : cuda_fail(cudaGetLastError(), "round64_check");
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
