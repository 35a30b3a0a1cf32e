// ig_internal.cuh — shared internals of libig_b200.so (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <future>
#include <mutex>
#include <thread>
#include <cstring>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <string>
#include <utility>
#include <vector>

#include "ig_b200.h"
#include "ig_error.hpp"

namespace igb {

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        int st = (e == cudaErrorMemoryAllocation) ? IG_E_OOM : IG_E_CUDA;
        fail(st, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" + std::to_string(line) + ")");
    }
}
#define IGB_CUDA(x) ::igb::cuda_check((x), #x, __FILE__, __LINE__)

struct Ctx;

// Stream-ordered device buffer (cudaMallocAsync on the context stream; the
// pool keeps freed blocks cached so repeated fits do not hit the driver).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(size_t n, cudaStream_t st) { alloc(n, st); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            bytes = o.bytes;
            s = o.s;
            persistent = o.persistent;
            o.p = nullptr;
            o.bytes = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t n, cudaStream_t st) {
        release();
        s = st;
        bytes = n;
        if (n) IGB_CUDA(cudaMallocAsync(&p, n, st));
    }
    void release() noexcept {
        if (p) {
            if (persistent)
                cudaFree(p);  // long-lived result objects may outlive the stream they were made on
            else
                cudaFreeAsync(p, s);
        }
        p = nullptr;
        bytes = 0;
    }
    // Mark as owned by a long-lived ABI object (model, candidate set, encoding).
    void persist() { persistent = true; }
    bool persistent = false;
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Matrix of packed rows resident on the device.
struct DevRows {
    DevBuf buf;
    size_t n = 0;
    size_t k = 0;
    uint32_t L = 0;
    int64_t* data() const { return buf.as<int64_t>(); }
};

// Hot kernels the bench reports a roofline for (ig_ctx_diag_kernel).
enum DiagKind { kDiagEnum = 0, kDiagSupport = 1, kDiagCover = 2, kDiagMatch = 3, kDiagKinds = 4 };
struct DiagStat {
    double ms = 0;          // CUDA-event time of the launches
    uint64_t work = 0;      // useful 64-bit word-ANDs they performed (counted exactly)
    uint64_t launches = 0;
};

// Progress of a long enumeration (ig_enumerate_candidates' ig_progress_fn,
// mine.hpp:31-33): the kernel publishes pairs done / candidates found into
// page-locked mapped memory after each tile; the calling thread polls it while
// the stream runs and calls fn.
struct ProgressHook {
    void (*fn)(uint64_t, uint64_t, uint64_t, void*) = nullptr;
    void* user = nullptr;
    unsigned long long* host = nullptr;  // [0] pairs done, [1] candidates found (mapped)
    unsigned long long* dev = nullptr;   // device alias of host
    unsigned long long* ctr = nullptr;   // device counters the kernel adds to
    uint64_t pairs_total = 0;
    uint64_t seen[2] = {0, 0};
};

// A persistent host thread running submitted tasks in order (the second class
// of a fit, the test index build): thread creation on every step cost tens of
// microseconds of idle GPU.
class Worker {
public:
    explicit Worker(int device) : th_([this, device] {
        cudaSetDevice(device);
        for (;;) {
            std::function<void()> task;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [this] { return stop_ || !q_.empty(); });
                if (q_.empty()) return;  // stopping
                task = std::move(q_.front());
                q_.pop_front();
            }
            task();
        }
    }) {}
    Worker(const Worker&) = delete;
    ~Worker() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        th_.join();
    }
    // run fn on the worker; the future completes when it returned (fn must not throw)
    std::future<void> submit(std::function<void()> fn) {
        auto task = std::make_shared<std::packaged_task<void()>>(std::move(fn));
        std::future<void> f = task->get_future();
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.emplace_back([task] { (*task)(); });
        }
        cv_.notify_one();
        return f;
    }

private:
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> q_;
    bool stop_ = false;
    std::thread th_;  // last: started once the queue exists
};

// A background job: on a persistent worker when there is one (no thread
// start per call), else on its own thread.
struct BgTask {
    std::thread th;
    std::future<void> fut;
    void start(Worker* w, std::function<void()> fn) {
        if (w)
            fut = w->submit(std::move(fn));
        else
            th = std::thread(std::move(fn));
    }
    void join() {
        if (th.joinable()) th.join();
        if (fut.valid()) fut.wait();
    }
};

struct Ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t aux = nullptr;  // second class's stream (for_both_classes)
    cudaStream_t copy = nullptr; // host->device prefetches (ig_columns_prefetch)
    cudaStream_t index = nullptr;  // background test-row encode + postings (ig_encode_rows)
    uint64_t launches = 0;
    int sm_count = 148;
    size_t smem_optin = 0;
    // diagnostics (bench roofline only; off on the timed path): per hot kernel,
    // CUDA-event time of its launches and their exact useful work
    bool diag = false;
    DiagStat diag_k[kDiagKinds];
    ProgressHook* progress = nullptr;  // set by ig_enumerate_candidates for one call
    Worker* worker = nullptr;          // owned by the ABI context; copies share it (may be null)
    // background jobs of an encode (owned by the ABI context, may be null): the
    // test rows' index, the training vocabulary's host text
    Worker* index_worker = nullptr;
    Worker* vocab_worker = nullptr;
    void diag_merge(const Ctx& o) {
        for (int i = 0; i < kDiagKinds; ++i) {
            diag_k[i].ms += o.diag_k[i].ms;
            diag_k[i].work += o.diag_k[i].work;
            diag_k[i].launches += o.diag_k[i].launches;
        }
    }
};

// Times one hot-kernel launch on the context stream with CUDA events when
// diagnostics are on (the stream is synchronised at end(): diagnostics only).
struct DiagSpan {
    Ctx& ctx;
    int kind;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    DiagSpan(Ctx& c, int k) : ctx(c), kind(k) {
        if (!ctx.diag) return;
        IGB_CUDA(cudaEventCreate(&e0));
        IGB_CUDA(cudaEventCreate(&e1));
        IGB_CUDA(cudaEventRecord(e0, ctx.stream));
    }
    DiagSpan(const DiagSpan&) = delete;
    // record the end of the timed launch (before any counting launch)
    void stop() {
        if (e1) IGB_CUDA(cudaEventRecord(e1, ctx.stream));
    }
    void end(uint64_t work) {
        if (!e0) return;
        IGB_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        IGB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        ctx.diag_k[kind].ms += ms;
        ctx.diag_k[kind].work += work;
        ctx.diag_k[kind].launches += 1;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        e0 = e1 = nullptr;
    }
    ~DiagSpan() {
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};

// Device->host readback of a small result (counts, flags, totals) and a wait
// for it, through a per-thread page-locked bounce buffer: a pageable
// destination is staged by the driver and can queue behind a large in-flight
// host->device copy (e.g. a columns prefetch) on the copy engines.
// page-locked bounce buffer from the library's host pool (ig_host_alloc): no
// per-thread cudaMallocHost / cudaFreeHost in the short-lived encode jobs
inline void read_back(const Ctx& ctx, void* host_dst, const void* d_src, size_t bytes) {
    if (!bytes) {
        IGB_CUDA(cudaStreamSynchronize(ctx.stream));
        return;
    }
    void* buf = nullptr;
    if (ig_host_alloc(std::max<size_t>(bytes, 4096), &buf) != IG_OK) fail(IG_E_OOM, "page-locked read-back buffer");
    struct Back {
        void* p;
        ~Back() { ig_host_free(p); }
    } back{buf};
    IGB_CUDA(cudaMemcpyAsync(buf, d_src, bytes, cudaMemcpyDeviceToHost, ctx.stream));
    IGB_CUDA(cudaStreamSynchronize(ctx.stream));
    std::memcpy(host_dst, buf, bytes);
}

// Device -> host result copy: straight into page-locked destinations (the
// library's host pool), through the bounce buffer otherwise.
inline void copy_to_host(const Ctx& ctx, void* host_dst, const void* d_src, size_t bytes) {
    cudaPointerAttributes a{};
    if (bytes && cudaPointerGetAttributes(&a, host_dst) == cudaSuccess && a.type == cudaMemoryTypeHost) {
        IGB_CUDA(cudaMemcpyAsync(host_dst, d_src, bytes, cudaMemcpyDeviceToHost, ctx.stream));
        IGB_CUDA(cudaStreamSynchronize(ctx.stream));
        return;
    }
    cudaGetLastError();  // older runtimes report (and record) an error for unregistered pointers
    read_back(ctx, host_dst, d_src, bytes);
}

// IG_TRACE=1: per-operation wall times on stderr (synchronises the stream at
// every mark; diagnostics only).
struct Trace {
    const Ctx& ctx;
    const char* what;
    int cls;
    bool on;
    double t0;
    static double now() {
        timespec ts;
        clock_gettime(CLOCK_MONOTONIC, &ts);
        return ts.tv_sec + ts.tv_nsec * 1e-9;
    }
    Trace(const Ctx& c, const char* w, int cl) : ctx(c), what(w), cls(cl), on(getenv("IG_TRACE") != nullptr), t0(0) {
        if (on) {
            cudaStreamSynchronize(ctx.stream);
            t0 = now();
        }
    }
    void mark(const char* step) {
        if (!on) return;
        cudaStreamSynchronize(ctx.stream);
        const double t = now();
        fprintf(stderr, "[ig trace] %s class %d %s %.3f ms\n", what, cls, step, (t - t0) * 1e3);
        t0 = t;
    }
};

inline size_t words_for(uint32_t L) { return (static_cast<size_t>(L) + 63) / 64; }

// Raise a kernel's dynamic shared-memory limit once per device and size (the
// attribute call costs a few microseconds of host time on every launch site).
#define IGB_SMEM_ATTR(ctx, kernel, bytes)                                                           \
    do {                                                                                            \
        static std::atomic<int> igb_smem_set_[64];                                                  \
        const int igb_dev_ = (ctx).device & 63, igb_b_ = (int)(bytes);                              \
        if (igb_smem_set_[igb_dev_].load(std::memory_order_relaxed) < igb_b_) {                     \
            IGB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, igb_b_)); \
            igb_smem_set_[igb_dev_].store(igb_b_, std::memory_order_relaxed);                       \
        }                                                                                           \
    } while (0)

// Every kernel launch goes through this so the context can report how many of
// its own kernels ran (bench `gpu_launches`) and catch launch errors at once.
#define IGB_LAUNCH(ctx, kernel, grid, block, smem, ...)                                   \
    do {                                                                                  \
        kernel<<<(grid), (block), (smem), (ctx).stream>>>(__VA_ARGS__);                   \
        IGB_CUDA(cudaGetLastError());                                                     \
        ++(ctx).launches;                                                                 \
    } while (0)

// ------------------------------------------------------------------ device primitives
__device__ __forceinline__ uint64_t mix64(uint64_t h) {
    // murmur3 fmix64
    h ^= h >> 33;
    h *= 0xff51afd7ed558ccdull;
    h ^= h >> 33;
    h *= 0xc4ceb9fe1a85ec53ull;
    h ^= h >> 33;
    return h;
}

// Fingerprint of a K-word candidate: NH over per-word keys (the UMAC inner
// hash), sum_w (lo_w + klo_w) * (hi_w + khi_w) mod 2^64 with 32-bit halves —
// one IMAD.WIDE per word — finalised with fmix64.  For rows of equal length
// and uniform keys two distinct rows collide with probability <= 2^-32; a new
// key set per collision level separates any pair that collided.  A fingerprint
// is only a bucket hint: every equality is confirmed on the full words.
struct Fp {
    uint64_t acc = 0;
    __device__ __forceinline__ void add(uint64_t w, uint64_t key) {
        acc += (uint64_t)((uint32_t)w + (uint32_t)key) * (uint64_t)((uint32_t)(w >> 32) + (uint32_t)(key >> 32));
    }
    __device__ __forceinline__ uint64_t final(uint32_t k) const {
        uint64_t f = mix64(acc + k);
        return f ? f : 1ull;  // 0 marks an empty hash slot
    }
};

// ------------------------------------------------------------------ host helpers
// (declared here, defined in the .cu files)
// Permutation putting rows in canonical words::less order (bitpack.hpp:59-68).
void sort_rows_canonical(Ctx& ctx, const int64_t* d_words, size_t n, size_t k, uint32_t* d_perm);
// Reference implementation: K stable 64-bit LSD radix passes (fallback).
void sort_rows_canonical_lsd(Ctx& ctx, const int64_t* d_words, size_t n, size_t k, uint32_t* d_perm);
// Distinct rows of d_rows in canonical order -> out (m x k); returns m.
// d_perm: the rows' canonical permutation when already known (else computed).
// o_perm (optional): receives that permutation.
size_t distinct_rows(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, DevBuf& out, const uint32_t* d_perm = nullptr,
                     DevBuf* o_perm = nullptr);
void gather_rows(Ctx& ctx, const int64_t* d_src, const uint32_t* d_perm, size_t n, size_t k, int64_t* d_dst);

}  // namespace igb
