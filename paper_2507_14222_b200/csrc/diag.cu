// diag.cu — integer-pipe peak micro-benchmark (the roofline denominator for the
// AND/POPC kernels; SURVEY.md §8(d) "Measure LOP3/POPC peaks with a micro-kernel").
#include "ig_internal.cuh"

namespace igb {
namespace {

__device__ __forceinline__ uint32_t lop3_andnot_or(uint32_t acc, uint32_t p, uint32_t x) {
    uint32_t r;
    // r = acc | (p & ~x): the per-half subset test of subset.cu, one LOP3.
    asm volatile("lop3.b32 %0, %1, %2, %3, 0xF2;" : "=r"(r) : "r"(p), "r"(x), "r"(acc));
    return r;
}

// 16 independent LOP3 chains per thread; every op depends on the previous one
// of its chain so nothing is hoisted.  ops = threads * iters * 16.
__global__ void __launch_bounds__(256) lop3_peak(uint32_t* out, int iters, uint32_t seed) {
    uint32_t a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u;
    const uint32_t p = seed ^ blockIdx.x, x = ~seed;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = lop3_andnot_or(a[i], a[(i + 1) & 15], x ^ p);
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) r ^= a[i];
    if (r == 0x12345678u) out[0] = r;
}

__global__ void __launch_bounds__(256) popc_peak(uint32_t* out, int iters, uint32_t seed) {
    uint32_t a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + 1) + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __popc(a[i]) + a[(i + 1) & 7];
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r ^= a[i];
    if (r == 0x12345678u) out[0] = r;
}

}  // namespace

// Returns LOP3.32 / s and POPC.32 / s sustained on the whole GPU.
void measure_int_peaks(Ctx& ctx, double* lop3_per_s, double* popc_per_s) {
    DevBuf o(16, ctx.stream);
    const int blocks = ctx.sm_count * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    IGB_CUDA(cudaEventCreate(&e0));
    IGB_CUDA(cudaEventCreate(&e1));
    float best = 1e30f, bestp = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
        IGB_CUDA(cudaEventRecord(e0, ctx.stream));
        IGB_LAUNCH(ctx, lop3_peak, blocks, threads, 0, o.as<uint32_t>(), iters, 12345u + rep);
        IGB_CUDA(cudaEventRecord(e1, ctx.stream));
        IGB_CUDA(cudaEventSynchronize(e1));
        float ms;
        IGB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (rep) best = std::min(best, ms);
        IGB_CUDA(cudaEventRecord(e0, ctx.stream));
        IGB_LAUNCH(ctx, popc_peak, blocks, threads, 0, o.as<uint32_t>(), iters, 777u + rep);
        IGB_CUDA(cudaEventRecord(e1, ctx.stream));
        IGB_CUDA(cudaEventSynchronize(e1));
        IGB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (rep) bestp = std::min(bestp, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double threads_total = (double)blocks * threads;
    *lop3_per_s = threads_total * iters * 16 / (best * 1e-3);
    *popc_per_s = threads_total * iters * 8 / (bestp * 1e-3);
}

}  // namespace igb
