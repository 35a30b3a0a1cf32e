// subset.cu — the (b & x) == b family: coverage (kernel 4), support (kernel 5)
// and the test-time matcher (kernel 6).
//
// Reference semantics:
//   words::is_subset            proj/include/ig/bitpack.hpp:37-43
//   covered_by_any / coverage   proj/src/kernels.cpp:59-65, 89-103, 139-154
//   score_one_test / fused      proj/src/kernels.cpp:40-46, 67-77, 105-118, 156-178
//   count_support               proj/include/ig/mine.hpp:42-44
//
// Layout: each thread owns one row in registers (a test row for the matcher, a
// candidate for support/coverage); the CTA streams the other operand through
// shared memory in chunks and every lane reads the same shared word
// (broadcast, conflict-free).  The per-word test is `own & ~streamed` (or the
// reverse), one LOP3 per 32-bit half, and the warp leaves a row as soon as no
// lane can still match (__any_sync == the warp ballot of north_star (4)).
#include <cub/cub.cuh>

#include "ig_internal.cuh"
#include "posting.cuh"
#include "subset.cuh"

namespace igb {

namespace {

constexpr int kThreads = 128;
constexpr int kChunk = 128;  // streamed rows per shared-memory chunk
constexpr unsigned kFull = 0xffffffffu;

enum Mode : int { kMatch = 0, kSupport = 1, kCover = 2 };

// MODE kMatch   : own = test rows,  stream = patterns (+scores); out = evidence
// MODE kSupport : own = candidates, stream = class rows;         out = support
// MODE kCover   : own = candidates, stream = opponent rows;      out = covered mask
// ORDERED (match only): one slice, checked signed add in pattern order —
// exactly the reference's checked_add sequence (kernels.cpp:67-77).
template <int KMAX, int MODE, bool ORDERED>
__global__ void __launch_bounds__(kThreads)
subset_scan(const int64_t* __restrict__ own, size_t n_own, const int64_t* __restrict__ stream,
            size_t n_stream, int k, const int64_t* __restrict__ scores, size_t slice_rows,
            int64_t* __restrict__ out_i64, uint64_t* __restrict__ partial, uint8_t* __restrict__ out_u8,
            int* __restrict__ overflow) {
    extern __shared__ int64_t smem[];
    int64_t* srow = smem;                          // kChunk * k words
    int64_t* sval = smem + (size_t)kChunk * k;     // kChunk scores (match)

    const size_t t = (size_t)blockIdx.x * kThreads + threadIdx.x;
    const bool active = t < n_own;
    uint64_t reg[KMAX];
#pragma unroll
    for (int w = 0; w < KMAX; ++w) reg[w] = (active && w < k) ? (uint64_t)own[t * k + w] : 0ull;

    const size_t s_begin = (size_t)blockIdx.y * slice_rows;
    const size_t s_end = min(n_stream, s_begin + slice_rows);

    int64_t acc = 0;         // ordered match
    uint64_t uacc = 0;       // unordered match (non-negative scores)
    bool ovf = false;
    int64_t count = 0;       // support
    bool covered = false;    // cover

    for (size_t base = s_begin; base < s_end; base += kChunk) {
        const int ch = (int)min((size_t)kChunk, s_end - base);
        __syncthreads();
        for (int i = threadIdx.x; i < ch * k; i += kThreads) srow[i] = stream[base * k + i];
        if (MODE == kMatch)
            for (int i = threadIdx.x; i < ch; i += kThreads) sval[i] = scores[base + i];
        __syncthreads();
        if (MODE == kCover) {
            if (__syncthreads_and(covered || !active)) break;
        }
        for (int r = 0; r < ch; ++r) {
            const int64_t* q = srow + (size_t)r * k;
            bool ok = active && !(MODE == kCover && covered);
#pragma unroll
            for (int w = 0; w < KMAX; ++w) {
                if (w < k) {
                    const uint64_t sw = (uint64_t)q[w];
                    // match: pattern (streamed) ⊆ test (own);  else own ⊆ streamed
                    const uint64_t bad = (MODE == kMatch) ? (sw & ~reg[w]) : (reg[w] & ~sw);
                    ok = ok && (bad == 0ull);
                    if (!__any_sync(kFull, ok)) break;
                }
            }
            if (ok) {
                if (MODE == kMatch) {
                    const int64_t s = sval[r];
                    if (ORDERED) {
                        const int64_t nacc = (int64_t)((uint64_t)acc + (uint64_t)s);
                        if (((acc ^ nacc) & (s ^ nacc)) < 0) ovf = true;  // signed wrap
                        acc = nacc;
                    } else {
                        uacc += (uint64_t)s;  // s >= 0 checked by the caller
                        if (uacc > (uint64_t)INT64_MAX) ovf = true;
                    }
                } else if (MODE == kSupport) {
                    ++count;
                } else {
                    covered = true;
                }
            }
        }
    }
    if (!active) return;
    if (MODE == kMatch) {
        if (ovf) atomicOr(overflow, 1);
        if (ORDERED)
            out_i64[t] = acc;
        else
            partial[(size_t)blockIdx.y * n_own + t] = ovf ? (uint64_t)INT64_MAX + 1 : uacc;
    } else if (MODE == kSupport) {
        partial[(size_t)blockIdx.y * n_own + t] = (uint64_t)count;
    } else {
        if (covered) out_u8[t] = 1;
    }
}

// Generic-K fallback (K > 64 words, e.g. CICIDS-shape): own row read from
// global memory (L1-resident) instead of registers.
template <int MODE>
__global__ void __launch_bounds__(kThreads)
subset_scan_wide(const int64_t* __restrict__ own, size_t n_own, const int64_t* __restrict__ stream,
                 size_t n_stream, int k, const int64_t* __restrict__ scores, size_t slice_rows,
                 int64_t* __restrict__ out_i64, uint64_t* __restrict__ partial,
                 uint8_t* __restrict__ out_u8, int* __restrict__ overflow, int ordered) {
    const size_t t = (size_t)blockIdx.x * kThreads + threadIdx.x;
    if (t >= n_own) return;
    const int64_t* me = own + t * k;
    const size_t s_begin = (size_t)blockIdx.y * slice_rows;
    const size_t s_end = min(n_stream, s_begin + slice_rows);
    int64_t acc = 0;
    uint64_t uacc = 0, count = 0;
    bool ovf = false;
    for (size_t r = s_begin; r < s_end; ++r) {
        const int64_t* q = stream + r * k;
        bool ok = true;
        for (int w = 0; w < k && ok; ++w) {
            const uint64_t a = (uint64_t)__ldg(me + w), b = (uint64_t)__ldg(q + w);
            ok = (MODE == kMatch) ? ((b & ~a) == 0) : ((a & ~b) == 0);
        }
        if (!ok) continue;
        if (MODE == kMatch) {
            const int64_t s = scores[r];
            if (ordered) {
                const int64_t nacc = (int64_t)((uint64_t)acc + (uint64_t)s);
                if (((acc ^ nacc) & (s ^ nacc)) < 0) ovf = true;
                acc = nacc;
            } else {
                uacc += (uint64_t)s;
                if (uacc > (uint64_t)INT64_MAX) ovf = true;
            }
        } else if (MODE == kSupport) {
            ++count;
        } else {
            out_u8[t] = 1;
            return;
        }
    }
    if (MODE == kMatch) {
        if (ovf) atomicOr(overflow, 1);
        if (ordered)
            out_i64[t] = acc;
        else
            partial[(size_t)blockIdx.y * n_own + t] = ovf ? (uint64_t)INT64_MAX + 1 : uacc;
    } else if (MODE == kSupport) {
        partial[(size_t)blockIdx.y * n_own + t] = count;
    }
}

// Sum `slices` partial u64 rows per own row; > INT64_MAX means overflow.
__global__ void reduce_partials(const uint64_t* __restrict__ partial, size_t n, int slices,
                                int64_t* __restrict__ out, int* __restrict__ overflow) {
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint64_t acc = 0;
    bool ovf = false;
    for (int s = 0; s < slices; ++s) {
        const uint64_t v = partial[(size_t)s * n + t];
        if (v > (uint64_t)INT64_MAX) ovf = true;
        acc += v;
        if (acc > (uint64_t)INT64_MAX) ovf = true;
    }
    if (ovf) atomicOr(overflow, 1);
    out[t] = (int64_t)acc;
}

__global__ void any_negative(const int64_t* __restrict__ s, size_t n, int* __restrict__ flag) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        if (s[i] < 0) {
            atomicOr(flag, 1);
            return;
        }
}

template <int MODE, bool ORDERED>
void launch_scan(Ctx& ctx, const int64_t* own, size_t n_own, const int64_t* stream, size_t n_stream,
                 size_t k, const int64_t* scores, int slices, size_t slice_rows, int64_t* out_i64,
                 uint64_t* partial, uint8_t* out_u8, int* overflow) {
    dim3 grid((unsigned)((n_own + kThreads - 1) / kThreads), (unsigned)slices);
    const int ki = (int)k;
    if (k <= 64) {
        const size_t smem = (size_t)kChunk * k * 8 + (MODE == kMatch ? kChunk * 8 : 0);
#define IGB_SCAN_CASE(KM)                                                                              \
    if (k <= KM) {                                                                                     \
        auto kern = subset_scan<KM, MODE, ORDERED>;                                                    \
        if (smem > 48 * 1024) IGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        IGB_LAUNCH(ctx, kern, grid, kThreads, smem, own, n_own, stream, n_stream, ki, scores, slice_rows,  \
                   out_i64, partial, out_u8, overflow);                                                \
        return;                                                                                        \
    }
        IGB_SCAN_CASE(2)
        IGB_SCAN_CASE(4)
        IGB_SCAN_CASE(8)
        IGB_SCAN_CASE(16)
        IGB_SCAN_CASE(32)
        IGB_SCAN_CASE(64)
#undef IGB_SCAN_CASE
    }
    IGB_LAUNCH(ctx, subset_scan_wide<MODE>, grid, kThreads, 0, own, n_own, stream, n_stream, ki, scores,
               slice_rows, out_i64, partial, out_u8, overflow, ORDERED ? 1 : 0);
}

// Split the streamed operand into slices so the grid covers the GPU even when
// the owned side is small.
int choose_slices(const Ctx& ctx, size_t n_own, size_t n_stream, size_t* slice_rows) {
    const size_t bx = (n_own + kThreads - 1) / kThreads;
    const size_t want = (size_t)ctx.sm_count * 8;
    size_t slices = bx >= want ? 1 : (want + bx - 1) / bx;
    const size_t max_slices = (n_stream + 2047) / 2048;  // keep >= 2048 rows per slice
    if (slices > max_slices) slices = max_slices;
    if (slices < 1) slices = 1;
    if (slices > 65535) slices = 65535;
    size_t rows = (n_stream + slices - 1) / slices;
    rows = (rows + kChunk - 1) / kChunk * kChunk;
    if (rows == 0) rows = kChunk;
    slices = (n_stream + rows - 1) / rows;
    if (slices < 1) slices = 1;
    *slice_rows = rows;
    return (int)slices;
}

}  // namespace

void coverage_any_dev(Ctx& ctx, const int64_t* d_pat, size_t np, const int64_t* d_opp, size_t no,
                      size_t k, uint8_t* d_mask) {
    IGB_CUDA(cudaMemsetAsync(d_mask, 0, np, ctx.stream));
    if (np == 0 || no == 0) return;
    if (postings_supported((uint32_t)(64 * k), no)) {
        Postings P;
        build_postings(ctx, d_opp, no, k, (uint32_t)(64 * k), P, true, true);
        posting_cover(ctx, d_pat, np, k, P, d_mask);
        return;
    }
    // The opponent side is never sliced: each candidate stops at its first cover.
    launch_scan<kCover, false>(ctx, d_pat, np, d_opp, no, k, nullptr, 1, no, nullptr, nullptr, d_mask,
                               nullptr);
}

void count_support_dev(Ctx& ctx, const int64_t* d_pat, size_t np, const int64_t* d_rows, size_t n,
                       size_t k, int64_t* d_support) {
    if (np == 0) return;
    if (n == 0) {
        IGB_CUDA(cudaMemsetAsync(d_support, 0, np * 8, ctx.stream));
        return;
    }
    if (postings_supported((uint32_t)(64 * k), n)) {
        Postings P;
        build_postings(ctx, d_rows, n, k, (uint32_t)(64 * k), P);
        posting_support(ctx, d_pat, np, k, P, d_support);
        return;
    }
    size_t slice_rows;
    const int slices = choose_slices(ctx, np, n, &slice_rows);
    DevBuf partial((size_t)slices * np * 8, ctx.stream);
    DevBuf flag(sizeof(int), ctx.stream);
    IGB_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx.stream));
    launch_scan<kSupport, false>(ctx, d_pat, np, d_rows, n, k, nullptr, slices, slice_rows, nullptr,
                                 partial.as<uint64_t>(), nullptr, nullptr);
    IGB_LAUNCH(ctx, reduce_partials, (unsigned)((np + 255) / 256), 256, 0, partial.as<uint64_t>(), np,
               slices, d_support, flag.as<int>());
}

int fused_score_dev(Ctx& ctx, const int64_t* d_pat, size_t np, const int64_t* d_scores,
                    const int64_t* d_tests, size_t nt, size_t k, int64_t* d_out) {
    if (nt == 0) return IG_OK;
    if (np == 0) {
        IGB_CUDA(cudaMemsetAsync(d_out, 0, nt * 8, ctx.stream));
        return IG_OK;
    }
    DevBuf flags(2 * sizeof(int), ctx.stream);
    int* d_flags = flags.as<int>();  // [0] overflow, [1] negative score present
    IGB_CUDA(cudaMemsetAsync(d_flags, 0, 2 * sizeof(int), ctx.stream));
    IGB_LAUNCH(ctx, any_negative, 256, 256, 0, d_scores, np, d_flags + 1);
    int h_flags[2];
    read_back(ctx, h_flags, d_flags, sizeof(h_flags));
    if (h_flags[1]) {
        // Mixed-sign scores: overflow depends on the order of partial sums, so
        // every test row walks the patterns in index order (kernels.cpp:70-75).
        launch_scan<kMatch, true>(ctx, d_tests, nt, d_pat, np, k, d_scores, 1, np, d_out, nullptr, nullptr,
                                  d_flags);
    } else if (postings_supported((uint32_t)(64 * k), nt)) {
        Postings P;
        build_postings(ctx, d_tests, nt, k, (uint32_t)(64 * k), P, true, true);
        int64_t total = 0;
        const bool fits = total_score_dev(ctx, d_scores, np, &total) == IG_OK;  // scores >= 0 here
        posting_match(ctx, d_pat, np, k, d_scores, P, d_out, d_flags, fits);
    } else {
        size_t slice_rows;
        const int slices = choose_slices(ctx, nt, np, &slice_rows);
        DevBuf partial((size_t)slices * nt * 8, ctx.stream);
        launch_scan<kMatch, false>(ctx, d_tests, nt, d_pat, np, k, d_scores, slices, slice_rows, nullptr,
                                   partial.as<uint64_t>(), nullptr, d_flags);
        IGB_LAUNCH(ctx, reduce_partials, (unsigned)((nt + 255) / 256), 256, 0, partial.as<uint64_t>(), nt,
                   slices, d_out, d_flags);
    }
    read_back(ctx, h_flags, d_flags, sizeof(int));
    return h_flags[0] ? IG_E_OVERFLOW : IG_OK;
}

}  // namespace igb
