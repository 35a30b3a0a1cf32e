// posting.cu — the vertical (posting-bitmap) form of the subset test, used for
// support (kernel 5), coverage (kernel 4) and the matcher (kernel 6).
//
// Same semantics as subset.cu (words::is_subset, bitpack.hpp:37-43), other
// data layout.  For a row set R of n rows, post[t] is the n-bit set of rows
// that contain bit t (all 64·K bit positions × W = ceil(n/64) words;
// L2-resident at NSL shape).  Then
//     {r ∈ R : b ⊆ r} = AND_{t ∈ b} post[t]
// so a pattern costs |b| word-ANDs per 64 rows instead of K word tests per row
// (|b| ≈ 17 tokens vs 64·K = 896 bits at NSL shape).  Rows are put in
// canonical order first so rows sharing tokens share posting words.  Each
// pattern's tokens are listed rarest first (document frequency over R); a warp
// walks the non-zero words of the rarest token (CSR list), 32 words per step,
// and ANDs the next tokens until no lane has a surviving row.  Exact and
// independent of every order involved:
//   support  = Σ popcount(...)
//   covered  = any word non-zero                             (kernels.cpp:59-65)
//   evidence: A[row] += s_p for each surviving bit, u64 atomics with overflow
//             detection; used only when all scores are ≥ 0, where "some prefix
//             overflows" ⟺ "the total exceeds INT64_MAX" (kernels.cpp:40-46).
#include <cub/cub.cuh>

#include <algorithm>

#include "ig_internal.cuh"
#include "posting.cuh"

namespace igb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxSorted = 64;  // token lists longer than this keep bit order past the rarest

unsigned grid_for(const Ctx& ctx, size_t work, int threads) {
    size_t g = (work + threads - 1) / threads;
    const size_t cap = (size_t)ctx.sm_count * 32;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

// Warp per (64-row block w, source word sw): 64x64 bit transpose with ballots.
// Rows are read through `perm` (canonical order) when given.
__global__ void transpose_rows(const int64_t* __restrict__ rows, const uint32_t* __restrict__ perm, size_t n, int k,
                               size_t W, unsigned long long* __restrict__ dense) {
    const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const size_t total = W * (size_t)k;
    for (size_t q = warp; q < total; q += ((size_t)gridDim.x * blockDim.x) >> 5) {
        const size_t w = q / k;
        const int sw = (int)(q % k);
        const size_t r0 = w * 64 + lane, r1 = r0 + 32;
        const size_t s0 = r0 < n ? (perm ? perm[r0] : r0) : 0, s1 = r1 < n ? (perm ? perm[r1] : r1) : 0;
        const uint64_t x0 = r0 < n ? (uint64_t)rows[s0 * k + sw] : 0ull;
        const uint64_t x1 = r1 < n ? (uint64_t)rows[s1 * k + sw] : 0ull;
        uint64_t mine_lo = 0, mine_hi = 0;  // lane b: bit sw*64+b (lo) and sw*64+32+b (hi)
#pragma unroll 8
        for (int b = 0; b < 64; ++b) {
            const uint32_t lo = __ballot_sync(kFull, (x0 >> b) & 1ull);
            const uint32_t hi = __ballot_sync(kFull, (x1 >> b) & 1ull);
            const uint64_t v = (uint64_t)lo | ((uint64_t)hi << 32);
            if ((b & 31) == lane) {
                if (b < 32)
                    mine_lo = v;
                else
                    mine_hi = v;
            }
        }
        const size_t t0 = (size_t)sw * 64 + lane, t1 = t0 + 32;
        dense[t0 * W + w] = mine_lo;
        dense[t1 * W + w] = mine_hi;
    }
}

// Warp per token: non-zero word count and document frequency.
__global__ void token_stats(const unsigned long long* __restrict__ dense, uint32_t L, size_t W,
                            uint32_t* __restrict__ nzc, uint32_t* __restrict__ df) {
    const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (size_t t = warp; t < L; t += ((size_t)gridDim.x * blockDim.x) >> 5) {
        uint32_t nz = 0, pc = 0;
        for (size_t w = lane; w < W; w += 32) {
            const unsigned long long v = dense[t * W + w];
            nz += v != 0ull;
            pc += __popcll(v);
        }
        for (int o = 16; o; o >>= 1) {
            nz += __shfl_xor_sync(kFull, nz, o);
            pc += __shfl_xor_sync(kFull, pc, o);
        }
        if (lane == 0) {
            nzc[t] = nz;
            df[t] = pc;
        }
    }
}

__global__ void fill_nonzero(const unsigned long long* __restrict__ dense, uint32_t L, size_t W,
                             const uint32_t* __restrict__ off, uint32_t* __restrict__ idx) {
    const size_t warp = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (size_t t = warp; t < L; t += ((size_t)gridDim.x * blockDim.x) >> 5) {
        uint32_t o = off[t];
        for (size_t w0 = 0; w0 < W; w0 += 32) {
            const size_t w = w0 + lane;
            const bool nz = w < W && dense[t * W + w] != 0ull;
            const uint32_t m = __ballot_sync(kFull, nz);
            if (nz) idx[o + __popc(m & ((1u << lane) - 1u))] = (uint32_t)w;
            o += __popc(m);
        }
    }
}

__global__ void pattern_token_count(const int64_t* __restrict__ pat, size_t np, int k, uint32_t* __restrict__ cnt) {
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (size_t)gridDim.x * blockDim.x) {
        uint32_t c = 0;
        for (int w = 0; w < k; ++w) c += __popcll((unsigned long long)pat[p * k + w]);
        cnt[p] = c;
    }
}

// Token list of each pattern sorted by (df, token) when it has at most
// kMaxSorted tokens; longer lists keep bit order after moving the rarest first.
__global__ void pattern_token_fill(const int64_t* __restrict__ pat, size_t np, int k, const uint32_t* __restrict__ df,
                                   const uint32_t* __restrict__ off, uint16_t* __restrict__ toks) {
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (size_t)gridDim.x * blockDim.x) {
        const uint32_t o = off[p];
        const uint32_t total = off[p + 1] - o;
        if (total <= kMaxSorted) {
            uint32_t key[kMaxSorted];
            int m = 0;
            for (int w = 0; w < k; ++w) {
                uint64_t x = (uint64_t)pat[p * k + w];
                while (x) {
                    const int b = __ffsll((long long)x) - 1;
                    x &= x - 1;
                    const uint32_t t = (uint32_t)w * 64 + b;
                    const uint32_t dt = df[t];
                    int i = m++;
                    while (i > 0) {
                        const uint32_t u = key[i - 1];
                        const uint32_t du = df[u];
                        if (du < dt || (du == dt && u < t)) break;
                        key[i] = u;
                        --i;
                    }
                    key[i] = t;
                }
            }
            for (int i = 0; i < m; ++i) toks[o + i] = (uint16_t)key[i];
        } else {
            uint32_t n = 0, best = 0, bestdf = 0xffffffffu;
            for (int w = 0; w < k; ++w) {
                uint64_t x = (uint64_t)pat[p * k + w];
                while (x) {
                    const int b = __ffsll((long long)x) - 1;
                    x &= x - 1;
                    const uint32_t t = (uint32_t)w * 64 + b;
                    if (df[t] < bestdf) {
                        bestdf = df[t];
                        best = n;
                    }
                    toks[o + n++] = (uint16_t)t;
                }
            }
            const uint16_t tmp = toks[o];
            toks[o] = toks[o + best];
            toks[o + best] = tmp;
        }
    }
}

enum Mode : int { kMatch = 0, kSupport = 1, kCover = 2 };

// Warp per pattern over the CSR token lists.
template <int MODE>
__global__ void __launch_bounds__(256)
posting_scan(const unsigned long long* __restrict__ dense, size_t W, const uint32_t* __restrict__ nz_off,
             const uint32_t* __restrict__ nz_idx, size_t n_rows, const uint32_t* __restrict__ tok_off,
             const uint16_t* __restrict__ toks, size_t np, const int64_t* __restrict__ scores,
             unsigned long long* __restrict__ acc, int64_t* __restrict__ support_out, uint8_t* __restrict__ cover_out,
             int* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    const size_t warps = ((size_t)gridDim.x * blockDim.x) >> 5;
    bool ovf = false;
    for (size_t p = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < np; p += warps) {
        const uint32_t o = tok_off[p];
        const uint32_t m = tok_off[p + 1] - o;
        if (m == 0) {
            // the empty pattern is a subset of every row
            if (MODE == kSupport) {
                if (lane == 0) support_out[p] = (int64_t)n_rows;
            } else if (MODE == kCover) {
                if (lane == 0) cover_out[p] = n_rows > 0 ? 1 : 0;
            } else {
                const unsigned long long s = (unsigned long long)scores[p];
                for (size_t r = lane; r < n_rows; r += 32) {
                    const unsigned long long old = atomicAdd(acc + r, s);
                    if (old + s > (unsigned long long)INT64_MAX) ovf = true;
                }
            }
            continue;
        }
        const uint32_t tl = lane < m ? (uint32_t)toks[o + lane] : 0u;
        const uint32_t t1 = __shfl_sync(kFull, tl, 0);
        const uint32_t beg = nz_off[t1], end = nz_off[t1 + 1];
        const unsigned long long* p1 = dense + (size_t)t1 * W;
        unsigned long long s = 0;
        if (MODE == kMatch) s = (unsigned long long)scores[p];
        uint32_t cnt = 0;
        bool hit = false;
        for (uint32_t j0 = beg; j0 < end; j0 += 32) {
            const uint32_t j = j0 + lane;
            const uint32_t w = j < end ? nz_idx[j] : 0u;
            unsigned long long mw = j < end ? p1[w] : 0ull;
            for (uint32_t i = 1; i < m; ++i) {
                if (!__any_sync(kFull, mw != 0ull)) break;
                const uint32_t t = i < 32 ? __shfl_sync(kFull, tl, i) : (uint32_t)toks[o + i];
                if (mw) mw &= dense[(size_t)t * W + w];
            }
            if (MODE == kSupport) {
                cnt += __popcll(mw);
            } else if (MODE == kCover) {
                if (__any_sync(kFull, mw != 0ull)) {
                    hit = true;
                    break;
                }
            } else {
                while (mw) {
                    const int b = __ffsll((long long)mw) - 1;
                    mw &= mw - 1;
                    const unsigned long long old = atomicAdd(acc + (size_t)w * 64 + b, s);
                    if (old + s > (unsigned long long)INT64_MAX) ovf = true;
                }
            }
        }
        if (MODE == kSupport) {
            for (int o2 = 16; o2; o2 >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o2);
            if (lane == 0) support_out[p] = (int64_t)cnt;
        } else if (MODE == kCover) {
            if (lane == 0) cover_out[p] = hit ? 1 : 0;
        }
    }
    if (MODE == kMatch && ovf) atomicOr(flags, 1);
}

__global__ void scatter_u64(const unsigned long long* __restrict__ src, const uint32_t* __restrict__ perm, size_t n,
                            int64_t* __restrict__ dst) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[perm[i]] = (int64_t)src[i];
}

// CSR token lists of `np` patterns ordered by the document frequency of P.
struct PatternTokens {
    DevBuf off, toks;
};

void pattern_tokens(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, PatternTokens& T) {
    DevBuf cnt((np + 1) * 4, ctx.stream);
    T.off.alloc((np + 1) * 4, ctx.stream);
    IGB_LAUNCH(ctx, pattern_token_count, grid_for(ctx, np, 256), 256, 0, d_pat, np, (int)k, cnt.as<uint32_t>());
    IGB_CUDA(cudaMemsetAsync(cnt.as<uint32_t>() + np, 0, 4, ctx.stream));
    size_t tb = 0;
    IGB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.as<uint32_t>(), T.off.as<uint32_t>(), (int64_t)np + 1,
                                           ctx.stream));
    DevBuf temp(tb, ctx.stream);
    IGB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, cnt.as<uint32_t>(), T.off.as<uint32_t>(), (int64_t)np + 1,
                                           ctx.stream));
    uint32_t total = 0;
    IGB_CUDA(cudaMemcpyAsync(&total, T.off.as<uint32_t>() + np, 4, cudaMemcpyDeviceToHost, ctx.stream));
    IGB_CUDA(cudaStreamSynchronize(ctx.stream));
    T.toks.alloc(std::max<size_t>(total, 1) * 2, ctx.stream);
    IGB_LAUNCH(ctx, pattern_token_fill, grid_for(ctx, np, 128), 128, 0, d_pat, np, (int)k, P.df.as<uint32_t>(),
               T.off.as<uint32_t>(), T.toks.as<uint16_t>());
}

template <int MODE>
void launch_scan(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, const int64_t* scores,
                 unsigned long long* acc, int64_t* support, uint8_t* cover, int* flags) {
    if (np == 0) return;
    PatternTokens T;
    pattern_tokens(ctx, d_pat, np, k, P, T);
    const size_t blocks = std::min<size_t>((np + 7) / 8, (size_t)ctx.sm_count * 64);
    IGB_LAUNCH(ctx, posting_scan<MODE>, (unsigned)blocks, 256, 0, P.dense.as<unsigned long long>(), P.W,
               P.nz_off.as<uint32_t>(), P.nz_idx.as<uint32_t>(), P.n, T.off.as<uint32_t>(), T.toks.as<uint16_t>(), np,
               scores, acc, support, cover, flags);
}

}  // namespace

bool postings_supported(uint32_t L, size_t n) { return words_for(L) * 64 < 65535 && n < 0xffffffffull; }

void build_postings(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, uint32_t /*logical_len*/, Postings& P,
                    bool canonical) {
    const uint32_t L = (uint32_t)(64 * k);  // every bit position, padding included
    P.L = L;
    P.n = n;
    P.W = (n + 63) / 64;
    const size_t W = std::max<size_t>(P.W, 1);
    P.dense.alloc((size_t)L * W * 8, ctx.stream);
    P.df.alloc((size_t)L * 4, ctx.stream);
    P.nz_off.alloc(((size_t)L + 1) * 4, ctx.stream);
    P.perm.release();
    DevBuf nzc(((size_t)L + 1) * 4, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(P.dense.p, 0, (size_t)L * W * 8, ctx.stream));
    if (canonical && n > 1) {
        P.perm.alloc(n * 4, ctx.stream);
        sort_rows_canonical(ctx, d_rows, n, k, P.perm.as<uint32_t>());
    }
    if (n && k) {
        const size_t warps = P.W * k;
        IGB_LAUNCH(ctx, transpose_rows, grid_for(ctx, warps * 32, 256), 256, 0, d_rows, P.perm.as<uint32_t>(), n,
                   (int)k, P.W, P.dense.as<unsigned long long>());
    }
    IGB_LAUNCH(ctx, token_stats, grid_for(ctx, (size_t)L * 32, 256), 256, 0, P.dense.as<unsigned long long>(), L,
               P.W, nzc.as<uint32_t>(), P.df.as<uint32_t>());
    IGB_CUDA(cudaMemsetAsync(nzc.as<uint32_t>() + L, 0, 4, ctx.stream));
    size_t tb = 0;
    IGB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, nzc.as<uint32_t>(), P.nz_off.as<uint32_t>(), (int64_t)L + 1,
                                           ctx.stream));
    DevBuf temp(tb, ctx.stream);
    IGB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, nzc.as<uint32_t>(), P.nz_off.as<uint32_t>(), (int64_t)L + 1,
                                           ctx.stream));
    uint32_t total = 0;
    IGB_CUDA(cudaMemcpyAsync(&total, P.nz_off.as<uint32_t>() + L, 4, cudaMemcpyDeviceToHost, ctx.stream));
    IGB_CUDA(cudaStreamSynchronize(ctx.stream));
    P.nz_total = total;
    P.nz_idx.alloc(std::max<size_t>(total, 1) * 4, ctx.stream);
    IGB_LAUNCH(ctx, fill_nonzero, grid_for(ctx, (size_t)L * 32, 256), 256, 0, P.dense.as<unsigned long long>(), L,
               P.W, P.nz_off.as<uint32_t>(), P.nz_idx.as<uint32_t>());
}

void posting_support(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, int64_t* d_support) {
    launch_scan<kSupport>(ctx, d_pat, np, k, P, nullptr, nullptr, d_support, nullptr, nullptr);
}

void posting_cover(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, uint8_t* d_mask) {
    launch_scan<kCover>(ctx, d_pat, np, k, P, nullptr, nullptr, nullptr, d_mask, nullptr);
}

void posting_match(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* d_scores, const Postings& P,
                   int64_t* d_out, int* d_overflow) {
    const size_t n = std::max<size_t>(P.n, 1);
    if (!P.perm.p) {
        IGB_CUDA(cudaMemsetAsync(d_out, 0, n * 8, ctx.stream));
        launch_scan<kMatch>(ctx, d_pat, np, k, P, d_scores, reinterpret_cast<unsigned long long*>(d_out), nullptr,
                            nullptr, d_overflow);
        return;
    }
    // accumulate in the postings' (canonical) row order, then scatter back
    DevBuf acc(n * 8, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(acc.p, 0, n * 8, ctx.stream));
    launch_scan<kMatch>(ctx, d_pat, np, k, P, d_scores, acc.as<unsigned long long>(), nullptr, nullptr, d_overflow);
    IGB_LAUNCH(ctx, scatter_u64, grid_for(ctx, P.n, 256), 256, 0, acc.as<unsigned long long>(), P.perm.as<uint32_t>(),
               P.n, d_out);
}

}  // namespace igb
