// posting.cu — the vertical (posting-bitmap) form of the subset test, used for
// support (kernel 5), coverage (kernel 4) and the matcher (kernel 6).
//
// Same semantics as subset.cu (words::is_subset, bitpack.hpp:37-43), other
// data layout.  For a row set R of n rows, post[t] is the n-bit set of rows
// that contain bit t (all 64·K bit positions × W = ceil(n/64) words;
// L2-resident at NSL shape).  Then
//     {r ∈ R : b ⊆ r} = AND_{t ∈ b} post[t]
// so a pattern costs |b| word-ANDs per 64 rows instead of K word tests per row
// (|b| ≈ 17 tokens vs 64·K = 896 bits at NSL shape).  Rows are ordered first
// so that rows sharing tokens share posting words: training rows canonically,
// test rows in cluster order (reflected-Gray lexicographic over tokens ranked
// most frequent first), which makes a pattern's matching rows long runs.  Each
// pattern's tokens are listed rarest first in one rank space (a PatternIndex,
// built once per pattern set and reused by every scan of it); patterns sharing
// their three rarest tokens (t1, t2, t3) share one word list, filtered from
// their (t1, t2) parent's list, and a warp walks that list 32 words per step,
// ANDing the next tokens until
// no lane has a surviving row.  Exact and independent of every order involved:
//   support  = Σ popcount(...)
//   covered  = any word non-zero                             (kernels.cpp:59-65)
//   evidence = Σ_p s_p over surviving rows, accumulated as a difference array
//              of runs (+s at a run's first row, -s after its last, then one
//              scan) when Σ s_p <= INT64_MAX, else with checked u64 atomics;
//              used only when all scores are >= 0, where "some prefix overflows"
//              ⟺ "the total exceeds INT64_MAX" (kernels.cpp:40-46).
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <type_traits>
#include <cstdlib>
#include <vector>

#include "ig_internal.cuh"
#include "posting.cuh"

namespace igb {

namespace {

constexpr unsigned kFull = 0xffffffffu;

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

// Token lists for rows wider than the rank-bitmap kernel takes (K > 64); df is
// staged in shared memory (L <= 64*K words of 4 bytes).
__global__ void pattern_token_fill(const int64_t* __restrict__ pat, size_t np, int k, const uint32_t* __restrict__ gdf,
                                   uint32_t L, const uint32_t* __restrict__ off, uint16_t* __restrict__ toks) {
    // Wide rows (K > 64): the kTop rarest tokens first, in (df, token) order
    // (they hold the group key), then the rest in bit order — O(|b| * kTop)
    // instead of a per-pattern sort.  Any order is exact; rarest-first only
    // makes the scans exit sooner.
    constexpr int kTop = 8;
    extern __shared__ uint32_t df[];
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) df[i] = gdf[i];
    __syncthreads();
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (size_t)gridDim.x * blockDim.x) {
        const uint32_t o = off[p];
        uint64_t top[kTop];
#pragma unroll
        for (int i = 0; i < kTop; ++i) top[i] = ~0ull;
        uint32_t m = 0;
        for (int w = 0; w < k; ++w) {
            uint64_t x = (uint64_t)pat[p * k + w];
            while (x) {
                const int b = __ffsll((long long)x) - 1;
                x &= x - 1;
                const uint32_t t = (uint32_t)w * 64 + b;
                const uint64_t kt = ((uint64_t)df[t] << 16) | t;
                ++m;
                if (kt < top[kTop - 1]) {
                    top[kTop - 1] = kt;
#pragma unroll
                    for (int i = kTop - 1; i > 0; --i)
                        if (top[i] < top[i - 1]) {
                            const uint64_t tmp = top[i];
                            top[i] = top[i - 1];
                            top[i - 1] = tmp;
                        }
                }
            }
        }
        const uint32_t nt = m < (uint32_t)kTop ? m : (uint32_t)kTop;
#pragma unroll
        for (int i = 0; i < kTop; ++i)
            if ((uint32_t)i < nt) toks[o + i] = (uint16_t)(top[i] & 0xffffu);
        if (m > (uint32_t)kTop) {
            const uint64_t thr = top[kTop - 1];
            uint32_t idx = kTop;
            for (int w = 0; w < k; ++w) {
                uint64_t x = (uint64_t)pat[p * k + w];
                while (x) {
                    const int b = __ffsll((long long)x) - 1;
                    x &= x - 1;
                    const uint32_t t = (uint32_t)w * 64 + b;
                    if ((((uint64_t)df[t] << 16) | t) > thr) toks[o + idx++] = (uint16_t)t;
                }
            }
        }
    }
}

// Rank-space variant: with byrank[] = tokens sorted by (df, token) and rank[]
// its inverse, re-indexing a pattern's bits by rank and reading them back in
// bit order lists its tokens rarest first with no per-pattern sort: O(|b| + K).
// The rank-space bitmap of each thread lives in shared memory (word-major,
// thread-minor: conflict-free) and is set with shared atomics whose result is
// unused, so consecutive bits do not wait on each other's read-modify-write
// (a local-memory array made every bit one dependent L1 round trip: -22 %).
// Staging the rows and the output through shared memory as well was slower
// (occupancy).
constexpr int kRankWords = 64;
constexpr int kFillThreads = 128;
template <int KW>
__global__ void __launch_bounds__(kFillThreads)
pattern_token_fill_rank(const int64_t* __restrict__ pat, size_t np, int k, const uint16_t* __restrict__ grank,
                        const uint16_t* __restrict__ gbyrank, uint32_t L, const uint32_t* __restrict__ off,
                        uint16_t* __restrict__ toks) {
    extern __shared__ uint32_t fsm[];
    uint32_t* rb = fsm;  // [2 * KW][kFillThreads]
    uint16_t* rank = reinterpret_cast<uint16_t*>(fsm + 2 * KW * kFillThreads);
    uint16_t* byrank = rank + L;
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) {
        rank[i] = grank[i];
        byrank[i] = gbyrank[i];
    }
    __syncthreads();
    // this thread's rank bitmap: a column of rb only it touches (plain
    // read-modify-writes, conflict-free across the warp), cleared as it is read
    uint32_t* my = rb + threadIdx.x;
    const int nw = 2 * k;  // 32-bit rank words
    for (int q = 0; q < nw; ++q) my[q * kFillThreads] = 0u;
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (size_t)gridDim.x * blockDim.x) {
        // the row's words first, all loads in flight at once (KW >= k)
        uint64_t row[KW];
#pragma unroll
        for (int w = 0; w < KW; ++w) row[w] = w < k ? (uint64_t)__ldg(pat + p * k + w) : 0ull;
#pragma unroll
        for (int w = 0; w < KW; ++w) {
            uint64_t x = row[w];
            while (x) {
                const int b = __ffsll((long long)x) - 1;
                x &= x - 1;
                const uint32_t r = rank[w * 64 + b];
                my[(r >> 5) * kFillThreads] |= 1u << (r & 31);
            }
        }
        // tokens out four at a time (one 8-byte store instead of four 2-byte
        // ones: the scattered 2-byte stores were one L2 write each)
        uint32_t o = off[p];
        unsigned long long buf = 0;
        uint32_t nb = 0;
        for (int q = 0; q < nw; ++q) {
            uint32_t y = my[q * kFillThreads];
            if (y) my[q * kFillThreads] = 0u;
            while (y) {
                const int b = __ffs((int)y) - 1;
                y &= y - 1;
                const uint16_t t = byrank[q * 32 + b];
                if (nb == 0 && (o & 3u)) {
                    toks[o++] = t;  // up to the next 8-byte boundary
                    continue;
                }
                buf |= (unsigned long long)t << (16 * nb);
                if (++nb == 4) {
                    *reinterpret_cast<unsigned long long*>(toks + o) = buf;
                    o += 4;
                    buf = 0;
                    nb = 0;
                }
            }
        }
        for (uint32_t i = 0; i < nb; ++i) toks[o + i] = (uint16_t)(buf >> (16 * i));
    }
}

__global__ void rank_keys(const uint32_t* __restrict__ df, uint32_t L, unsigned long long* __restrict__ key,
                          uint16_t* __restrict__ tok, bool descending) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < L; t += gridDim.x * blockDim.x) {
        key[t] = ((unsigned long long)(descending ? 0xffffffffu - df[t] : df[t]) << 16) | t;
        tok[t] = (uint16_t)t;
    }
}

// Small token universes (L <= kRankCount): rank by counting against the keys
// staged in shared memory — one launch instead of a radix sort's passes.
constexpr uint32_t kRankCount = 4096;
__global__ void rank_by_key_count(const uint32_t* __restrict__ df, uint32_t L, bool descending,
                                  uint16_t* __restrict__ rank, uint16_t* __restrict__ byrank) {
    __shared__ unsigned long long key[kRankCount];
    for (uint32_t t = threadIdx.x; t < L; t += blockDim.x)
        key[t] = ((unsigned long long)(descending ? 0xffffffffu - df[t] : df[t]) << 16) | t;
    __syncthreads();
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < L; t += gridDim.x * blockDim.x) {
        const unsigned long long k = key[t];
        uint32_t r = 0;
        for (uint32_t j = 0; j < L; ++j) r += key[j] < k ? 1u : 0u;
        rank[t] = (uint16_t)r;
        byrank[r] = (uint16_t)t;
    }
}

__global__ void invert_rank(const uint16_t* __restrict__ byrank, uint32_t L, uint16_t* __restrict__ rank) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < L; r += gridDim.x * blockDim.x) rank[byrank[r]] = (uint16_t)r;
}

__global__ void minus_one(uint32_t* __restrict__ v, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) v[i] -= 1;
}

enum Mode : int { kMatch = 0, kSupport = 1, kCover = 2, kMatchChecked = 3 };

// dst[perm[i]] = src[group ? group[i] : i] for every canonical position i.
__global__ void scatter_u64(const unsigned long long* __restrict__ src, const uint32_t* __restrict__ perm,
                            const uint32_t* __restrict__ group, size_t n, int64_t* __restrict__ dst) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[perm[i]] = (int64_t)src[group ? group[i] : i];
}

__global__ void row_heads(const int64_t* __restrict__ rows, const uint32_t* __restrict__ perm, size_t n, int k,
                          uint32_t* __restrict__ head) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = 1;
        if (i > 0) {
            const int64_t* a = rows + (size_t)perm[i] * k;
            const int64_t* b = rows + (size_t)perm[i - 1] * k;
            h = 0;
            for (int w = 0; w < k; ++w)
                if (a[w] != b[w]) {
                    h = 1;
                    break;
                }
        }
        head[i] = h;
    }
}

// exclusive sum of heads -> group index of each position (heads start a new group)
__global__ void fix_group(const uint32_t* __restrict__ head, size_t n, uint32_t* __restrict__ group) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        group[i] = group[i] + head[i] - 1;
}

// Pattern-index helper kernels (host functions below, outside this namespace).
__global__ void add_u32(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint32_t n,
                        uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = a[i] + b[i];
}

// subset index: the chosen source patterns' token-list extents
__global__ void sub_lists(const uint32_t* __restrict__ src_beg, const uint32_t* __restrict__ src_len,
                          const uint32_t* __restrict__ src_of, size_t n, uint32_t* __restrict__ beg,
                          uint32_t* __restrict__ len) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const uint32_t s = src_of[i];
        beg[i] = src_beg[s];
        len[i] = src_len[s];
    }
}

__global__ void fill_u32(uint32_t* __restrict__ p, size_t n, uint32_t v) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

__global__ void scatter_pos(const uint32_t* __restrict__ src_of, size_t n, uint32_t* __restrict__ inv) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        inv[src_of[i]] = (uint32_t)i;
}

// walk the source's group order, keeping the chosen patterns (their new index)
// and their old group id
__global__ void map_order(const uint32_t* __restrict__ order, const uint32_t* __restrict__ gid, size_t n,
                          const uint32_t* __restrict__ inv, uint32_t* __restrict__ val, uint32_t* __restrict__ og,
                          uint8_t* __restrict__ keep) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const uint32_t p = inv[order[i]];
        val[i] = p;
        og[i] = gid[i];
        keep[i] = p != 0xffffffffu ? 1 : 0;
    }
}

__global__ void gather_u64k(const unsigned long long* __restrict__ src, const uint32_t* __restrict__ idx, size_t n,
                            unsigned long long* __restrict__ dst) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[idx[i]];
}



// ------------------------------------------------------------------ grouped scan
// Patterns sharing their two rarest tokens (t1, t2) share the word list
// S = {(w, post[t1][w] & post[t2][w]) != 0}: it is built once per group (warp per
// group over the non-zero words of t1) and every pattern of the group walks S
// instead of all non-zero words of t1, ANDing only its remaining tokens.  At
// C3 ~1M patterns fall into ~35k groups, so most of the (t1, t2) work is shared.
constexpr uint32_t kNoTok = 0xffffu;

// sort key of a pattern: its q rarest tokens (t1, t2, t3, ...; absent = all
// ones), b bits each, t1 most significant (q*b <= 64 bits, one radix sort).
// The group is (t1, t2, t3).  expand_keys
// restores the group part as (t1 << 32) | (t2 << 16) | t3 with kNoTok, which
// sorts identically.
__global__ void group_keys(const uint32_t* __restrict__ tok_beg, const uint32_t* __restrict__ tok_len,
                           const uint16_t* __restrict__ toks, size_t np, int b, int q,
                           unsigned long long* __restrict__ key, uint32_t* __restrict__ idx) {
    const unsigned long long none = (1ull << b) - 1ull;
    for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < np; p += (size_t)gridDim.x * blockDim.x) {
        const uint32_t o = tok_beg[p], m = tok_len[p];
        unsigned long long k = 0;
        for (int i = 0; i < q; ++i) k = (k << b) | ((uint32_t)i < m ? (unsigned long long)toks[o + i] : none);
        key[p] = k;
        idx[p] = (uint32_t)p;
    }
}

__global__ void expand_keys(unsigned long long* __restrict__ key, size_t n, int b, int q) {
    const unsigned long long none = (1ull << b) - 1ull;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const unsigned long long x = key[i];
        unsigned long long t[3] = {(x >> ((q - 1) * b)) & none, (x >> ((q - 2) * b)) & none, (x >> ((q - 3) * b)) & none};
        for (auto& v : t)
            if (v == none) v = kNoTok;
        key[i] = (t[0] << 32) | (t[1] << 16) | t[2];
    }
}

template <class K>
__global__ void group_heads(const K* __restrict__ key, size_t np, uint8_t* __restrict__ head,
                            uint32_t* __restrict__ head32) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (size_t)gridDim.x * blockDim.x) {
        const uint8_t h = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
        head[i] = h;
        head32[i] = h;
    }
}

// parent (t1, t2) key of every (t1, t2, t3) group
__global__ void parent_keys(const unsigned long long* __restrict__ gkey, size_t G, uint32_t* __restrict__ pk) {
    for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < G; g += (size_t)gridDim.x * blockDim.x)
        pk[g] = (uint32_t)(gkey[g] >> 16);
}

// upper bound of a 3-group's list: its parent's upper bound
__global__ void child_bound(const uint32_t* __restrict__ pid, size_t G, const unsigned long long* __restrict__ pub,
                            unsigned long long* __restrict__ ub) {
    for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < G; g += (size_t)gridDim.x * blockDim.x)
        ub[g] = pub[pid[g]];
}

// Warp per (t1, t2, t3) group: its parent (t1, t2) list filtered by post[t3].
__global__ void child_lists(const unsigned long long* __restrict__ gkey, const uint32_t* __restrict__ pid, size_t G,
                            const unsigned long long* __restrict__ dense, size_t W,
                            const unsigned long long* __restrict__ poff, const uint32_t* __restrict__ plen,
                            const uint32_t* __restrict__ pw, const unsigned long long* __restrict__ pm,
                            const unsigned long long* __restrict__ goff, uint32_t* __restrict__ glen,
                            uint32_t* __restrict__ ew, unsigned long long* __restrict__ em) {
    const int lane = threadIdx.x & 31;
    const size_t warps = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t g = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < G; g += warps) {
        const uint32_t t3 = (uint32_t)(gkey[g] & 0xffffu);
        const uint32_t par = pid[g];
        const unsigned long long pb = poff[par], base = goff[g];
        const uint32_t len = plen[par];
        uint32_t cnt = 0;
        for (uint32_t j0 = 0; j0 < len; j0 += 32) {
            const uint32_t j = j0 + lane;
            uint32_t w = 0;
            unsigned long long m = 0;
            if (j < len) {
                w = pw[pb + j];
                m = pm[pb + j];
                if (t3 != kNoTok) m &= dense[(size_t)t3 * W + w];
            }
            const uint32_t bal = __ballot_sync(kFull, m != 0ull);
            if (m) {
                const uint32_t pos = cnt + __popc(bal & ((1u << lane) - 1u));
                ew[base + pos] = w;
                em[base + pos] = m;
            }
            cnt += __popc(bal);
        }
        if (lane == 0) glen[g] = cnt;
    }
}

// upper bound of each group's list: non-zero words of t1 (all words without t1)
__global__ void group_bound(const uint32_t* __restrict__ gkey, size_t G, const uint32_t* __restrict__ nz_off,
                            size_t W, unsigned long long* __restrict__ ub) {
    for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < G; g += (size_t)gridDim.x * blockDim.x) {
        const uint32_t t1 = gkey[g] >> 16;
        ub[g] = t1 == kNoTok ? (unsigned long long)W : (unsigned long long)(nz_off[t1 + 1] - nz_off[t1]);
    }
}

// Warp per group: S = non-zero (w, post[t1][w] & post[t2][w]).
__global__ void group_lists(const uint32_t* __restrict__ gkey, size_t G, const unsigned long long* __restrict__ dense,
                            size_t W, size_t n_rows, const uint32_t* __restrict__ nz_off,
                            const uint32_t* __restrict__ nz_idx, const unsigned long long* __restrict__ goff,
                            uint32_t* __restrict__ glen, uint32_t* __restrict__ ew, unsigned long long* __restrict__ em) {
    const int lane = threadIdx.x & 31;
    const size_t warps = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t g = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < G; g += warps) {
        const uint32_t t1 = gkey[g] >> 16, t2 = gkey[g] & 0xffffu;
        const uint32_t beg = t1 == kNoTok ? 0u : nz_off[t1];
        const uint32_t end = t1 == kNoTok ? (uint32_t)W : nz_off[t1 + 1];
        const unsigned long long base = goff[g];
        uint32_t cnt = 0;
        for (uint32_t j0 = beg; j0 < end; j0 += 32) {
            const uint32_t j = j0 + lane;
            unsigned long long m = 0;
            uint32_t w = 0;
            if (j < end) {
                if (t1 == kNoTok) {
                    w = j;
                    const size_t lo = (size_t)w * 64;
                    m = n_rows - lo >= 64 ? ~0ull : ((1ull << (n_rows - lo)) - 1ull);
                } else {
                    w = nz_idx[j];
                    m = dense[(size_t)t1 * W + w];
                    if (t2 != kNoTok) m &= dense[(size_t)t2 * W + w];
                }
            }
            const uint32_t bal = __ballot_sync(kFull, m != 0ull);
            if (m) {
                const uint32_t pos = cnt + __popc(bal & ((1u << lane) - 1u));
                ew[base + pos] = w;
                em[base + pos] = m;
            }
            cnt += __popc(bal);
        }
        if (lane == 0) glen[g] = cnt;
    }
}

// Warp-cooperative scatter of the set bits of every lane's (word w, mask mw):
// bit q of the warp's concatenated hits goes to lane q % 32, which finds its
// source lane by binary search over the shuffled prefix counts and the bit with
// __fns, so the REDs are spread evenly over the lanes instead of each lane
// walking its own mask (the masks are very uneven).  Call with all 32 lanes.
template <bool CHECKED>
__device__ __forceinline__ void warp_scatter_hits(uint32_t w, unsigned long long mw, unsigned long long s,
                                                  unsigned long long* __restrict__ acc, bool& ovf) {
    const int lane = threadIdx.x & 31;
    const uint32_t lo = (uint32_t)mw, hi = (uint32_t)(mw >> 32);
    const uint32_t c = __popc(lo) + __popc(hi);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - c;
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    for (uint32_t q0 = 0; q0 < total; q0 += 32) {
        const uint32_t q = q0 + lane;
        int L = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
            const uint32_t e = __shfl_sync(kFull, excl, L + step);
            if (e <= q) L += step;
        }
        const uint32_t r = q - __shfl_sync(kFull, excl, L);
        const uint32_t slo = __shfl_sync(kFull, lo, L), shi = __shfl_sync(kFull, hi, L);
        const uint32_t sw = __shfl_sync(kFull, w, L);
        if (q < total) {
            const uint32_t plo = __popc(slo);
            const uint32_t bit = r < plo ? __fns(slo, 0, (int)r + 1) : 32u + __fns(shi, 0, (int)(r - plo) + 1);
            unsigned long long* dst = acc + (size_t)sw * 64 + bit;
            if (CHECKED) {
                const unsigned long long old = atomicAdd(dst, s);
                if (old + s > (unsigned long long)INT64_MAX) ovf = true;
            } else {
                atomicAdd(dst, s);
            }
        }
    }
}

// Warp per pattern (in group order): walk the group's list, AND tokens 3.., then
// match (difference-array runs) / support (popcount) / cover (any).
//
// ld_tok: posting word of token t at the lane's column, col + t * (W * 8)
// bytes, the address formed by one IMAD.WIDE.U32 on the FMA pipe (the
// multiplier is a runtime value, so it is not strength-reduced into the
// 64-bit add + LEA pair that would land on the ALU pipe this kernel saturates).
// Through L1 (ld.global.nc): 64 % of the sectors hit there (neighbouring
// patterns share tokens); L2-only loads (.cg, .L1::no_allocate) measured
// 40-80 % slower.
__device__ __forceinline__ unsigned long long ld_tok(const unsigned long long* col, uint32_t t, uint32_t wbytes) {
    unsigned long long v;
    asm("{\n\t.reg .u64 a;\n\tmad.wide.u32 a, %1, %2, %3;\n\tld.global.nc.u64 %0, [a];\n\t}"
        : "=l"(v) : "r"(t), "r"(wbytes), "l"(col));
    return v;
}

// COUNT (diagnostics): the same control flow with every output suppressed;
// each lane counts the posting word-ANDs it performs on live list words (the
// useful work of the roofline), summed into *work.
template <int MODE, bool COUNT = false>
__global__ void __launch_bounds__(256)
grouped_scan(const unsigned long long* __restrict__ dense, size_t W, size_t n_rows,
             const uint32_t* __restrict__ tok_beg, const uint32_t* __restrict__ tok_len,
             const uint16_t* __restrict__ toks, size_t np,
             const uint32_t* __restrict__ order, const uint32_t* __restrict__ gid,
             const unsigned long long* __restrict__ goff, const uint32_t* __restrict__ glen,
             const uint32_t* __restrict__ ew, const unsigned long long* __restrict__ em,
             const int64_t* __restrict__ scores, unsigned long long* __restrict__ acc,
             int64_t* __restrict__ support_out, uint8_t* __restrict__ cover_out, int* __restrict__ flags,
             unsigned long long* __restrict__ work, const uint32_t* __restrict__ sel) {
    const int lane = threadIdx.x & 31;
    const size_t warps = ((size_t)gridDim.x * blockDim.x) >> 5;
    // matcher: per warp, the current pattern's tokens 3..34, read four at a
    // time as one 16-byte broadcast instead of four shuffles (C3 matcher -3 %;
    // support and coverage patterns are too short to repay the store)
    constexpr bool kSmemTok = MODE == kMatch || MODE == kMatchChecked;
    __shared__ __align__(16) uint32_t s_off[8][32];
    uint32_t* so = s_off[(threadIdx.x >> 5) & 7];
    bool ovf = false;
    unsigned long long nand = 0;  // COUNT only
    for (size_t i0 = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i0 < np; i0 += warps) {
        const size_t i = sel ? sel[i0] : i0;  // np positions: all, or the selected subset
        const uint32_t p = order[i];
        const uint32_t g = gid[i];
        const uint32_t o = tok_beg[p];
        const uint32_t m = tok_len[p];
        const uint32_t Wu = (uint32_t)W, wb = Wu * 8u;
        // lane l holds token l (l < m); lanes past the pattern repeat token 0,
        // whose posting already contains every surviving word of the group
        // list, so ANDing it again is a no-op
        const uint32_t t0 = m ? (uint32_t)toks[o] : 0u;
        const uint32_t tl = lane < m ? (uint32_t)toks[o + lane] : t0;
        if (kSmemTok) {
            __syncwarp();  // the previous pattern's tokens are read
            so[lane >= 3 ? lane - 3 : 29 + lane] = lane >= 3 ? tl : t0;
            __syncwarp();
        }
        const unsigned long long base = goff[g];
        const uint32_t len = glen[g];
        unsigned long long s = 0;
        if (MODE == kMatch || MODE == kMatchChecked) s = (unsigned long long)scores[p];
        uint32_t cnt = 0;
        bool hit = false;
        for (uint32_t j0 = 0; j0 < len; j0 += 32) {
            const uint32_t j = j0 + lane;
            const uint32_t w = j < len ? ew[base + j] : 0u;
            unsigned long long mw = j < len ? em[base + j] : 0ull;
            const unsigned long long* col = dense + w;
            // tokens 3..31 (0..2 are the group key, already applied in the
            // list), four per round; offsets past the pattern are token 0's
            // (no-ops); the rare tail past 32 is read from memory
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int t = 3 + 4 * q;
                if ((uint32_t)t >= m) break;
                const bool live = mw != 0ull;
                if (!__any_sync(kFull, live)) break;
                uint4 tw;
                if (kSmemTok) {
                    tw = reinterpret_cast<const uint4*>(so)[q];
                } else {  // compile-time shuffle lanes; 32..34 wrap to tokens 0..2 (no-ops)
                    tw.x = __shfl_sync(kFull, tl, t);
                    tw.y = __shfl_sync(kFull, tl, (t + 1) & 31);
                    tw.z = __shfl_sync(kFull, tl, (t + 2) & 31);
                    tw.w = __shfl_sync(kFull, tl, (t + 3) & 31);
                }
                if (COUNT && live) nand += min(4u, m - (uint32_t)t);
                if (live) mw &= (ld_tok(col, tw.x, wb) & ld_tok(col, tw.y, wb)) & (ld_tok(col, tw.z, wb) & ld_tok(col, tw.w, wb));
            }
            for (uint32_t t = 32; t < m; ++t) {
                if (!__any_sync(kFull, mw != 0ull)) break;
                const uint32_t tt = toks[o + t];
                if (COUNT && mw) ++nand;
                if (mw) mw &= ld_tok(col, tt, wb);
            }
            if (MODE == kSupport) {
                cnt += __popcll(mw);
            } else if (MODE == kCover) {
                if (__any_sync(kFull, mw != 0ull)) {
                    hit = true;
                    break;
                }
            } else if (!COUNT) {
                if (__any_sync(kFull, mw != 0ull)) {
                    if (MODE == kMatch) {
                        // difference array: +s at each run start, -s after each run end
                        // every run has one start and one end: one loop retires both;
                        // ctz(x) = popc(~x & (x - 1)) avoids the 64-bit find-first sequence
                        // (each lane walks its own runs: dealing the runs over the
                        // whole warp measured 20 % slower)
                        unsigned long long st = mw & ~(mw << 1), en = mw & ~(mw >> 1);
                        unsigned long long* row = acc + (size_t)w * 64;
                        while (st) {
                            __builtin_assume(en != 0ull);
                            const unsigned long long st1 = st - 1, en1 = en - 1;
                            atomicAdd(row + __popcll(~st & st1), s);
                            atomicAdd(row + 1 + __popcll(~en & en1), 0ull - s);
                            st &= st1;
                            en &= en1;
                        }
                    } else {
                        warp_scatter_hits<true>(w, mw, s, acc, ovf);
                    }
                }
            }
        }
        if (COUNT) continue;
        if (MODE == kSupport) {
            for (int o2 = 16; o2; o2 >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o2);
            if (lane == 0) support_out[p] = (int64_t)cnt;
        } else if (MODE == kCover) {
            if (lane == 0) cover_out[p] = hit ? 1 : 0;
        }
    }
    if (COUNT) {
        for (int o2 = 16; o2; o2 >>= 1) nand += __shfl_xor_sync(kFull, nand, o2);
        if (lane == 0 && nand) atomicAdd(work, nand);
        return;
    }
    if (MODE == kMatchChecked && ovf) atomicOr(flags, 1);
}

// difference array of one mask: +s at each run start, -s after each run end
// (ctz(x) = popc(~x & (x - 1)) avoids the 64-bit find-first sequence)
__device__ __forceinline__ void scatter_runs(unsigned long long mw, unsigned long long s, unsigned long long* row) {
    unsigned long long st = mw & ~(mw << 1), en = mw & ~(mw >> 1);
    while (st) {
        __builtin_assume(en != 0ull);
        const unsigned long long st1 = st - 1, en1 = en - 1;
        atomicAdd(row + __popcll(~st & st1), s);
        atomicAdd(row + 1 + __popcll(~en & en1), 0ull - s);
        st &= st1;
        en &= en1;
    }
}

// Short lists (support and coverage at C3: 10-20 words per pattern; the
// matcher at C4: 20-22) leave half of a warp's lanes idle: a warp takes two
// neighbouring patterns, each on a half-warp, whenever both group lists fit 16
// words; otherwise it runs them one after the other on the full warp, as
// grouped_scan does, the pattern's tokens read from a per-warp shared-memory
// row (one 16-byte broadcast per four tokens).
template <int MODE, bool COUNT = false>
__global__ void __launch_bounds__(256)
half_scan(const unsigned long long* __restrict__ dense, size_t W, const uint32_t* __restrict__ tok_beg,
          const uint32_t* __restrict__ tok_len, const uint16_t* __restrict__ toks, size_t np,
          const uint32_t* __restrict__ order, const uint32_t* __restrict__ gid,
          const unsigned long long* __restrict__ goff, const uint32_t* __restrict__ glen,
          const uint32_t* __restrict__ ew, const unsigned long long* __restrict__ em,
          const int64_t* __restrict__ scores, unsigned long long* __restrict__ acc,
          int64_t* __restrict__ support_out, uint8_t* __restrict__ cover_out, unsigned long long* __restrict__ work,
          const uint32_t* __restrict__ sel) {
    static_assert(MODE == kSupport || MODE == kCover || MODE == kMatch, "half_scan: support, coverage or match");
    const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
    const unsigned hmask = half ? 0xffff0000u : 0x0000ffffu;
    const uint32_t Wu = (uint32_t)W, wb = Wu * 8u;
    // per warp and half: tokens 3..34 of the half's pattern (past it: token 0)
    __shared__ __align__(16) uint32_t s_tok[8][2][32];
    uint32_t(*st)[32] = s_tok[(threadIdx.x >> 5) & 7];
    const size_t warps = ((size_t)gridDim.x * blockDim.x) >> 5;
    const size_t npairs = (np + 1) / 2;
    unsigned long long nand = 0;
    for (size_t pi = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; pi < npairs; pi += warps) {
        const size_t ih0 = 2 * pi + (size_t)half;
        const bool has = ih0 < np;
        uint32_t p = 0, o = 0, m = 0, len = 0;
        unsigned long long base = 0, sc = 0;
        if (has) {
            const size_t ih = sel ? sel[ih0] : ih0;  // np positions: all, or the selected subset
            p = order[ih];
            const uint32_t g = gid[ih];
            o = tok_beg[p];
            m = tok_len[p];
            len = glen[g];
            base = goff[g];
            if (MODE == kMatch) sc = (unsigned long long)scores[p];
        }
        const uint32_t lenA = __shfl_sync(kFull, len, 0), lenB = __shfl_sync(kFull, len, 16);
        if (lenA <= 16 && lenB <= 16) {
            const uint32_t t0 = m ? (uint32_t)toks[o] : 0u;
            __syncwarp();  // the previous pair's tokens are read
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const uint32_t t = (uint32_t)hl + 16u * r;
                st[half][t >= 3 ? t - 3 : 29 + t] = (t < m && t >= 3) ? (uint32_t)toks[o + t] : t0;
            }
            __syncwarp();
            const uint32_t w = (uint32_t)hl < len ? ew[base + hl] : 0u;
            unsigned long long mw = (uint32_t)hl < len ? em[base + hl] : 0ull;
            const unsigned long long* col = dense + w;
            const uint32_t mmax = max(__shfl_sync(kFull, m, 0), __shfl_sync(kFull, m, 16));
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t t = 3u + 4u * q;
                if (t >= mmax) break;
                const bool live = mw != 0ull && t < m;
                if (!__any_sync(kFull, live)) break;
                const uint4 tw = reinterpret_cast<const uint4*>(st[half])[q];
                if (COUNT && live) nand += min(4u, m - t);
                if (live) mw &= (ld_tok(col, tw.x, wb) & ld_tok(col, tw.y, wb)) & (ld_tok(col, tw.z, wb) & ld_tok(col, tw.w, wb));
            }
            for (uint32_t t = 32; t < mmax; ++t) {  // rare tail
                const bool live = mw != 0ull && t < m;
                if (!__any_sync(kFull, live)) break;
                if (COUNT && live) ++nand;
                if (live) mw &= ld_tok(col, toks[o + t], wb);
            }
            if (COUNT) continue;
            if (MODE == kSupport) {
                uint32_t cnt = __popcll(mw);
                for (int o2 = 8; o2; o2 >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o2);
                if (hl == 0 && has) support_out[p] = (int64_t)cnt;
            } else if (MODE == kCover) {
                const unsigned hit = __ballot_sync(kFull, mw != 0ull) & hmask;
                if (hl == 0 && has) cover_out[p] = hit ? 1 : 0;
            } else if (mw) {
                scatter_runs(mw, sc, acc + (size_t)w * 64);
            }
            continue;
        }
        // full warp, one pattern after the other
        for (int h = 0; h < 2; ++h) {
            const size_t i = 2 * pi + (size_t)h;
            if (i >= np) break;
            const uint32_t pp = __shfl_sync(kFull, p, 16 * h), oo = __shfl_sync(kFull, o, 16 * h);
            const uint32_t mm = __shfl_sync(kFull, m, 16 * h), ll = h ? lenB : lenA;
            const unsigned long long bb = __shfl_sync(kFull, base, 16 * h);
            const unsigned long long ss = __shfl_sync(kFull, sc, 16 * h);
            const uint32_t t0 = mm ? (uint32_t)toks[oo] : 0u;
            const uint32_t tl = (uint32_t)lane < mm ? (uint32_t)toks[oo + lane] : t0;
            __syncwarp();  // the previous pattern's tokens are read
            st[0][lane >= 3 ? lane - 3 : 29 + lane] = lane >= 3 ? tl : t0;
            __syncwarp();
            uint32_t cnt = 0;
            bool hit = false;
            for (uint32_t j0 = 0; j0 < ll; j0 += 32) {
                const uint32_t j = j0 + lane;
                const uint32_t w = j < ll ? ew[bb + j] : 0u;
                unsigned long long mw = j < ll ? em[bb + j] : 0ull;
                const unsigned long long* col = dense + w;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int t = 3 + 4 * q;
                    if ((uint32_t)t >= mm) break;
                    const bool live = mw != 0ull;
                    if (!__any_sync(kFull, live)) break;
                    const uint4 tw = reinterpret_cast<const uint4*>(st[0])[q];
                    if (COUNT && live) nand += min(4u, mm - (uint32_t)t);
                    if (live) mw &= (ld_tok(col, tw.x, wb) & ld_tok(col, tw.y, wb)) & (ld_tok(col, tw.z, wb) & ld_tok(col, tw.w, wb));
                }
                for (uint32_t t = 32; t < mm; ++t) {
                    if (!__any_sync(kFull, mw != 0ull)) break;
                    if (COUNT && mw) ++nand;
                    if (mw) mw &= ld_tok(col, toks[oo + t], wb);
                }
                if (MODE == kSupport) {
                    cnt += __popcll(mw);
                } else if (MODE == kCover) {
                    if (__any_sync(kFull, mw != 0ull)) {
                        hit = true;
                        break;
                    }
                } else if (!COUNT && mw) {
                    scatter_runs(mw, ss, acc + (size_t)w * 64);
                }
            }
            if (COUNT) continue;
            if (MODE == kSupport) {
                for (int o2 = 16; o2; o2 >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o2);
                if (lane == 0) support_out[pp] = (int64_t)cnt;
            } else if (MODE == kCover && lane == 0) {
                cover_out[pp] = hit ? 1 : 0;
            }
        }
    }
    if (COUNT) {
        for (int o2 = 16; o2; o2 >>= 1) nand += __shfl_xor_sync(kFull, nand, o2);
        if (lane == 0 && nand) atomicAdd(work, nand);
    }
}

// IG_SCAN_STATS=1 (development): shape of one scan on stderr — patterns per
// group, list words per pattern (lane occupancy of a warp per pattern), tokens
// per pattern.
void scan_stats(Ctx& ctx, int mode, const PatternIndex& I, const DevBuf& glen, size_t G, size_t np) {
    std::vector<uint32_t> gl(G), gid(np), len(np), order(np);
    read_back(ctx, gl.data(), glen.p, G * 4);
    read_back(ctx, gid.data(), I.gid.p, np * 4);
    read_back(ctx, len.data(), I.len.p, np * 4);
    read_back(ctx, order.data(), I.order.p, np * 4);
    std::vector<uint64_t> pg(G, 0);
    uint64_t words = 0, rounds = 0, hist[8] = {0, 0, 0, 0, 0, 0, 0, 0}, toks = 0;
    for (size_t i = 0; i < np; ++i) {
        const uint32_t l = gl[gid[i]];
        ++pg[gid[i]];
        words += l;
        rounds += (l + 31) / 32;
        int b = 0;
        while (b < 7 && (1u << (b + 1)) <= l) ++b;  // bucket: [2^b, 2^(b+1)), last = >= 128
        ++hist[l == 0 ? 0 : std::min(b + 1, 7)];
        toks += len[order[i]];
    }
    {
        // staging estimate: words a group-shared SMEM tile of every token of the
        // group (tokens 3..) would load, against the dense per-pattern ANDs
        std::vector<uint32_t> beg(np);
        read_back(ctx, beg.data(), I.beg.p, np * 4);
        uint32_t tmax = 0;
        for (size_t p = 0; p < np; ++p) tmax = std::max(tmax, beg[p] + len[p]);
        std::vector<uint16_t> toks(tmax);
        read_back(ctx, toks.data(), I.toks->p, (size_t)tmax * 2);
        {
            // per task (<= 64 patterns of one group of >= 4): tokens common to
            // all its patterns (ANDed once per task), residual tokens per pattern
            std::vector<uint32_t> cntt(65536, 0);
            uint64_t base_ands = 0, resid_ands = 0, resid_union = 0, small_ands = 0, ntask = 0, csum = 0;
            size_t i = 0;
            while (i < np) {
                size_t e = i;
                while (e < np && gid[e] == gid[i]) ++e;
                const uint32_t g = gid[i];
                if (e - i < 4) {
                    for (size_t j = i; j < e; ++j) {
                        const uint32_t p = order[j];
                        small_ands += (uint64_t)(len[p] > 3 ? len[p] - 3 : 0) * gl[g];
                    }
                    i = e;
                    continue;
                }
                for (size_t t0 = i; t0 < e; t0 += 64) {
                    const size_t t1 = std::min(e, t0 + 64), n = t1 - t0;
                    std::vector<uint16_t> used;
                    for (size_t j = t0; j < t1; ++j) {
                        const uint32_t p = order[j];
                        for (uint32_t t = 3; t < len[p]; ++t) {
                            const uint16_t tk = toks[beg[p] + t];
                            if (cntt[tk]++ == 0) used.push_back(tk);
                        }
                    }
                    uint32_t c = 0, ru = 0;
                    for (uint16_t tk : used) {
                        if (cntt[tk] == n)
                            ++c;
                        else
                            ++ru;
                    }
                    for (size_t j = t0; j < t1; ++j) {
                        const uint32_t p = order[j];
                        const uint32_t m3 = len[p] > 3 ? len[p] - 3 : 0;
                        resid_ands += (uint64_t)(m3 - c) * gl[g];
                    }
                    for (uint16_t tk : used) cntt[tk] = 0;
                    base_ands += (uint64_t)c * gl[g];
                    resid_union += (uint64_t)ru * gl[g];
                    csum += c;
                    ++ntask;
                }
                i = e;
            }
            fprintf(stderr,
                    "[ig scan] mode %d tasks %llu: common tokens/task %.1f, base ANDs %.3g, residual ANDs %.3g (dense), "
                    "residual rows staged %.3g, small-group ANDs %.3g (dense)\n",
                    mode, (unsigned long long)ntask, ntask ? (double)csum / ntask : 0.0, (double)base_ands,
                    (double)resid_ands, (double)resid_union, (double)small_ands);
        }
        std::vector<uint32_t> seen(65536, 0xffffffffu);
        uint64_t staged = 0, dense_ands = 0, ucnt = 0, uhist[6] = {0, 0, 0, 0, 0, 0};
        size_t i = 0;
        while (i < np) {
            const uint32_t g = gid[i];
            uint32_t u = 0;
            size_t j = i;
            for (; j < np && gid[j] == g; ++j) {
                const uint32_t p = order[j];
                for (uint32_t t = 3; t < len[p]; ++t) {
                    const uint16_t tk = toks[beg[p] + t];
                    if (seen[tk] != g) {
                        seen[tk] = g;
                        ++u;
                    }
                }
                dense_ands += (uint64_t)(len[p] > 3 ? len[p] - 3 : 0) * gl[g];
            }
            staged += (uint64_t)u * gl[g];
            ucnt += u;
            uhist[u <= 16 ? 0 : u <= 32 ? 1 : u <= 64 ? 2 : u <= 128 ? 3 : u <= 256 ? 4 : 5] += j - i;
            i = j;
        }
        fprintf(stderr,
                "[ig scan] mode %d staging: union tokens/group %.1f, staged words %.3g vs dense pattern ANDs %.3g "
                "(x%.2f) | patterns in groups with union <=16:%llu <=32:%llu <=64:%llu <=128:%llu <=256:%llu "
                ">256:%llu\n",
                mode, (double)ucnt / G, (double)staged, (double)dense_ands,
                staged ? (double)dense_ands / staged : 0.0, (unsigned long long)uhist[0],
                (unsigned long long)uhist[1], (unsigned long long)uhist[2], (unsigned long long)uhist[3],
                (unsigned long long)uhist[4], (unsigned long long)uhist[5]);
    }
    uint64_t pgh[6] = {0, 0, 0, 0, 0, 0};
    for (size_t g = 0; g < G; ++g) {
        const uint64_t c = pg[g];
        pgh[c <= 1 ? 0 : c <= 4 ? 1 : c <= 16 ? 2 : c <= 64 ? 3 : c <= 256 ? 4 : 5] += c;
    }
    fprintf(stderr,
            "[ig scan] mode %d np %zu G %zu G2 %zu W %s | list words/pattern %.2f, lane occupancy %.3f | patterns "
            "with list len 0:%llu 1:%llu 2-3:%llu 4-7:%llu 8-15:%llu 16-31:%llu 32-63:%llu >=64:%llu | patterns in "
            "groups of <=1:%llu <=4:%llu <=16:%llu <=64:%llu <=256:%llu >256:%llu | tokens/pattern %.2f\n",
            mode, np, G, I.G2, "-", (double)words / np, rounds ? (double)words / (32.0 * rounds) : 0.0,
            (unsigned long long)hist[0], (unsigned long long)hist[1], (unsigned long long)hist[2],
            (unsigned long long)hist[3], (unsigned long long)hist[4], (unsigned long long)hist[5],
            (unsigned long long)hist[6], (unsigned long long)hist[7], (unsigned long long)pgh[0],
            (unsigned long long)pgh[1], (unsigned long long)pgh[2], (unsigned long long)pgh[3],
            (unsigned long long)pgh[4], (unsigned long long)pgh[5], (double)toks / np);
}

constexpr unsigned long long kListBudget = 3ull << 30;  // bytes of scan lists allocated from bounds
#ifndef IG_HALF_MATCH_MAX_W
#define IG_HALF_MATCH_MAX_W 1024
#endif
constexpr size_t kHalfMatchMaxW = IG_HALF_MATCH_MAX_W;  // the matcher pairs short lists when W <= this

template <int MODE>
void launch_scan(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, const PatternIndex* I,
                 const int64_t* scores, unsigned long long* acc, int64_t* support, uint8_t* cover, int* flags) {
    if (np == 0) return;
    Trace tr(ctx, MODE == kSupport ? "scan:support" : MODE == kCover ? "scan:cover" : "scan:match", -1);
    PatternIndex local;
    if (!I) {  // no shared index: rank the tokens by this postings' document frequency
        RankSpace R;
        make_rank_space(ctx, P.df.as<uint32_t>(), P.L, R);
        build_pattern_index(ctx, d_pat, np, k, R, local);
        I = &local;
        tr.mark("pattern_index");
    }
    const uint32_t* sel = I->sel.p ? I->sel.as<uint32_t>() : nullptr;
    if ((sel ? I->nsel : I->np) != np) fail(IG_E_CUDA, "pattern index does not match the pattern set");
    const size_t G = I->G, G2 = I->G2;
    // parent (t1, t2) lists S2 = non-zero (w, post[t1][w] & post[t2][w]) in P,
    // then each (t1, t2, t3) group's list S = S2 filtered by post[t3]
    // Both list levels are sized before either is built, with one read-back:
    // a parent list holds at most nnz(post[t1]) words (its upper bound), and a
    // child list at most its parent's bound.
    DevBuf ub((G2 + 1) * 8, ctx.stream), poff((G2 + 1) * 8, ctx.stream), plen(G2 * 4 + 4, ctx.stream);
    DevBuf ub3((G + 1) * 8, ctx.stream), goff((G + 1) * 8, ctx.stream), glen(G * 4 + 4, ctx.stream);
    if (G2)
        IGB_LAUNCH(ctx, group_bound, grid_for(ctx, G2, 256), 256, 0, I->pkey.as<uint32_t>(), G2,
                   P.nz_off.as<uint32_t>(), P.W, ub.as<unsigned long long>());
    IGB_CUDA(cudaMemsetAsync(ub.as<unsigned long long>() + G2, 0, 8, ctx.stream));
    if (G)
        IGB_LAUNCH(ctx, child_bound, grid_for(ctx, G, 256), 256, 0, I->pid.as<uint32_t>(), G, ub.as<unsigned long long>(),
                   ub3.as<unsigned long long>());
    IGB_CUDA(cudaMemsetAsync(ub3.as<unsigned long long>() + G, 0, 8, ctx.stream));
    size_t tb4 = 0;
    IGB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb4, ub.as<unsigned long long>(), poff.as<unsigned long long>(),
                                           (int64_t)std::max(G, G2) + 1, ctx.stream));
    DevBuf temp4(tb4, ctx.stream);
    IGB_CUDA(cub::DeviceScan::ExclusiveSum(temp4.p, tb4, ub.as<unsigned long long>(), poff.as<unsigned long long>(),
                                           (int64_t)G2 + 1, ctx.stream));
    IGB_CUDA(cub::DeviceScan::ExclusiveSum(temp4.p, tb4, ub3.as<unsigned long long>(), goff.as<unsigned long long>(),
                                           (int64_t)G + 1, ctx.stream));
    // Every list is at most W words long, so G2·W and G·W entries bound both
    // levels: when that fits kListBudget, allocate the bound (the pool keeps
    // the pages mapped; only the written entries are touched) and skip the
    // read-back of the exact sizes — one host round trip less per scan.
    const unsigned long long Wl = std::max<unsigned long long>(P.W, 1);
    unsigned long long E2E[2] = {(unsigned long long)G2 * Wl, (unsigned long long)G * Wl};
    static const bool exact_sizes = getenv("IG_SCAN_EXACT_SIZES") != nullptr;  // A/B
    if (exact_sizes || (E2E[0] + E2E[1]) * 12 > kListBudget) {
        DevBuf both(16, ctx.stream);
        IGB_CUDA(cudaMemcpyAsync(both.p, poff.as<unsigned long long>() + G2, 8, cudaMemcpyDeviceToDevice, ctx.stream));
        IGB_CUDA(cudaMemcpyAsync(both.as<unsigned long long>() + 1, goff.as<unsigned long long>() + G, 8,
                                 cudaMemcpyDeviceToDevice, ctx.stream));
        read_back(ctx, E2E, both.p, 16);
    }
    const unsigned long long E2 = E2E[0], E = E2E[1];
    DevBuf pw(std::max<unsigned long long>(E2, 1) * 4, ctx.stream), pm(std::max<unsigned long long>(E2, 1) * 8, ctx.stream);
    if (G2)
        IGB_LAUNCH(ctx, group_lists, grid_for(ctx, G2 * 32, 256), 256, 0, I->pkey.as<uint32_t>(), G2,
                   P.dense.as<unsigned long long>(), P.W, P.n, P.nz_off.as<uint32_t>(), P.nz_idx.as<uint32_t>(),
                   poff.as<unsigned long long>(), plen.as<uint32_t>(), pw.as<uint32_t>(), pm.as<unsigned long long>());
    DevBuf ew(std::max<unsigned long long>(E, 1) * 4, ctx.stream), em(std::max<unsigned long long>(E, 1) * 8, ctx.stream);
    if (G)
        IGB_LAUNCH(ctx, child_lists, grid_for(ctx, G * 32, 256), 256, 0, I->gkey.as<unsigned long long>(),
                   I->pid.as<uint32_t>(), G, P.dense.as<unsigned long long>(), P.W, poff.as<unsigned long long>(),
                   plen.as<uint32_t>(), pw.as<uint32_t>(), pm.as<unsigned long long>(), goff.as<unsigned long long>(),
                   glen.as<uint32_t>(), ew.as<uint32_t>(), em.as<unsigned long long>());
    tr.mark("group_lists");
    if (getenv("IG_SCAN_STATS")) scan_stats(ctx, MODE, *I, glen, G, np);
    const size_t blocks = std::min<size_t>((np + 7) / 8, (size_t)ctx.sm_count * 64);
    DiagSpan dspan(ctx, MODE == kSupport ? kDiagSupport : MODE == kCover ? kDiagCover : kDiagMatch);
    static const int half_env = getenv("IG_HALF_SCAN") ? atoi(getenv("IG_HALF_SCAN")) : 1;  // A/B
    auto launch = [&](auto count_tag, unsigned long long* work) {
        constexpr bool C = decltype(count_tag)::value;
        if constexpr (MODE == kSupport || MODE == kCover || MODE == kMatch) {
            // (the matcher: only where its lists are short — the test
            // postings' width bounds every list; C3's 1,513-word postings give
            // 80-90-word matcher lists, C4's 464-word ones 20-22)
            if (half_env && (MODE != kMatch || P.W <= kHalfMatchMaxW)) {
                const size_t hblocks = std::min<size_t>((np + 15) / 16, (size_t)ctx.sm_count * 64);
                IGB_LAUNCH(ctx, (half_scan<MODE, C>), (unsigned)hblocks, 256, 0, P.dense.as<unsigned long long>(), P.W,
                           I->beg.as<uint32_t>(), I->len.as<uint32_t>(), I->toks->as<uint16_t>(), np,
                           I->order.as<uint32_t>(), I->gid.as<uint32_t>(), goff.as<unsigned long long>(),
                           glen.as<uint32_t>(), ew.as<uint32_t>(), em.as<unsigned long long>(), scores, acc, support,
                           cover, work, sel);
                return;
            }
        }
        IGB_LAUNCH(ctx, (grouped_scan<MODE, C>), (unsigned)blocks, 256, 0, P.dense.as<unsigned long long>(), P.W,
                   P.n, I->beg.as<uint32_t>(), I->len.as<uint32_t>(), I->toks->as<uint16_t>(), np,
                   I->order.as<uint32_t>(), I->gid.as<uint32_t>(), goff.as<unsigned long long>(),
                   glen.as<uint32_t>(), ew.as<uint32_t>(), em.as<unsigned long long>(), scores, acc, support,
                   cover, flags, work, sel);
    };
    launch(std::false_type{}, nullptr);
    tr.mark("grouped_scan");
    if (ctx.diag) {
        // the same launch again with outputs suppressed, counting its word-ANDs
        dspan.stop();
        DevBuf w(8, ctx.stream);
        IGB_CUDA(cudaMemsetAsync(w.p, 0, 8, ctx.stream));
        launch(std::true_type{}, w.as<unsigned long long>());
        unsigned long long hw = 0;
        read_back(ctx, &hw, w.p, 8);
        dspan.end(hw);
    }
}

}  // namespace

// ------------------------------------------------------------------ pattern index
void make_rank_space(Ctx& ctx, const uint32_t* d_df, uint32_t L, RankSpace& R, bool descending) {
    R.L = L;
    R.df.alloc((size_t)L * 4, ctx.stream);
    IGB_CUDA(cudaMemcpyAsync(R.df.p, d_df, (size_t)L * 4, cudaMemcpyDeviceToDevice, ctx.stream));
    R.rank.alloc((size_t)L * 2, ctx.stream);
    R.byrank.alloc((size_t)L * 2, ctx.stream);
    if (L <= kRankCount) {
        IGB_LAUNCH(ctx, rank_by_key_count, (L + 255) / 256, 256, 0, d_df, L, descending, R.rank.as<uint16_t>(),
                   R.byrank.as<uint16_t>());
        return;
    }
    DevBuf key((size_t)L * 8, ctx.stream), key2((size_t)L * 8, ctx.stream), tok((size_t)L * 2, ctx.stream);
    IGB_LAUNCH(ctx, rank_keys, grid_for(ctx, L, 256), 256, 0, d_df, L, key.as<unsigned long long>(),
               tok.as<uint16_t>(), descending);
    size_t tb = 0;
    IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<unsigned long long>(), key2.as<unsigned long long>(),
                                             tok.as<uint16_t>(), R.byrank.as<uint16_t>(), (int64_t)L, 0, 64, ctx.stream));
    DevBuf temp(tb, ctx.stream);
    IGB_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, tb, key.as<unsigned long long>(), key2.as<unsigned long long>(),
                                             tok.as<uint16_t>(), R.byrank.as<uint16_t>(), (int64_t)L, 0, 64, ctx.stream));
    IGB_LAUNCH(ctx, invert_rank, grid_for(ctx, L, 256), 256, 0, R.byrank.as<uint16_t>(), L, R.rank.as<uint16_t>());
}

void combined_rank_space(Ctx& ctx, const Postings& A, const Postings& B, RankSpace& R) {
    if (A.L != B.L) fail(IG_E_CUDA, "combined_rank_space: postings of different widths");
    DevBuf df((size_t)A.L * 4, ctx.stream);
    IGB_LAUNCH(ctx, add_u32, grid_for(ctx, A.L, 256), 256, 0, A.df.as<uint32_t>(), B.df.as<uint32_t>(), A.L,
               df.as<uint32_t>());
    make_rank_space(ctx, df.as<uint32_t>(), A.L, R);
}

void build_pattern_index(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const RankSpace& R, PatternIndex& I,
                         uint32_t max_tokens) {
    Trace tr(ctx, "pattern_index", -1);
    I.np = np;
    I.G = 0;
    I.beg.alloc((np + 1) * 4, ctx.stream);  // CSR offsets (np + 1)
    I.len.alloc((np + 1) * 4, ctx.stream);
    I.order.alloc(std::max<size_t>(np, 1) * 4, ctx.stream);
    I.gid.alloc(std::max<size_t>(np, 1) * 4, ctx.stream);
    I.gkey.alloc(std::max<size_t>(np, 1) * 8, ctx.stream);
    // CSR token lists, rarest first in R
    if (np)
        IGB_LAUNCH(ctx, pattern_token_count, grid_for(ctx, np, 256), 256, 0, d_pat, np, (int)k, I.len.as<uint32_t>());
    IGB_CUDA(cudaMemsetAsync(I.len.as<uint32_t>() + np, 0, 4, ctx.stream));
    size_t tb = 0;
    IGB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, I.len.as<uint32_t>(), I.beg.as<uint32_t>(), (int64_t)np + 1,
                                           ctx.stream));
    DevBuf temp(tb, ctx.stream);
    IGB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, I.len.as<uint32_t>(), I.beg.as<uint32_t>(), (int64_t)np + 1,
                                           ctx.stream));
    // token list space: np * max_tokens when the caller bounds a pattern's
    // tokens (no read-back), else the exact total
    uint64_t total = (uint64_t)np * std::min<uint32_t>(max_tokens, (uint32_t)(64 * k));
    if (!max_tokens || total > 0xffffffffull) {
        uint32_t t32 = 0;
        read_back(ctx, &t32, I.beg.as<uint32_t>() + np, 4);
        total = t32;
    }
    I.toks = std::make_shared<DevBuf>();
    I.toks->alloc(std::max<size_t>(total, 1) * 2, ctx.stream);
    if (np == 0) return;
    const uint32_t L = R.L;
    if (k <= kRankWords) {
#define IGB_FILL_RANK(KW)                                                                                          \
    {                                                                                                              \
        const size_t smem = (size_t)L * 4 + (size_t)2 * KW * kFillThreads * 4;                                    \
        if (smem > 48 * 1024)                                                                                      \
            IGB_SMEM_ATTR(ctx, pattern_token_fill_rank<KW>, (int)smem);                                           \
        IGB_LAUNCH(ctx, pattern_token_fill_rank<KW>, grid_for(ctx, np, kFillThreads), kFillThreads, smem, d_pat,   \
                   np, (int)k,                                                                                     \
                   R.rank.as<uint16_t>(), R.byrank.as<uint16_t>(), L, I.beg.as<uint32_t>(), I.toks->as<uint16_t>()); \
    }
        if (k <= 16)
            IGB_FILL_RANK(16)
        else if (k <= 32)
            IGB_FILL_RANK(32)
        else
            IGB_FILL_RANK(64)
#undef IGB_FILL_RANK
    } else {
        const size_t smem = (size_t)L * 4;
        if (smem > 48 * 1024)
            IGB_SMEM_ATTR(ctx, pattern_token_fill, smem);
        IGB_LAUNCH(ctx, pattern_token_fill, grid_for(ctx, np, 128), 128, smem, d_pat, np, (int)k,
                   R.df.as<uint32_t>(), L, I.beg.as<uint32_t>(), I.toks->as<uint16_t>());
    }
    tr.mark("token_lists");
    // group patterns by their three rarest tokens
    int b = 1;
    while ((1u << b) <= L) ++b;  // token ids < L < 2^b - 1 stays free for "absent"
    // tokens in the sort key: the group (t1, t2, t3).  Sorting further tokens
    // (neighbours sharing prefixes) only served the prefix-sharing scans that
    // were measured slower and costs radix passes.
    const int q = 3;
    DevBuf key(np * 8, ctx.stream), key2(np * 8, ctx.stream), idx(np * 4, ctx.stream);
    IGB_LAUNCH(ctx, group_keys, grid_for(ctx, np, 256), 256, 0, I.beg.as<uint32_t>(), I.len.as<uint32_t>(),
               I.toks->as<uint16_t>(), np, b, q, key.as<unsigned long long>(), idx.as<uint32_t>());
    size_t tb1 = 0;
    IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb1, key.as<unsigned long long>(), key2.as<unsigned long long>(),
                                             idx.as<uint32_t>(), I.order.as<uint32_t>(), (int64_t)np, 0, q * b,
                                             ctx.stream));
    DevBuf temp1(tb1, ctx.stream);
    IGB_CUDA(cub::DeviceRadixSort::SortPairs(temp1.p, tb1, key.as<unsigned long long>(), key2.as<unsigned long long>(),
                                             idx.as<uint32_t>(), I.order.as<uint32_t>(), (int64_t)np, 0, q * b,
                                             ctx.stream));
    IGB_LAUNCH(ctx, expand_keys, grid_for(ctx, np, 256), 256, 0, key2.as<unsigned long long>(), np, b, q);
    group_ids(ctx, key2.as<unsigned long long>(), np, I);
    tr.mark("group_sort");
}

// gid (0-based, per sorted position) and gkey (per group) from the sorted keys,
// then the (t1, t2) parent of every group (pid, pkey)
void group_ids(Ctx& ctx, const unsigned long long* d_sorted_key, size_t np, PatternIndex& I) {
    DevBuf head(np, ctx.stream), head32(np * 4, ctx.stream), nsel(8, ctx.stream);
    IGB_LAUNCH(ctx, group_heads<unsigned long long>, grid_for(ctx, np, 256), 256, 0, d_sorted_key, np,
               head.as<uint8_t>(), head32.as<uint32_t>());
    size_t tb2 = 0, tb3 = 0;
    IGB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb2, head32.as<uint32_t>(), I.gid.as<uint32_t>(), (int64_t)np,
                                           ctx.stream));
    IGB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb3, d_sorted_key, head.as<uint8_t>(),
                                        I.gkey.as<unsigned long long>(), nsel.as<int64_t>(), (int64_t)np, ctx.stream));
    DevBuf temp2(std::max(tb2, tb3), ctx.stream);
    IGB_CUDA(cub::DeviceScan::InclusiveSum(temp2.p, tb2, head32.as<uint32_t>(), I.gid.as<uint32_t>(), (int64_t)np,
                                           ctx.stream));
    IGB_CUDA(cub::DeviceSelect::Flagged(temp2.p, tb3, d_sorted_key, head.as<uint8_t>(),
                                        I.gkey.as<unsigned long long>(), nsel.as<int64_t>(), (int64_t)np, ctx.stream));
    IGB_LAUNCH(ctx, minus_one, grid_for(ctx, np, 256), 256, 0, I.gid.as<uint32_t>(), np);
    int64_t G = 0;
    read_back(ctx, &G, nsel.p, 8);
    I.G = (size_t)G;
    // parents: the groups are sorted by (t1, t2, t3), so equal (t1, t2) are adjacent
    const size_t Gs = std::max<size_t>(I.G, 1);
    I.pid.alloc(Gs * 4, ctx.stream);
    I.pkey.alloc(Gs * 4, ctx.stream);
    I.G2 = 0;
    if (!G) return;
    DevBuf pk(Gs * 4, ctx.stream), ph(Gs, ctx.stream), ph32(Gs * 4, ctx.stream);
    IGB_LAUNCH(ctx, parent_keys, grid_for(ctx, I.G, 256), 256, 0, I.gkey.as<unsigned long long>(), I.G,
               pk.as<uint32_t>());
    IGB_LAUNCH(ctx, group_heads<uint32_t>, grid_for(ctx, I.G, 256), 256, 0, pk.as<uint32_t>(), I.G, ph.as<uint8_t>(),
               ph32.as<uint32_t>());
    size_t tb4 = 0, tb5 = 0;
    IGB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb4, ph32.as<uint32_t>(), I.pid.as<uint32_t>(), (int64_t)I.G,
                                           ctx.stream));
    IGB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb5, pk.as<uint32_t>(), ph.as<uint8_t>(), I.pkey.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)I.G, ctx.stream));
    DevBuf temp3(std::max(tb4, tb5), ctx.stream);
    IGB_CUDA(cub::DeviceScan::InclusiveSum(temp3.p, tb4, ph32.as<uint32_t>(), I.pid.as<uint32_t>(), (int64_t)I.G,
                                           ctx.stream));
    IGB_CUDA(cub::DeviceSelect::Flagged(temp3.p, tb5, pk.as<uint32_t>(), ph.as<uint8_t>(), I.pkey.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)I.G, ctx.stream));
    IGB_LAUNCH(ctx, minus_one, grid_for(ctx, I.G, 256), 256, 0, I.pid.as<uint32_t>(), I.G);
    int64_t G2 = 0;
    read_back(ctx, &G2, nsel.p, 8);
    I.G2 = (size_t)G2;
}

void subset_pattern_index(Ctx& ctx, const PatternIndex& S, const uint32_t* d_src_of, size_t n, PatternIndex& I) {
    Trace tr(ctx, "subset_index", -1);
    I.np = n;
    I.G = 0;
    I.beg.alloc(std::max<size_t>(n, 1) * 4, ctx.stream);
    I.len.alloc(std::max<size_t>(n, 1) * 4, ctx.stream);
    I.order.alloc(std::max<size_t>(n, 1) * 4, ctx.stream);
    I.gid.alloc(std::max<size_t>(n, 1) * 4, ctx.stream);
    I.gkey.alloc(std::max<size_t>(n, 1) * 8, ctx.stream);
    I.toks = S.toks;  // token lists are shared with the source index, not copied
    if (n == 0) return;
    IGB_LAUNCH(ctx, sub_lists, grid_for(ctx, n, 256), 256, 0, S.beg.as<uint32_t>(), S.len.as<uint32_t>(), d_src_of, n,
               I.beg.as<uint32_t>(), I.len.as<uint32_t>());
    tr.mark("token_lists");
    // the source's group order restricted to the subset keeps its key order
    const size_t ns = S.np;
    DevBuf inv(ns * 4, ctx.stream), val(ns * 4, ctx.stream), og(ns * 4, ctx.stream), keep(ns, ctx.stream),
        og2(std::max<size_t>(n, 1) * 4, ctx.stream), key(std::max<size_t>(n, 1) * 8, ctx.stream), nsel(8, ctx.stream);
    IGB_LAUNCH(ctx, fill_u32, grid_for(ctx, ns, 256), 256, 0, inv.as<uint32_t>(), ns, 0xffffffffu);
    IGB_LAUNCH(ctx, scatter_pos, grid_for(ctx, n, 256), 256, 0, d_src_of, n, inv.as<uint32_t>());
    IGB_LAUNCH(ctx, map_order, grid_for(ctx, ns, 256), 256, 0, S.order.as<uint32_t>(), S.gid.as<uint32_t>(), ns,
               inv.as<uint32_t>(), val.as<uint32_t>(), og.as<uint32_t>(), keep.as<uint8_t>());
    size_t tb1 = 0;
    IGB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb1, val.as<uint32_t>(), keep.as<uint8_t>(), I.order.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)ns, ctx.stream));
    DevBuf temp1(tb1, ctx.stream);
    IGB_CUDA(cub::DeviceSelect::Flagged(temp1.p, tb1, val.as<uint32_t>(), keep.as<uint8_t>(), I.order.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)ns, ctx.stream));
    IGB_CUDA(cub::DeviceSelect::Flagged(temp1.p, tb1, og.as<uint32_t>(), keep.as<uint8_t>(), og2.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)ns, ctx.stream));
    // group key of every kept position = the source group's key
    IGB_LAUNCH(ctx, gather_u64k, grid_for(ctx, n, 256), 256, 0, S.gkey.as<unsigned long long>(), og2.as<uint32_t>(), n,
               key.as<unsigned long long>());
    group_ids(ctx, key.as<unsigned long long>(), n, I);
    tr.mark("groups");
}

namespace {
__global__ void position_keep(const uint32_t* __restrict__ order, size_t n, const uint8_t* __restrict__ flag,
                              uint8_t* __restrict__ keep, uint32_t* __restrict__ pos) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        keep[i] = flag[order[i]] ? 0 : 1;
        pos[i] = (uint32_t)i;
    }
}
}  // namespace

size_t select_unflagged_positions(Ctx& ctx, PatternIndex& I, const uint8_t* d_flag, size_t count) {
    const size_t n = I.np;
    I.sel.alloc(std::max<size_t>(n, 1) * 4, ctx.stream);
    I.nsel = 0;
    if (n == 0) return 0;
    DevBuf keep(n, ctx.stream), pos(n * 4, ctx.stream), nsel(8, ctx.stream);
    IGB_LAUNCH(ctx, position_keep, grid_for(ctx, n, 256), 256, 0, I.order.as<uint32_t>(), n, d_flag,
               keep.as<uint8_t>(), pos.as<uint32_t>());
    size_t tb = 0;
    IGB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, pos.as<uint32_t>(), keep.as<uint8_t>(), I.sel.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)n, ctx.stream));
    DevBuf temp(tb, ctx.stream);
    IGB_CUDA(cub::DeviceSelect::Flagged(temp.p, tb, pos.as<uint32_t>(), keep.as<uint8_t>(), I.sel.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)n, ctx.stream));
    I.nsel = count;  // (the caller's compaction of the same flags counted them)
    return I.nsel;
}

namespace {
// token document frequencies straight from packed rows (block histogram in smem)
__global__ void row_token_df(const int64_t* __restrict__ rows, size_t n, int k, uint32_t* __restrict__ df) {
    extern __shared__ uint32_t h[];
    const int L = 64 * k;
    for (int t = threadIdx.x; t < L; t += blockDim.x) h[t] = 0;
    __syncthreads();
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n * (size_t)k; q += (size_t)gridDim.x * blockDim.x) {
        uint64_t x = (uint64_t)rows[q];
        const int w = (int)(q % k);
        while (x) {
            atomicAdd(h + w * 64 + (__ffsll((long long)x) - 1), 1u);
            x &= x - 1;
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < L; t += blockDim.x)
        if (h[t]) atomicAdd(df + t, h[t]);
}

// rows re-spelled with token t at sort position pos[t] (MSB-first per word)
__global__ void permute_row_bits(const int64_t* __restrict__ rows, size_t n, int k, const uint16_t* __restrict__ pos,
                                 int64_t* __restrict__ out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        for (int w = 0; w < k; ++w) out[i * k + w] = 0;
        for (int w = 0; w < k; ++w) {
            uint64_t x = (uint64_t)rows[i * k + w];
            while (x) {
                const int b = __ffsll((long long)x) - 1;
                x &= x - 1;
                const uint32_t r = pos[w * 64 + b];
                out[i * k + (r >> 6)] |= (int64_t)(1ull << (63 - (r & 63)));
            }
        }
    }
}
// reflected-Gray rank of a MSB-first bit vector: b = prefix XOR of g
__global__ void gray_to_binary(int64_t* __restrict__ rows, size_t n, int k) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint64_t carry = 0;  // parity of all earlier bits, as 0 or ~0
        for (int w = 0; w < k; ++w) {
            uint64_t x = (uint64_t)rows[i * k + w];
            x ^= x >> 1;
            x ^= x >> 2;
            x ^= x >> 4;
            x ^= x >> 8;
            x ^= x >> 16;
            x ^= x >> 32;
            x ^= carry;
            rows[i * k + w] = (int64_t)x;
            carry = (x & 1ull) ? ~0ull : 0ull;
        }
    }
}
}  // namespace

void cluster_order(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, uint32_t* d_perm) {
    const uint32_t L = (uint32_t)(64 * k);
    if (n < 2 || (size_t)L * 4 > (size_t)ctx.smem_optin) {
        sort_rows_canonical(ctx, d_rows, n, k, d_perm);
        return;
    }
    if ((size_t)L * 4 > 48 * 1024)
        IGB_SMEM_ATTR(ctx, row_token_df, (int)L * 4);
    DevBuf df((size_t)L * 4, ctx.stream), prow(n * k * 8, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(df.p, 0, (size_t)L * 4, ctx.stream));
    IGB_LAUNCH(ctx, row_token_df, std::max(1, ctx.sm_count * 2), 256, (size_t)L * 4, d_rows, n, (int)k,
               df.as<uint32_t>());
    RankSpace R;
    make_rank_space(ctx, df.as<uint32_t>(), L, R, true);
    IGB_LAUNCH(ctx, permute_row_bits, grid_for(ctx, n, 256), 256, 0, d_rows, n, (int)k, R.rank.as<uint16_t>(),
               prow.as<int64_t>());
    IGB_LAUNCH(ctx, gray_to_binary, grid_for(ctx, n, 256), 256, 0, prow.as<int64_t>(), n, (int)k);
    sort_rows_canonical(ctx, prow.as<int64_t>(), n, k, d_perm);
}

bool postings_supported(uint32_t L, size_t n) {
    // token ids fit u16, and every posting's word offset (token * W) fits u32
    return words_for(L) * 64 < 65535 && n < 0xffffffffull &&
           (uint64_t)words_for(L) * 64 * ((n + 63) / 64) < 0xffffffffull;
}

void build_postings(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, uint32_t /*logical_len*/, Postings& P,
                    bool canonical, bool distinct, const uint32_t* d_perm) {
    const uint32_t L = (uint32_t)(64 * k);  // every bit position, padding included
    P.L = L;
    P.n_src = n;
    P.perm.release();
    P.group.release();
    P.rep.release();
    if ((canonical || distinct) && n > 1) {
        P.perm.alloc(n * 4, ctx.stream);
        if (d_perm)
            IGB_CUDA(cudaMemcpyAsync(P.perm.p, d_perm, n * 4, cudaMemcpyDeviceToDevice, ctx.stream));
        else
            cluster_order(ctx, d_rows, n, k, P.perm.as<uint32_t>());
    }
    size_t nd = n;
    const uint32_t* rows_of = P.perm.as<uint32_t>();  // posting row -> source row
    if (distinct && n > 1) {
        // identical rows are adjacent in canonical order: one posting row per distinct row
        DevBuf head(n * 4, ctx.stream), nsel(8, ctx.stream);
        P.group.alloc(n * 4, ctx.stream);
        P.rep.alloc(n * 4, ctx.stream);
        IGB_LAUNCH(ctx, row_heads, grid_for(ctx, n, 256), 256, 0, d_rows, P.perm.as<uint32_t>(), n, (int)k,
                   head.as<uint32_t>());
        size_t tb = 0;
        IGB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, head.as<uint32_t>(), P.group.as<uint32_t>(), (int64_t)n,
                                               ctx.stream));
        size_t tb2 = 0;
        IGB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, P.perm.as<uint32_t>(), head.as<uint32_t>(),
                                            P.rep.as<uint32_t>(), nsel.as<int64_t>(), (int64_t)n, ctx.stream));
        DevBuf temp(std::max(tb, tb2), ctx.stream);
        // group[i] = (#heads in [0, i]) - 1: exclusive sum of heads shifted by the head at i
        IGB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, head.as<uint32_t>(), P.group.as<uint32_t>(), (int64_t)n,
                                               ctx.stream));
        IGB_CUDA(cub::DeviceSelect::Flagged(temp.p, tb2, P.perm.as<uint32_t>(), head.as<uint32_t>(),
                                            P.rep.as<uint32_t>(), nsel.as<int64_t>(), (int64_t)n, ctx.stream));
        IGB_LAUNCH(ctx, fix_group, grid_for(ctx, n, 256), 256, 0, head.as<uint32_t>(), n, P.group.as<uint32_t>());
        int64_t m = 0;
        read_back(ctx, &m, nsel.p, 8);
        nd = (size_t)m;
        rows_of = P.rep.as<uint32_t>();
    }
    P.n = nd;
    P.W = (nd + 63) / 64;
    const size_t W = std::max<size_t>(P.W, 1);
    P.dense.alloc((size_t)L * W * 8, ctx.stream);
    P.df.alloc((size_t)L * 4, ctx.stream);
    P.nz_off.alloc(((size_t)L + 1) * 4, ctx.stream);
    DevBuf nzc(((size_t)L + 1) * 4, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(P.dense.p, 0, (size_t)L * W * 8, ctx.stream));
    if (nd && k) {
        const size_t warps = P.W * k;
        IGB_LAUNCH(ctx, transpose_rows, grid_for(ctx, warps * 32, 256), 256, 0, d_rows, rows_of, nd, (int)k, P.W,
                   P.dense.as<unsigned long long>());
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
    // (sized for every word non-zero: half the dense bytes, no read-back)
    P.nz_idx.alloc(std::max<size_t>((size_t)L * P.W, 1) * 4, ctx.stream);
    IGB_LAUNCH(ctx, fill_nonzero, grid_for(ctx, (size_t)L * 32, 256), 256, 0, P.dense.as<unsigned long long>(), L,
               P.W, P.nz_off.as<uint32_t>(), P.nz_idx.as<uint32_t>());
}

void posting_support(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, int64_t* d_support,
                     const PatternIndex* I) {
    launch_scan<kSupport>(ctx, d_pat, np, k, P, I, nullptr, nullptr, d_support, nullptr, nullptr);
}

void posting_cover(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, uint8_t* d_mask,
                   const PatternIndex* I) {
    launch_scan<kCover>(ctx, d_pat, np, k, P, I, nullptr, nullptr, nullptr, d_mask, nullptr);
}

void posting_match(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* d_scores, const Postings& P,
                   int64_t* d_out, int* d_overflow, bool sum_fits, const PatternIndex* I) {
    const size_t n = std::max<size_t>(P.n, 1);
    if (P.group.p == nullptr && P.perm.p == nullptr && P.n_src != P.n) fail(IG_E_CUDA, "posting_match: bad postings");
    // sum_fits: Σ scores <= INT64_MAX, so no evidence sum can overflow: run-based
    // difference array + scan (fire-and-forget REDs).  Otherwise per-match
    // checked atomics.
    DevBuf acc((n + 64 + 1) * 8, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(acc.p, 0, (n + 64 + 1) * 8, ctx.stream));
    if (sum_fits) {
        launch_scan<kMatch>(ctx, d_pat, np, k, P, I, d_scores, acc.as<unsigned long long>(), nullptr, nullptr,
                            d_overflow);
        size_t tb = 0;
        IGB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, acc.as<unsigned long long>(), acc.as<unsigned long long>(),
                                               (int64_t)n, ctx.stream));
        DevBuf temp(tb, ctx.stream);
        IGB_CUDA(cub::DeviceScan::InclusiveSum(temp.p, tb, acc.as<unsigned long long>(), acc.as<unsigned long long>(),
                                               (int64_t)n, ctx.stream));
    } else {
        launch_scan<kMatchChecked>(ctx, d_pat, np, k, P, I, d_scores, acc.as<unsigned long long>(), nullptr, nullptr,
                                   d_overflow);
    }
    if (!P.perm.p) {
        IGB_CUDA(cudaMemcpyAsync(d_out, acc.p, std::max<size_t>(P.n, 1) * 8, cudaMemcpyDeviceToDevice, ctx.stream));
        return;
    }
    // accumulated in the postings' (canonical) row order: scatter back to source rows
    IGB_LAUNCH(ctx, scatter_u64, grid_for(ctx, P.n_src, 256), 256, 0, acc.as<unsigned long long>(),
               P.perm.as<uint32_t>(), P.group.as<uint32_t>(), P.n_src, d_out);
}

}  // namespace igb
