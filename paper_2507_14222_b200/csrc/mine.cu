// mine.cu — candidate enumeration (kernel 2), exact dedup (kernel 3), scores,
// canonical ordering.
//
// Reference semantics: enumerate_candidates proj/include/ig/mine.hpp:35-40 with
// SPEC.md:301-309 (B^c = {x_i ∩ x_j : i<j, non-empty} ∪ X^c, dedup by content,
// canonical words::less order, bitpack.hpp:59-68); score_patterns / total_score
// mine.hpp:46-51.
//
// Design (B200): class rows are L2-resident (≤17 MB for NSL shape).  A CTA owns
// a 64×64 tile of the upper triangle (u ≤ v; the diagonal u == v yields the
// union term X_u itself).  Both row blocks are staged in shared memory with an
// odd row stride (conflict-free 64-bit lane access).  Each pair's AND is
// fingerprinted and inserted into one device-wide open-addressing table of
// 16-byte slots {fingerprint, representative pair (u,v)} claimed with a single
// 128-bit atom.cas.  An insert that meets an equal fingerprint re-materialises
// the representative's words from L2 and compares all K words: equal → duplicate;
// different → a genuine 64-bit collision, deferred to a second table with a new
// seed (levels repeat until empty), so the result is exact by construction.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <ctime>

#include "ig_internal.cuh"
#include "subset.cuh"

namespace igb {

namespace {

constexpr int kPairThreads = 256;
constexpr uint64_t kRepInit = 0ull;  // slot.y = ((u << 32) | v) + 1 once written; all-zero slot = empty

struct Table {
    ulonglong2* slots;
    uint64_t mask;
    uint2* reps;
    unsigned long long* count;
    unsigned long long limit;  // max distinct before the table is declared full
    uint2* ovf;
    unsigned long long* ovf_count;
    unsigned long long ovf_cap;
    unsigned long long* collisions;
    int* fail;  // bit0 table full, bit1 overflow list full, bit2 retry list full
    uint2* retry;                     // pairs the tile-local table could not place (inserted after the kernel)
    unsigned long long* retry_count;
    unsigned long long retry_cap;
    uint64_t seed;
    const unsigned long long* keys;  // K fingerprint keys of this level (derived from seed)
    uint64_t fp_mask;                // ~0; narrowed only by the IG_TEST_FP_BITS collision test knob
};

__device__ __forceinline__ ulonglong2 cas128(ulonglong2* addr, ulonglong2 cmp, ulonglong2 val) {
    ulonglong2 old;
    asm volatile(
        "{\n\t.reg .b128 c, n, o;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 n, {%4, %5};\n\t"
        "atom.global.cas.b128 o, [%6], c, n;\n\t"
        "mov.b128 {%0, %1}, o;\n\t}"
        : "=l"(old.x), "=l"(old.y)
        : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(addr)
        : "memory");
    return old;
}

// Per-word fingerprint keys of one hash level (splitmix64 stream of the seed).
constexpr uint64_t kOwnerSeed = 0x6a09e667f3bcc909ull;
__global__ void fp_keys(uint64_t seed, int k, unsigned long long* __restrict__ keys) {
    for (int w = threadIdx.x; w < k; w += blockDim.x) keys[w] = mix64(seed + 0x9e3779b97f4a7c15ull * (uint64_t)(w + 1));
}

__device__ __forceinline__ uint64_t ld_volatile(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// Insert candidate (u,v) with fingerprint fp.  `b(w)` yields word w of the
// candidate; X is the class row matrix used to re-materialise representatives.
// Per-CTA staging of new representatives (pair_enum): a claim takes a slot in
// shared memory (a shared atomic, not an L2 round trip on the one hot counter);
// the CTA reserves its range of the reps list once per tile.
constexpr int kStageReps = 1024;
struct RepStage {
    uint2* reps;          // shared [kStageReps]
    unsigned int* count;  // shared
};

template <class WordFn>
__device__ void table_insert(const Table& T, const int64_t* __restrict__ X, int k, uint32_t u, uint32_t v,
                             uint64_t fp, WordFn b, const RepStage* stage = nullptr) {
    const uint64_t rep = (((uint64_t)u << 32) | v) + 1;
    uint64_t s = (fp ^ T.seed) & T.mask;
    for (uint64_t probes = 0; probes <= T.mask; ++probes, s = (s + 1) & T.mask) {
        if ((probes & 63) == 63 && *(volatile int*)T.fail) return;  // long probe into a full table
        ulonglong2* slot = T.slots + s;
        ulonglong2 cur;
        cur.x = ld_volatile(&slot->x);
        cur.y = kRepInit;  // loaded below only when the fingerprint matches
        if (cur.x == 0) {
            const ulonglong2 old = cas128(slot, make_ulonglong2(0ull, 0ull), make_ulonglong2(fp, rep));
            if (old.x == 0) {
                if (stage) {
                    const unsigned int i = atomicAdd(stage->count, 1u);
                    if (i < (unsigned int)kStageReps) {
                        stage->reps[i] = make_uint2(u, v);
                        return;
                    }
                    // staging full: straight to the reps list
                    const unsigned long long idx = atomicAdd(T.count, 1ull);
                    if (idx < T.limit)
                        T.reps[idx] = make_uint2(u, v);
                    else
                        atomicOr(T.fail, 1);
                    return;
                }
                // warp-aggregated slot in the reps list: the count is one hot address
                const unsigned int mask = __activemask();
                const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
                unsigned long long base = 0;
                if (lane == leader) base = atomicAdd(T.count, (unsigned long long)__popc(mask));
                base = __shfl_sync(mask, base, leader);
                const unsigned long long idx = base + __popc(mask & ((1u << lane) - 1u));
                if (idx < T.limit)
                    T.reps[idx] = make_uint2(u, v);
                else
                    atomicOr(T.fail, 1);
                return;
            }
            cur = old;
        }
        if (cur.x != fp) continue;
        uint64_t r = cur.y;
        while (r == kRepInit) r = ld_volatile(&slot->y);  // not loaded yet, or the winner's store is in flight
        --r;
        const uint32_t ru = (uint32_t)(r >> 32), rv = (uint32_t)r;
        const int64_t* a = X + (size_t)ru * k;
        const int64_t* c = X + (size_t)rv * k;
        // the representative's words in chunks of independent loads: one L2
        // round trip per chunk instead of one per word (the word-at-a-time
        // early-exit loop was the largest stall of pair_enum)
        constexpr int kChunk = 7;
        bool same = true;
        for (int w0 = 0; w0 < k && same; w0 += kChunk) {
            uint64_t va[kChunk], vc[kChunk];
#pragma unroll
            for (int j = 0; j < kChunk; ++j)
                if (w0 + j < k) {
                    va[j] = (uint64_t)__ldg(a + w0 + j);
                    vc[j] = (uint64_t)__ldg(c + w0 + j);
                }
#pragma unroll
            for (int j = 0; j < kChunk; ++j)
                if (w0 + j < k) same &= ((va[j] & vc[j]) == (uint64_t)b(w0 + j));
        }
        if (same) return;
        // equal fingerprint, different content: defer to the next level
        atomicAdd(T.collisions, 1ull);
        const unsigned long long o = atomicAdd(T.ovf_count, 1ull);
        if (o < T.ovf_cap)
            T.ovf[o] = make_uint2(u, v);
        else
            atomicOr(T.fail, 2);
        return;
    }
    atomicOr(T.fail, 1);
}

// TMA (bulk async copy) of a row block into shared memory, completion tracked
// by an mbarrier's transaction count (sm_90+ cp.async.bulk)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_rows(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

// x[w] = a[w] & b[w] for w < KC; two words per shared-memory load for K = 14
template <int KC>
__device__ __forceinline__ void load_and_x(const int64_t* a, const int64_t* b, uint64_t* x) {
    if (KC != 14) {
#pragma unroll
        for (int w = 0; w < KC; ++w) x[w] = (uint64_t)(a[w] & b[w]);
        return;
    }
#pragma unroll
    for (int w = 0; w + 1 < KC; w += 2) {
        const ulonglong2 va = *reinterpret_cast<const ulonglong2*>(a + w);
        const ulonglong2 vb = *reinterpret_cast<const ulonglong2*>(b + w);
        x[w] = va.x & vb.x;
        x[w + 1] = va.y & vb.y;
    }
    if (KC & 1) x[KC - 1] = (uint64_t)(a[KC - 1] & b[KC - 1]);
}

__device__ __forceinline__ void tile_of(uint64_t t, uint32_t& bi, uint32_t& bj) {
    // t enumerates (bi <= bj) column by column: t = bj(bj+1)/2 + bi
    uint64_t j = (uint64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while (j * (j + 1) / 2 > t) --j;
    while ((j + 1) * (j + 2) / 2 <= t) ++j;
    bj = (uint32_t)j;
    bi = (uint32_t)(t - j * (j + 1) / 2);
}

// One CTA per 64x64 tile of the triangle u <= v (grid-stride over tiles).
// Pairs are first deduplicated inside the tile (shared-memory hash of
// fingerprint tags, exact compare on the tile's staged rows), so only the first
// pair of each distinct content in a tile probes the device-wide table.
constexpr int kLocalSlots = 4096;
constexpr int kLocalProbes = 64;  // then the pair goes to the retry list (adversarial fingerprints only)
constexpr size_t kProjectRows = 16384;  // distinct class rows from which off-diagonal tiles are projected

// KC > 0: the row width K is a compile-time constant (the common NSL shapes),
// so the word loops unroll; KC <= 16 also keeps the pair's AND in registers
// for the duplicate check.
template <int TILE, int KC, bool PROJ>
__global__ void __launch_bounds__(kPairThreads, KC == 17 ? 4 : KC > 0 && KC <= 16 ? 5 : 6)
pair_enum(const int64_t* __restrict__ X, uint32_t n, int k_rt, int stride, uint64_t n_tiles, Table T,
          uint64_t tile_begin, uint64_t tile_step, unsigned long long* __restrict__ prog_ctr,
          unsigned long long* __restrict__ prog_host, int use_tma) {
    const int k = KC > 0 ? KC : k_rt;
    constexpr bool kRegs = KC > 0 && KC <= 17;
    extern __shared__ int64_t sm[];
    unsigned int* local = reinterpret_cast<unsigned int*>(sm);  // kLocalSlots 32-bit entries
    int64_t* sI = sm + kLocalSlots / 2;
    int64_t* sJ = sI + (size_t)TILE * stride;
    unsigned long long* sKey = reinterpret_cast<unsigned long long*>(sJ + (size_t)TILE * stride);  // k fingerprint keys
    unsigned long long* sOr = sKey + k;  // 2k: OR of block I's rows, then of block J's
    __shared__ unsigned long long s_h[2][TILE];     // hash of each projected row
    __shared__ uint8_t s_list[2][TILE];             // distinct projected rows of I and J
    __shared__ int s_cnt[2];
    __shared__ uint2 s_reps[kStageReps];
    __shared__ unsigned int s_nrep;
    __shared__ unsigned long long s_base;
    __shared__ int s_stop;
    __shared__ unsigned long long s_pairs;  // pairs of the tile just finished (progress)
    __shared__ alignas(8) uint64_t s_bar;   // TMA row-block arrival
    // row blocks arrive by TMA when the shared layout is the global one (the
    // stride is K itself: K = 14, or odd K in the generic kernels) and the
    // block is full
    const bool tma = use_tma && stride == k;
    unsigned phase = 0;
    if (tma && threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const RepStage stage{s_reps, &s_nrep};
    for (int w = threadIdx.x; w < k; w += kPairThreads) sKey[w] = T.keys[w];
    if (threadIdx.x == 0) {
        s_nrep = 0;
        s_pairs = 0;
    }
    for (uint64_t it = blockIdx.x;; it += gridDim.x) {
        const uint64_t t = tile_begin + it * tile_step;  // this rank's tiles: begin, begin + step, ...
        // the previous tile's staged representatives -> one reserved range of
        // the reps list; one reader for the failure flag, so the whole block
        // leaves together
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned int n = min(s_nrep, (unsigned int)kStageReps);
            s_base = n ? atomicAdd(T.count, (unsigned long long)n) : 0ull;
            s_stop = *(volatile int*)T.fail;
            if (prog_ctr && s_pairs) {
                // publish progress to the polling host thread (values only grow;
                // the host keeps the largest it has seen)
                const unsigned long long d = atomicAdd(prog_ctr, s_pairs) + s_pairs;
                *(volatile unsigned long long*)prog_host = d;
                *(volatile unsigned long long*)(prog_host + 1) = s_base + n;
                s_pairs = 0;
            }
        }
        __syncthreads();
        {
            const unsigned int n = min(s_nrep, (unsigned int)kStageReps);
            for (unsigned int i = threadIdx.x; i < n; i += kPairThreads) {
                const unsigned long long idx = s_base + i;
                if (idx < T.limit)
                    T.reps[idx] = s_reps[i];
                else
                    atomicOr(T.fail, 1);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) s_nrep = 0;
        if (t >= n_tiles || s_stop) return;
        uint32_t bi, bj;
        tile_of(t, bi, bj);
        const uint32_t i0 = bi * TILE, j0 = bj * TILE;
        if (threadIdx.x == 0 && prog_ctr) {
            const unsigned long long ri = min((uint32_t)TILE, n - i0), rj = min((uint32_t)TILE, n - j0);
            s_pairs = bi == bj ? ri * (ri + 1) / 2 : ri * rj;
        }
        const bool tI = tma && i0 + TILE <= n, tJ = tma && j0 + TILE <= n;
        if ((tI || tJ) && threadIdx.x == 0) {
            // the previous tile's generic-proxy writes (projection) are complete
            // (barrier above); order them before the async-proxy overwrite
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const unsigned bytes = (unsigned)(TILE * k * 8);
            mbar_expect_tx(&s_bar, (tI ? bytes : 0u) + (tJ ? bytes : 0u));
            if (tI) tma_load_rows(sI, X + (size_t)i0 * k, bytes, &s_bar);
            if (tJ) tma_load_rows(sJ, X + (size_t)j0 * k, bytes, &s_bar);
        }
        if (!tI || !tJ)
            for (int q = threadIdx.x; q < TILE * k; q += kPairThreads) {
                const int r = q / k, w = q % k;
                if (!tI) sI[r * stride + w] = (i0 + r < n) ? X[(size_t)(i0 + r) * k + w] : 0;
                if (!tJ) sJ[r * stride + w] = (j0 + r < n) ? X[(size_t)(j0 + r) * k + w] : 0;
            }
        for (int q = threadIdx.x; q < kLocalSlots; q += kPairThreads) local[q] = 0u;
        if (tI || tJ) {
            mbar_wait(&s_bar, phase);
            phase ^= 1u;
        }
        // plain: pairs numbered q = r * TILE + c over the whole tile (diagonal
        // tiles, or projection off); else over the blocks' distinct projections
        const bool plain = !PROJ || bi == bj;
        const int nrI = (int)min((uint32_t)TILE, n - i0), nrJ = plain ? 0 : (int)min((uint32_t)TILE, n - j0);
        if (!plain) {
            // Row equivalence within an off-diagonal tile: with OR_J the OR of
            // block J's rows, x_u & x_v = (x_u & OR_J) & (x_v & OR_I) for every
            // u in I, v in J.  So each block is projected onto the other's OR
            // and only its distinct projections are paired — the tile's set of
            // intersections is unchanged (exact), and rows that differ only in
            // tokens the other block never holds (prototype mutations) collapse.
            __syncthreads();
            // ORs: a warp per word, two rows per lane, shuffle reduction
            for (int q = threadIdx.x >> 5; q < 2 * k; q += kPairThreads / 32) {
                const int side = q >= k, w = side ? q - k : q, lane = threadIdx.x & 31;
                const int64_t* src = side ? sJ : sI;
                const int nr = side ? nrJ : nrI;
                unsigned long long acc = 0;
                for (int r = lane; r < nr; r += 32) acc |= (unsigned long long)src[r * stride + w];
                for (int o = 16; o; o >>= 1) acc |= __shfl_xor_sync(0xffffffffu, acc, o);
                if (lane == 0) sOr[q] = acc;
            }
            __syncthreads();
            for (int q = threadIdx.x; q < TILE * k; q += kPairThreads) {
                const int r = q / k, w = q % k;
                sI[r * stride + w] &= (int64_t)sOr[k + w];
                sJ[r * stride + w] &= (int64_t)sOr[w];
            }
            __syncthreads();
            for (int q = threadIdx.x; q < 2 * TILE; q += kPairThreads) {
                const int side = q >= TILE, r = side ? q - TILE : q;
                const int64_t* row = (side ? sJ : sI) + r * stride;
                unsigned long long h = 0x9e3779b97f4a7c15ull;
                for (int w = 0; w < k; ++w) h = mix64(h ^ (unsigned long long)row[w]);
                s_h[side][r] = h;
            }
            __syncthreads();
            // a row is listed iff no earlier row of its block has the same projection
            if (threadIdx.x < 64) {
                const int side = threadIdx.x >> 5, lane = threadIdx.x & 31;
                const int nr = side ? nrJ : nrI;
                const int64_t* blk = side ? sJ : sI;
                int cnt = 0;
                for (int r0 = 0; r0 < TILE; r0 += 32) {
                    const int r = r0 + lane;
                    bool first = r < nr;
                    if (first) {
                        const unsigned long long h = s_h[side][r];
                        for (int r2 = 0; r2 < r && first; ++r2) {
                            if (s_h[side][r2] != h) continue;
                            bool same = true;
                            for (int w = 0; w < k && same; ++w) same = blk[r * stride + w] == blk[r2 * stride + w];
                            first = !same;
                        }
                    }
                    const unsigned int bal = __ballot_sync(0xffffffffu, first);
                    if (first) s_list[side][cnt + __popc(bal & ((1u << lane) - 1u))] = (uint8_t)r;
                    cnt += __popc(bal);
                }
                if (lane == 0) s_cnt[side] = cnt;
            }
        }
        __syncthreads();
        const int nI = plain ? TILE : s_cnt[0], nJ = plain ? TILE : s_cnt[1];
        const int npairs = nI * nJ;
        for (int q0 = 0; q0 < npairs; q0 += kPairThreads) {
            // every lane runs the same trip count (npairs need not be a multiple
            // of the block): re-converge the warp each pair so the AND +
            // fingerprint work runs on full warps (lanes otherwise drift apart
            // after the data-dependent probe paths)
            __syncwarp();
            const int q = q0 + (int)threadIdx.x;
            if (q >= npairs) continue;
            const int r = plain ? q / TILE : s_list[0][q / nJ], c = plain ? q % TILE : s_list[1][q % nJ];
            const uint32_t u = i0 + r, v = j0 + c;
            if (u >= n || v >= n || u > v) continue;
            const int64_t* a = sI + r * stride;
            const int64_t* b = sJ + c * stride;
            Fp fp;
            uint64_t nz = 0;
            uint64_t xr[kRegs ? KC : 1];
            if constexpr (kRegs) {
                // K = 14: 128-bit shared loads (the row stride is 14 = 2 mod 4
                // words, so rows are 16-byte aligned and the 8 lanes of a
                // quarter-warp hit 8 distinct 4-bank groups); K = 17: 64-bit
                load_and_x<KC>(a, b, xr);
#pragma unroll
                for (int w = 0; w < KC; ++w) {
                    nz |= xr[w];
                    fp.add(xr[w], sKey[w]);
                }
            } else {
                for (int w = 0; w < k; ++w) {
                    const uint64_t x = (uint64_t)(a[w] & b[w]);
                    nz |= x;
                    fp.add(x, sKey[w]);
                }
            }
            if (!nz) continue;  // SPEC.md:338 empty intersections dropped at the source
            const uint64_t f = (fp.final(k) & T.fp_mask) | 1ull;
            // local entry: 20-bit tag from the fingerprint's top bits (never zero;
            // the slot comes from its low bits) | 12-bit pair index within the tile.
            // A tag match is only a hint: the words decide.
            const unsigned int entry = ((unsigned int)(f >> 44) | 1u) << 12 | (unsigned int)q;
            bool dup = false, placed = false;
            uint32_t s = (uint32_t)(f & (kLocalSlots - 1));
            for (int probe = 0; probe < kLocalProbes; ++probe, s = (s + 1) & (kLocalSlots - 1)) {
                unsigned int cur = local[s];
                if (cur == 0u) {
                    cur = atomicCAS(local + s, 0u, entry);
                    if (cur == 0u) {  // first of its content in this tile
                        placed = true;
                        break;
                    }
                }
                if ((cur >> 12) != (entry >> 12)) continue;
                const int q2 = (int)(cur & 0xfffu);  // in this tile's pair numbering (projected lists)
                const int64_t* a2 = sI + (plain ? q2 / TILE : s_list[0][q2 / nJ]) * stride;
                const int64_t* b2 = sJ + (plain ? q2 % TILE : s_list[1][q2 % nJ]) * stride;
                bool same = true;
                if constexpr (kRegs) {
                    uint64_t y[KC];
                    load_and_x<KC>(a2, b2, y);
#pragma unroll
                    for (int w = 0; w < KC; ++w) same &= y[w] == xr[w];
                } else {
                    for (int w = 0; w < k && same; ++w) same = ((a2[w] & b2[w]) == (a[w] & b[w]));
                }
                if (same) {
                    dup = true;
                    break;
                }
            }
            // the first of its content (placed) is inserted into the device
            // table after the tile, on full warps (inline, the inserts ran
            // ~2.5 lanes wide); a pair the local table could not place within
            // kLocalProbes probes (only with adversarial fingerprints) is
            // inserted into the same table by a follow-up launch
            if (!dup && !placed) {
                const unsigned long long o = atomicAdd(T.retry_count, 1ull);
                if (o < T.retry_cap)
                    T.retry[o] = make_uint2(u, v);
                else
                    atomicOr(T.fail, 4);
            }
        }
        // deferred inserts: each warp compacts its 512 local slots in place to
        // the pair indices they hold, then inserts them 32 at a time
        __syncthreads();
        {
            const int lane = threadIdx.x & 31;
            constexpr int kPer = kLocalSlots / (kPairThreads / 32);
            unsigned int* mine = local + (threadIdx.x >> 5) * kPer;
            int cnt = 0;
            for (int c0 = 0; c0 < kPer; c0 += 32) {
                const unsigned int ent = mine[c0 + lane];
                const unsigned int bal = __ballot_sync(0xffffffffu, ent != 0u);
                __syncwarp();
                if (ent) mine[cnt + __popc(bal & ((1u << lane) - 1u))] = ent & 0xfffu;
                cnt += __popc(bal);
                __syncwarp();
            }
            for (int i = lane; i < cnt; i += 32) {
                const int qq = (int)mine[i];
                const int r = plain ? qq / TILE : s_list[0][qq / nJ], c = plain ? qq % TILE : s_list[1][qq % nJ];
                const int64_t* a = sI + r * stride;
                const int64_t* b = sJ + c * stride;
                Fp fp;
#pragma unroll
                for (int w = 0; w < k; ++w) fp.add((uint64_t)(a[w] & b[w]), sKey[w]);
                const uint64_t f = (fp.final(k) & T.fp_mask) | 1ull;
                table_insert(T, X, k, i0 + r, j0 + c, f, [&](int w) { return a[w] & b[w]; }, &stage);
            }
        }
    }
}

// Re-insert deferred (collided) pairs into a fresh level with a new seed.
__global__ void pair_insert_list(const int64_t* __restrict__ X, int k, const uint2* __restrict__ list,
                                 size_t n_list, Table T) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_list;
         i += (size_t)gridDim.x * blockDim.x) {
        if (*(volatile int*)T.fail) return;  // table full: the host retries with a larger one
        const uint2 p = list[i];
        const int64_t* a = X + (size_t)p.x * k;
        const int64_t* b = X + (size_t)p.y * k;
        Fp fp;
        for (int w = 0; w < k; ++w) fp.add((uint64_t)(__ldg(a + w) & __ldg(b + w)), __ldg(T.keys + w));
        table_insert(T, X, k, p.x, p.y, (fp.final(k) & T.fp_mask) | 1ull,
                     [&](int w) { return __ldg(a + w) & __ldg(b + w); });
    }
}

__global__ void materialize(const int64_t* __restrict__ X, int k, const uint2* __restrict__ reps, size_t n,
                            int64_t* __restrict__ out) {
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n * k;
         q += (size_t)gridDim.x * blockDim.x) {
        const size_t i = q / k;
        const int w = (int)(q % k);
        const uint2 p = reps[i];
        out[q] = X[(size_t)p.x * k + w] & X[(size_t)p.y * k + w];
    }
}

__global__ void gather_key(const int64_t* __restrict__ words, const uint32_t* __restrict__ perm, size_t n,
                           int k, int w, uint64_t* __restrict__ key) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        key[i] = (uint64_t)words[(size_t)perm[i] * k + w];
}

__global__ void iota_u32(uint32_t* p, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

__global__ void gather_rows_k(const int64_t* __restrict__ src, const uint32_t* __restrict__ perm, size_t n,
                              int k, int64_t* __restrict__ dst) {
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n * k;
         q += (size_t)gridDim.x * blockDim.x)
        dst[q] = src[(size_t)perm[q / k] * k + (q % k)];
}

__global__ void gather_i64(const int64_t* __restrict__ src, const uint32_t* __restrict__ perm, size_t n,
                           int64_t* __restrict__ dst) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[perm[i]];
}

__global__ void score_k(const int64_t* __restrict__ pat, size_t n, int k, const int64_t* __restrict__ sup,
                        int64_t* __restrict__ score, int* __restrict__ ovf) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        int64_t size = 0;
        for (int w = 0; w < k; ++w) size += __popcll((unsigned long long)pat[i * k + w]);
        const int64_t sq = size * size;  // size <= 64k bits: no overflow
        const int64_t f = sup[i];
        int64_t s;
        // f * sq overflows int64 iff |f| > INT64_MAX / sq (sq > 0; f >= 0 here)
        if (sq != 0 && (f > INT64_MAX / sq || f < INT64_MIN / sq)) {
            atomicOr(ovf, 1);
            s = 0;
        } else {
            s = f * sq;
        }
        score[i] = s;
    }
}

// Checked Σ in 128-bit per block, combined on the host.
__global__ void sum128(const int64_t* __restrict__ s, size_t n, unsigned long long* __restrict__ out_lo,
                       long long* __restrict__ out_hi) {
    __int128 acc = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc += s[i];
    typedef cub::BlockReduce<long long, 256> BR;
    __shared__ typename BR::TempStorage t1, t2;
    // split into (hi, lo32) pieces that fit long long sums across 256 threads
    const long long hi = (long long)(acc >> 32);
    const long long lo = (long long)(acc & 0xffffffff);
    const long long shi = BR(t1).Sum(hi);
    __syncthreads();
    const long long slo = BR(t2).Sum(lo);
    if (threadIdx.x == 0) {
        out_lo[blockIdx.x] = (unsigned long long)slo;
        out_hi[blockIdx.x] = shi;
    }
}

unsigned grid_for(const Ctx& ctx, size_t work, int threads) {
    size_t g = (work + threads - 1) / threads;
    const size_t cap = (size_t)ctx.sm_count * 32;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

struct TableMem {
    DevBuf slots, reps, ovf, ctr, keys, retry;  // ctr: count, ovf_count, collisions, fail, retry_count
    Table make(Ctx& ctx, uint64_t cap, uint64_t ovf_cap, uint64_t seed, size_t k, uint64_t retry_cap = 1) {
        keys.alloc(std::max<size_t>(k, 1) * 8, ctx.stream);
        IGB_LAUNCH(ctx, fp_keys, 1, 256, 0, seed, (int)k, keys.as<unsigned long long>());
        slots.alloc(cap * sizeof(ulonglong2), ctx.stream);
        IGB_CUDA(cudaMemsetAsync(slots.p, 0, cap * sizeof(ulonglong2), ctx.stream));  // empty slot = {0, 0}
        const uint64_t limit = cap / 4 * 3;
        reps.alloc(limit * sizeof(uint2), ctx.stream);
        ovf.alloc(ovf_cap * sizeof(uint2), ctx.stream);
        ctr.alloc(5 * sizeof(unsigned long long), ctx.stream);
        IGB_CUDA(cudaMemsetAsync(ctr.p, 0, 5 * sizeof(unsigned long long), ctx.stream));
        retry.alloc(std::max<uint64_t>(retry_cap, 1) * sizeof(uint2), ctx.stream);
        Table T;
        T.slots = slots.as<ulonglong2>();
        T.mask = cap - 1;
        T.reps = reps.as<uint2>();
        T.count = ctr.as<unsigned long long>();
        T.limit = limit;
        T.ovf = ovf.as<uint2>();
        T.ovf_count = ctr.as<unsigned long long>() + 1;
        T.ovf_cap = ovf_cap;
        T.collisions = ctr.as<unsigned long long>() + 2;
        T.fail = reinterpret_cast<int*>(ctr.as<unsigned long long>() + 3);
        T.retry = retry.as<uint2>();
        T.retry_count = ctr.as<unsigned long long>() + 4;
        T.retry_cap = std::max<uint64_t>(retry_cap, 1);
        T.seed = seed;
        T.keys = keys.as<unsigned long long>();
        T.fp_mask = ~0ull;
        if (const char* e = std::getenv("IG_TEST_FP_BITS")) {  // test knob: force fingerprint collisions
            const int bits = std::atoi(e);
            if (bits > 0 && bits < 64) T.fp_mask = (1ull << bits) - 1;
        }
        return T;
    }
};

// Calling thread: report progress while the enumeration runs on the stream.
void poll_progress(Ctx& ctx) {
    ProgressHook& p = *ctx.progress;
    for (;;) {
        const cudaError_t q = cudaStreamQuery(ctx.stream);
        const unsigned long long d = *(volatile unsigned long long*)p.host;
        const unsigned long long f = *(volatile unsigned long long*)(p.host + 1);
        if (d > p.seen[0] || f > p.seen[1]) {
            p.seen[0] = std::max<uint64_t>(p.seen[0], d);
            p.seen[1] = std::max<uint64_t>(p.seen[1], f);
            if (p.seen[0] < p.pairs_total) p.fn(p.seen[0], p.pairs_total, p.seen[1], p.user);
        }
        if (q != cudaErrorNotReady) break;
        struct timespec ts = {0, 500000};  // 0.5 ms
        nanosleep(&ts, nullptr);
    }
}

uint64_t next_pow2(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

__global__ void pair_window_k(const int64_t* __restrict__ left, const int64_t* __restrict__ rows, size_t cnt, int k,
                              int64_t* __restrict__ out) {
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt * k; q += (size_t)gridDim.x * blockDim.x)
        out[q] = left[q % k] & rows[q];
}

}  // namespace

void pair_window_dev(Ctx& ctx, const int64_t* d_left, const int64_t* d_rows, size_t cnt, size_t k, int64_t* d_out) {
    IGB_LAUNCH(ctx, pair_window_k, grid_for(ctx, cnt * k, 256), 256, 0, d_left, d_rows, cnt, (int)k, d_out);
}

void sort_rows_canonical_lsd(Ctx& ctx, const int64_t* d_words, size_t n, size_t k, uint32_t* d_perm) {
    if (n == 0) return;
    IGB_LAUNCH(ctx, iota_u32, grid_for(ctx, n, 256), 256, 0, d_perm, n);
    if (n == 1) return;
    DevBuf keys(n * 8, ctx.stream), keys2(n * 8, ctx.stream), perm2(n * 4, ctx.stream);
    size_t temp_bytes = 0;
    IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                             d_perm, perm2.as<uint32_t>(), (int64_t)n, 0, 64, ctx.stream));
    DevBuf temp(temp_bytes, ctx.stream);
    uint32_t* cur = d_perm;
    uint32_t* alt = perm2.as<uint32_t>();
    // LSD over words K-1 .. 0 with a stable radix sort: lexicographic unsigned order.
    for (int w = (int)k - 1; w >= 0; --w) {
        IGB_LAUNCH(ctx, gather_key, grid_for(ctx, n, 256), 256, 0, d_words, cur, n, (int)k, w, keys.as<uint64_t>());
        IGB_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, temp_bytes, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                                 cur, alt, (int64_t)n, 0, 64, ctx.stream));
        std::swap(cur, alt);
    }
    if (cur != d_perm) IGB_CUDA(cudaMemcpyAsync(d_perm, cur, n * 4, cudaMemcpyDeviceToDevice, ctx.stream));
}

void gather_rows(Ctx& ctx, const int64_t* d_src, const uint32_t* d_perm, size_t n, size_t k, int64_t* d_dst) {
    if (n == 0) return;
    IGB_LAUNCH(ctx, gather_rows_k, grid_for(ctx, n * k, 256), 256, 0, d_src, d_perm, n, (int)k, d_dst);
}

void canonical_order(Ctx& ctx, DevRows& rows, DevBuf* a, DevBuf* b, DevBuf* o_perm) {
    const size_t n = rows.n, k = rows.k;
    if (n < 2) return;
    DevBuf perm(n * 4, ctx.stream);
    sort_rows_canonical(ctx, rows.data(), n, k, perm.as<uint32_t>());
    DevBuf sorted(n * k * 8, ctx.stream);
    gather_rows(ctx, rows.data(), perm.as<uint32_t>(), n, k, sorted.as<int64_t>());
    rows.buf = std::move(sorted);
    for (DevBuf* pay : {a, b}) {
        if (!pay || !pay->p) continue;
        DevBuf t(n * 8, ctx.stream);
        IGB_LAUNCH(ctx, gather_i64, grid_for(ctx, n, 256), 256, 0, pay->as<int64_t>(), perm.as<uint32_t>(), n,
                   t.as<int64_t>());
        *pay = std::move(t);
    }
    if (o_perm) *o_perm = std::move(perm);
}

__global__ void compose_k(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, size_t n,
                          uint32_t* __restrict__ out) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        out[i] = a[b ? b[i] : i];
}

void compose_u32(Ctx& ctx, const uint32_t* a, const uint32_t* b, size_t n, uint32_t* out) {
    if (n) IGB_LAUNCH(ctx, compose_k, grid_for(ctx, n, 256), 256, 0, a, b, n, out);
}

// Identical rows give identical intersections, so B^c over the distinct rows
// (canonical order, which also groups similar rows into the same tiles) equals
// B^c over all rows with up to quadratically fewer pairs.
void enumerate_dev(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, uint32_t L, DevRows& out,
                   EnumStats* stats, const uint32_t* d_perm) {
    DevBuf U;
    const size_t m = distinct_rows(ctx, d_rows, n, k, U, d_perm);
    if (ctx.progress) ctx.progress->pairs_total = (uint64_t)m * (m + 1) / 2;
    PairSource src;  // every tile of the triangle
    DevBuf reps;
    const uint64_t c = dedup_pairs(ctx, U.as<int64_t>(), m, k, src, reps, stats);
    materialize_pairs(ctx, U.as<int64_t>(), k, reps.as<uint2>(), c, L, out);
    if (stats) {
        stats->pairs = n ? (uint64_t)n * (n - 1) / 2 : 0;
        stats->distinct_rows = m;
    }
}

void materialize_pairs(Ctx& ctx, const int64_t* d_rows, size_t k, const uint2* d_reps, uint64_t count, uint32_t L,
                       DevRows& out) {
    out.k = k;
    out.L = L;
    out.n = count;
    out.buf.alloc(std::max<uint64_t>(count * k, 1) * 8, ctx.stream);
    if (count * k)
        IGB_LAUNCH(ctx, materialize, grid_for(ctx, count * k, 256), 256, 0, d_rows, (int)k, d_reps, count, out.data());
}

uint64_t dedup_pairs(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, const PairSource& src, DevBuf& reps_out,
                     EnumStats* stats) {
    reps_out.alloc(8, ctx.stream);
    if (n == 0) return 0;
    if (n > 0xffffffffull) fail(IG_E_INVALID_ARG, "enumerate: more than 2^32 rows");
    // shared row stride: the K = 14 kernel reads rows as 16-byte words,
    // conflict-free when the stride is 2 (mod 4) words; the others read 8-byte
    // words, conflict-free with an odd stride (K = 17 with 16-byte words and
    // stride 18 measured slower: more spills)
    int stride = (int)(k | 1);
    if (k == 14) stride = 14;  // the K = 14 kernel's 16-byte loads (14 = 2 mod 4)
    int tile_rows = 64;
    while (tile_rows > 16 && (size_t)kLocalSlots * 4 + 2 * (size_t)tile_rows * stride * 8 + 3 * k * 8 > 190 * 1024)
        tile_rows /= 2;
    const uint64_t blocks = (n + tile_rows - 1) / tile_rows;
    const uint64_t n_tiles = blocks * (blocks + 1) / 2;
    const uint64_t my_tiles = src.list ? 0 : (n_tiles > src.tile_begin ? (n_tiles - src.tile_begin + src.tile_step - 1) / src.tile_step : 0);
    const uint64_t pairs = src.list ? src.n_list : (uint64_t)n * (n - 1) / 2 / src.tile_step;
    // 64-row tiles; narrower tiles for wide rows (CICIDS shape, K up to ~750) so
    // both row blocks still fit in shared memory
    const int tile = tile_rows;
    const size_t smem = (size_t)kLocalSlots * 4 + 2 * (size_t)tile * stride * 8 + 3 * k * 8;  // + keys, ORs
    if (smem > 190 * 1024) fail(IG_E_INVALID_ARG, "enumerate: rows wider than the shared-memory tile (K > 700)");
#define IGB_PAIR_ATTR(T_, K_)                                                                                 \
    IGB_SMEM_ATTR(ctx, (pair_enum<T_, K_, false>), smem);                                                 \
    IGB_SMEM_ATTR(ctx, (pair_enum<T_, K_, true>), smem)
    IGB_PAIR_ATTR(64, 0);
    IGB_PAIR_ATTR(64, 14);
    IGB_PAIR_ATTR(64, 17);
    IGB_PAIR_ATTR(32, 0);
    IGB_PAIR_ATTR(16, 0);
#undef IGB_PAIR_ATTR

    // Initial capacity from a sub-linear guess of the distinct count; doubled
    // (x4) and rerun if the table fills.  Results never depend on capacity.
    // a list source (received records) is already deduplicated per sender:
    // nearly every record is distinct
    uint64_t guess = src.list ? 2 * src.n_list + 1024
                              : (uint64_t)(4.0 * std::pow((double)(pairs + n), 0.8)) + 2 * n + 1024;
    uint64_t cap = next_pow2(std::max<uint64_t>(guess, 1u << 16));
    const uint64_t bound = src.list ? src.n_list : std::min<uint64_t>(my_tiles * (uint64_t)tile * tile, pairs * src.tile_step + n);
    const uint64_t max_cap = next_pow2(2 * bound + 1024);
    if (cap > max_cap) cap = max_cap;
    int retries = 0;
    uint64_t retry_cap = 1u << 14;  // tile-local overflow pairs (grows x8 when exceeded)
    bool retry_grow = false;
    std::vector<DevBuf> level_reps;  // per level: reps
    std::vector<uint64_t> level_counts;
    uint64_t collisions_total = 0;
    for (;;) {
        level_reps.clear();
        level_counts.clear();
        collisions_total = 0;
        bool ok = true;
        DevBuf pending;   // uint2 pairs deferred from the previous level
        uint64_t n_pending = 0;
        for (int level = 0;; ++level) {
            TableMem tm;
            const uint64_t lcap = level == 0 ? cap : next_pow2(4 * n_pending + 1024);
            const uint64_t ovf_cap = level == 0 ? std::max<uint64_t>(1u << 20, cap / 64) : n_pending + 1;
            Table T = tm.make(ctx, lcap, ovf_cap, 0x2545f4914f6cdd1dull * (uint64_t)(level + 1), k,
                              level == 0 && !src.list ? retry_cap : 1);
            if (level == 0 && src.list) {
                if (src.n_list)
                    IGB_LAUNCH(ctx, pair_insert_list, grid_for(ctx, src.n_list, 256), 256, 0, d_rows, (int)k, src.list,
                               src.n_list, T);
            } else if (level == 0) {
                const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(my_tiles, (uint64_t)ctx.sm_count * 16));
                DiagSpan dspan(ctx, kDiagEnum);
                // row projection pays off when blocks hold many rows of the same
                // prototype (C4: 1.16x faster), not on small classes (C3: 1.13x
                // slower); the results are identical either way
                const int project = n >= kProjectRows ? 1 : 0;
                static const int use_tma = getenv("IG_TMA") ? atoi(getenv("IG_TMA")) : 1;  // A/B
                unsigned long long* pc = ctx.progress ? ctx.progress->ctr : nullptr;
                unsigned long long* ph = ctx.progress ? ctx.progress->dev : nullptr;
                if (my_tiles) {
#define IGB_PAIR_ENUM(T_, K_, P_)                                                                             \
    IGB_LAUNCH(ctx, (pair_enum<T_, K_, P_>), grid, kPairThreads, smem, d_rows, (uint32_t)n, (int)k, stride,   \
               n_tiles, T, src.tile_begin, src.tile_step, pc, ph, use_tma)
#define IGB_PAIR_ENUM_P(T_, K_)          \
    if (project)                         \
        IGB_PAIR_ENUM(T_, K_, true);     \
    else                                 \
        IGB_PAIR_ENUM(T_, K_, false)
                    if (tile == 64 && k == 14) {
                        IGB_PAIR_ENUM_P(64, 14);
                    } else if (tile == 64 && k == 17) {
                        IGB_PAIR_ENUM_P(64, 17);
                    } else if (tile == 64) {
                        IGB_PAIR_ENUM_P(64, 0);
                    } else if (tile == 32) {
                        IGB_PAIR_ENUM_P(32, 0);
                    } else {
                        IGB_PAIR_ENUM_P(16, 0);
                    }
#undef IGB_PAIR_ENUM_P
#undef IGB_PAIR_ENUM
                }
                if (ctx.diag) {
                    // useful work: K word-ANDs per pair (u <= v) of this launch's tiles
                    dspan.stop();
                    uint64_t tile_pairs = 0;
                    for (uint64_t t = src.tile_begin; t < n_tiles; t += src.tile_step) {
                        uint64_t j = (uint64_t)((std::sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
                        while (j * (j + 1) / 2 > t) --j;
                        while ((j + 1) * (j + 2) / 2 <= t) ++j;
                        const uint64_t i = t - j * (j + 1) / 2;
                        const uint64_t ri = std::min<uint64_t>(tile, n - i * tile), rj = std::min<uint64_t>(tile, n - j * tile);
                        tile_pairs += i == j ? ri * (ri + 1) / 2 : ri * rj;
                    }
                    dspan.end(tile_pairs * k);
                }
            } else {
                IGB_LAUNCH(ctx, pair_insert_list, grid_for(ctx, n_pending, 256), 256, 0, d_rows, (int)k,
                           pending.as<uint2>(), n_pending, T);
            }
            if (ctx.progress) poll_progress(ctx);
            unsigned long long h[5];
            read_back(ctx, h, tm.ctr.p, sizeof(h));
            if ((h[3] & 4u) && !(h[3] & 3u)) {  // retry list too small: grow it, redo the level
                retry_cap = std::max<uint64_t>(retry_cap * 8, h[4]);
                ok = false;
                retry_grow = true;
                break;
            }
            if (h[4] && !(h[3] & 0xffffffffu)) {  // pairs the tile-local tables could not place
                IGB_LAUNCH(ctx, pair_insert_list, grid_for(ctx, h[4], 256), 256, 0, d_rows, (int)k, tm.retry.as<uint2>(),
                           h[4], T);
                read_back(ctx, h, tm.ctr.p, sizeof(h));
            }
            const int failbits = (int)(h[3] & 0xffffffffu);
            if (failbits) {
                ok = false;
                break;
            }
            level_counts.push_back(h[0]);
            collisions_total += h[2];
            level_reps.push_back(std::move(tm.reps));
            if (h[1] == 0) break;
            pending = std::move(tm.ovf);
            n_pending = h[1];
            if (level > 64) fail(IG_E_CUDA, "enumerate: fingerprint collision levels did not converge");
        }
        if (ok) break;
        if (retry_grow) {
            retry_grow = false;
            continue;
        }
        if (cap >= max_cap) fail(IG_E_OOM, "enumerate: candidate table cannot grow further");
        cap = std::min<uint64_t>(cap * 4, max_cap);
        ++retries;
    }
    uint64_t total = 0;
    for (auto c : level_counts) total += c;
    reps_out.alloc(std::max<uint64_t>(total, 1) * sizeof(uint2), ctx.stream);
    uint64_t off = 0;
    for (size_t l = 0; l < level_reps.size(); ++l) {
        const uint64_t c = level_counts[l];
        if (c)
            IGB_CUDA(cudaMemcpyAsync(reps_out.as<uint2>() + off, level_reps[l].p, c * sizeof(uint2),
                                     cudaMemcpyDeviceToDevice, ctx.stream));
        off += c;
    }
    if (stats) {
        stats->pairs = pairs;
        stats->table_slots = cap;
        stats->retries = retries;
        stats->levels = (int)level_reps.size();
        stats->collisions = collisions_total;
    }
    return total;
}

namespace {
// Owner of a candidate = its content fingerprint (unseeded, identical on every
// rank because the distinct canonical rows are) mod world.
__global__ void owner_of(const int64_t* __restrict__ X, int k, const uint2* __restrict__ reps, uint64_t n, int world,
                         const unsigned long long* __restrict__ keys, uint32_t* __restrict__ owner,
                         unsigned long long* __restrict__ counts) {
    // per-block histogram in shared memory: one global atomic per block and owner
    extern __shared__ unsigned int hist[];
    for (int r = threadIdx.x; r < world; r += blockDim.x) hist[r] = 0;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 p = reps[i];
        const int64_t* a = X + (size_t)p.x * k;
        const int64_t* b = X + (size_t)p.y * k;
        Fp fp;
        for (int w = 0; w < k; ++w) fp.add((uint64_t)(a[w] & b[w]), keys[w]);
        const uint32_t o = (uint32_t)((fp.final(k) >> 32) % (uint64_t)world);
        owner[i] = o;
        atomicAdd(hist + o, 1u);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < world; r += blockDim.x)
        if (hist[r]) atomicAdd(counts + r, (unsigned long long)hist[r]);
}
}  // namespace

void bucket_by_owner(Ctx& ctx, const int64_t* d_rows, size_t k, const uint2* d_reps, uint64_t count, int world,
                     DevBuf& send, std::vector<uint64_t>& counts) {
    counts.assign(world, 0);
    send.alloc(std::max<uint64_t>(count, 1) * sizeof(uint2), ctx.stream);
    if (count == 0) return;
    DevBuf owner(count * 4, ctx.stream), cnt(world * 8, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(cnt.p, 0, world * 8, ctx.stream));
    DevBuf keys(std::max<size_t>(k, 1) * 8, ctx.stream);
    IGB_LAUNCH(ctx, fp_keys, 1, 256, 0, kOwnerSeed, (int)k, keys.as<unsigned long long>());
    IGB_LAUNCH(ctx, owner_of, grid_for(ctx, count, 256), 256, (size_t)world * 4, d_rows, (int)k, d_reps, count, world,
               keys.as<unsigned long long>(), owner.as<uint32_t>(), cnt.as<unsigned long long>());
    // records grouped by owner: one stable radix sort on the owner id (a
    // scatter through per-owner cursors would serialise on a few hot atomics)
    int bits = 1;
    while ((1 << bits) < world) ++bits;
    DevBuf owner2(count * 4, ctx.stream);
    size_t tb = 0;
    IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, owner.as<uint32_t>(), owner2.as<uint32_t>(),
                                             reinterpret_cast<const unsigned long long*>(d_reps),
                                             send.as<unsigned long long>(), (int64_t)count, 0, bits, ctx.stream));
    DevBuf temp(tb, ctx.stream);
    IGB_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, tb, owner.as<uint32_t>(), owner2.as<uint32_t>(),
                                             reinterpret_cast<const unsigned long long*>(d_reps),
                                             send.as<unsigned long long>(), (int64_t)count, 0, bits, ctx.stream));
    read_back(ctx, counts.data(), cnt.p, world * 8);
}

int score_dev(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* d_support, int64_t* d_score) {
    if (np == 0) return IG_OK;
    DevBuf flag(sizeof(int), ctx.stream);
    IGB_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx.stream));
    IGB_LAUNCH(ctx, score_k, grid_for(ctx, np, 256), 256, 0, d_pat, np, (int)k, d_support, d_score, flag.as<int>());
    int h = 0;
    read_back(ctx, &h, flag.p, sizeof(int));
    return h ? IG_E_OVERFLOW : IG_OK;
}

// score_patterns then total_score (mine.hpp:46-51): the score kernel and the
// per-block 128-bit partial sums (plus the score overflow flag) are left in
// `buf`; score_total_collect reads them back once, when the caller's stream
// has drained anyway (the fit defers it to its end: nothing downstream needs
// the total on the host).
unsigned score_total_launch(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* d_support,
                            int64_t* d_score, DevBuf& buf) {
    if (np == 0) return 0;
    const unsigned g = std::min<unsigned>(grid_for(ctx, np, 256), 1024);
    buf.alloc((2 * (size_t)g + 1) * 8, ctx.stream);
    unsigned long long* lo = buf.as<unsigned long long>();
    long long* hi = reinterpret_cast<long long*>(lo + g);
    int* flag = reinterpret_cast<int*>(lo + 2 * g);
    IGB_CUDA(cudaMemsetAsync(flag, 0, 8, ctx.stream));
    IGB_LAUNCH(ctx, score_k, grid_for(ctx, np, 256), 256, 0, d_pat, np, (int)k, d_support, d_score, flag);
    IGB_LAUNCH(ctx, sum128, g, 256, 0, d_score, np, lo, hi);
    return g;
}

int score_total_collect(Ctx& ctx, const DevBuf& buf, unsigned g, int64_t* total) {
    *total = 0;
    if (g == 0) return IG_OK;
    std::vector<unsigned long long> h(2 * (size_t)g + 1);
    read_back(ctx, h.data(), buf.p, h.size() * 8);
    if (*reinterpret_cast<const int*>(&h[2 * g])) return IG_E_OVERFLOW;
    __int128 acc = 0;
    for (unsigned i = 0; i < g; ++i) acc += ((__int128)(long long)h[g + i] << 32) + (__int128)h[i];
    if (acc > (__int128)INT64_MAX || acc < (__int128)INT64_MIN) return IG_E_OVERFLOW;
    *total = (int64_t)acc;
    return IG_OK;
}

int score_total_dev(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* d_support, int64_t* d_score,
                    int64_t* total) {
    DevBuf buf;
    const unsigned g = score_total_launch(ctx, d_pat, np, k, d_support, d_score, buf);
    return score_total_collect(ctx, buf, g, total);
}

int total_score_dev(Ctx& ctx, const int64_t* d_score, size_t np, int64_t* total) {
    *total = 0;
    if (np == 0) return IG_OK;
    const unsigned g = std::min<unsigned>(grid_for(ctx, np, 256), 1024);
    DevBuf lo(g * 8, ctx.stream), hi(g * 8, ctx.stream);
    IGB_LAUNCH(ctx, sum128, g, 256, 0, d_score, np, lo.as<unsigned long long>(), hi.as<long long>());
    std::vector<unsigned long long> hl(2 * (size_t)g);
    read_back(ctx, hl.data(), lo.p, g * 8);
    read_back(ctx, hl.data() + g, hi.p, g * 8);
    __int128 acc = 0;
    for (unsigned i = 0; i < g; ++i) acc += ((__int128)(long long)hl[g + i] << 32) + (__int128)hl[i];
    // Scores are non-negative (support >= 0), so the running-sum overflow of
    // total_score (mine.hpp:50-51) happens iff the exact total exceeds INT64_MAX.
    if (acc > (__int128)INT64_MAX || acc < (__int128)INT64_MIN) return IG_E_OVERFLOW;
    *total = (int64_t)acc;
    return IG_OK;
}

namespace {
__global__ void flag_to_keep(const uint8_t* f, size_t n, uint8_t* keep) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        keep[i] = f[i] ? 0 : 1;
}
__global__ void compact_rows_k(const int64_t* __restrict__ src, const uint32_t* __restrict__ idx, size_t m, int k,
                               int64_t* __restrict__ dst) {
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < m * k; q += (size_t)gridDim.x * blockDim.x)
        dst[q] = src[(size_t)idx[q / k] * k + q % k];
}
}  // namespace

size_t compact_unflagged(Ctx& ctx, const int64_t* d_words, const int64_t* d_sup, const int64_t* d_sc,
                         const uint8_t* d_flag, size_t n, size_t k, int64_t* o_words, int64_t* o_sup,
                         int64_t* o_sc, DevBuf* o_idx) {
    if (n == 0) return 0;
    DevBuf keep(n, ctx.stream), idx(n * 4, ctx.stream), nsel(8, ctx.stream), iota(n * 4, ctx.stream);
    IGB_LAUNCH(ctx, flag_to_keep, grid_for(ctx, n, 256), 256, 0, d_flag, n, keep.as<uint8_t>());
    IGB_LAUNCH(ctx, iota_u32, grid_for(ctx, n, 256), 256, 0, iota.as<uint32_t>(), n);
    size_t tb = 0;
    IGB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.as<uint32_t>(), keep.as<uint8_t>(), idx.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)n, ctx.stream));
    DevBuf temp(tb, ctx.stream);
    IGB_CUDA(cub::DeviceSelect::Flagged(temp.p, tb, iota.as<uint32_t>(), keep.as<uint8_t>(), idx.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)n, ctx.stream));
    int64_t m = 0;
    read_back(ctx, &m, nsel.p, 8);
    if (m) {
        IGB_LAUNCH(ctx, compact_rows_k, grid_for(ctx, m * k, 256), 256, 0, d_words, idx.as<uint32_t>(), (size_t)m,
                   (int)k, o_words);
        if (d_sup) IGB_LAUNCH(ctx, gather_i64, grid_for(ctx, m, 256), 256, 0, d_sup, idx.as<uint32_t>(), (size_t)m, o_sup);
        if (d_sc) IGB_LAUNCH(ctx, gather_i64, grid_for(ctx, m, 256), 256, 0, d_sc, idx.as<uint32_t>(), (size_t)m, o_sc);
    }
    if (o_idx) *o_idx = std::move(idx);
    return (size_t)m;
}

}  // namespace igb
