// sort.cu — canonical (words::less, bitpack.hpp:59-68) ordering of K-word rows
// with rank-compressed keys.
//
// Lexicographic order over K unsigned 64-bit words only depends on the order of
// the values inside each word column.  Each column of a candidate / pattern set
// takes few distinct values (C3 pure dictionaries: 63..1,970 per column, ~135
// bits of dense ranks for all 14 words), so every word is replaced by its dense
// rank among the column's distinct values and the ranks are packed MSB-first
// into ceil(B/64) 64-bit keys.  One stable radix sort per packed key word
// (LSD) then yields exactly the canonical order, with ~B/8 radix digit passes
// instead of 8·K.  Distinct values are found with one open-addressing hash set
// per column (16-byte slots claimed by a 128-bit CAS), ranked by sorting the
// (column, value) list, and written back into the slots.  Falls back to the
// K-pass LSD sort when the tables would be too large.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "ig_internal.cuh"

namespace igb {
namespace {

unsigned grid_for(const Ctx& ctx, size_t work, int threads) {
    size_t g = (work + threads - 1) / threads;
    const size_t cap = (size_t)ctx.sm_count * 32;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

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


// slot = {value, tag}; tag 0 = empty, 1 = present, 2 + rank after ranking.
__global__ void column_insert(const int64_t* __restrict__ words, size_t n, int k, ulonglong2* __restrict__ tables,
                              uint32_t slots, unsigned int* __restrict__ counts, int* __restrict__ full) {
    const size_t total = n * (size_t)k;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const int w = (int)(q % k);
        const unsigned long long v = (unsigned long long)words[q];
        ulonglong2* T = tables + (size_t)w * slots;
        uint32_t s = (uint32_t)(mix64(v) & (slots - 1));
        for (uint32_t probe = 0;; ++probe, s = (s + 1) & (slots - 1)) {
            if (probe >= slots) {
                atomicOr(full, 1);
                return;
            }
            // plain (L1-cacheable) reads: popular values would otherwise hammer
            // one L2 line per column.  A slot changes once, {0,0} -> {v,1}, by
            // a 128-bit CAS, so a stale read can only show it empty (the CAS
            // below then returns the real content) and a non-zero tag always
            // comes with its value.
            ulonglong2 e;  // one 16-byte load (value and tag from the same snapshot)
            asm("ld.global.v2.u64 {%0, %1}, [%2];" : "=l"(e.x), "=l"(e.y) : "l"(T + s));
            if (e.y == 0) {
                const ulonglong2 old = cas128(T + s, make_ulonglong2(0ull, 0ull), make_ulonglong2(v, 1ull));
                if (old.y == 0) {
                    // load check only on the (rare) insert path: past half load the
                    // host retries with a larger table
                    if (atomicAdd(counts + w, 1u) + 1 >= slots / 2) atomicOr(full, 1);
                    break;
                }
                if (old.x == v) break;
                continue;
            }
            if (e.x == v) break;
        }
    }
}

// Occupied slots -> (column, value, slot) entries.
__global__ void column_collect(const ulonglong2* __restrict__ tables, int k, uint32_t slots,
                               unsigned long long* __restrict__ vals, uint32_t* __restrict__ where,
                               unsigned int* __restrict__ n_out) {
    const size_t total = (size_t)k * slots;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const ulonglong2 e = tables[q];
        if (e.y != 0) {
            const unsigned int o = atomicAdd(n_out, 1u);
            vals[o] = e.x;
            where[o] = (uint32_t)q;
        }
    }
}

__global__ void column_of(const uint32_t* __restrict__ where, size_t m, uint32_t slots, uint32_t* __restrict__ col) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x)
        col[i] = where[i] / slots;
}

// After sorting entries by (column, value): rank = position - column start.
__global__ void write_ranks(const uint32_t* __restrict__ where, size_t m, uint32_t slots,
                            const unsigned int* __restrict__ col_start, ulonglong2* __restrict__ tables) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (size_t)gridDim.x * blockDim.x) {
        const uint32_t q = where[i];
        const uint32_t w = q / slots;
        tables[q].y = 2ull + (i - col_start[w]);
    }
}

// Small columns (every column <= kRankSmall distinct values): per-column
// segments of the distinct values, then each value's rank = #smaller values
// of its column, counted against the column staged in shared memory.
constexpr uint32_t kRankSmall = 4096;
constexpr int kParamCols = 64;  // small per-column tables travel as kernel parameters
struct Starts {
    unsigned int v[kParamCols + 1];
};

__global__ void init_cursor(Starts st, int k, unsigned int* __restrict__ cursor) {
    for (int w = threadIdx.x; w <= k; w += blockDim.x) cursor[w] = st.v[w];
}
__global__ void column_collect_seg(const ulonglong2* __restrict__ tables, int k, uint32_t slots,
                                   unsigned int* __restrict__ cursor, unsigned long long* __restrict__ vals,
                                   uint32_t* __restrict__ where) {
    const size_t total = (size_t)k * slots;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const ulonglong2 e = tables[q];
        if (e.y != 0) {
            const unsigned int o = atomicAdd(cursor + q / slots, 1u);
            vals[o] = e.x;
            where[o] = (uint32_t)q;
        }
    }
}

__global__ void column_rank_small(const unsigned long long* __restrict__ vals, const uint32_t* __restrict__ where,
                                  Starts st, ulonglong2* __restrict__ tables) {
    __shared__ unsigned long long sv[kRankSmall];
    const int w = blockIdx.x;
    const uint32_t b = st.v[w], d = st.v[w + 1] - b;
    const uint32_t i = blockIdx.y * blockDim.x + threadIdx.x;
    if (blockIdx.y * blockDim.x >= d) return;  // whole block past this column (uniform)
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) sv[j] = vals[b + j];
    __syncthreads();
    if (i >= d) return;
    const unsigned long long v = sv[i];
    uint32_t r = 0;
    for (uint32_t j = 0; j < d; ++j) r += sv[j] < v ? 1u : 0u;
    tables[where[b + i]].y = 2ull + r;
}

struct Field {
    int key;    // packed key word
    int shift;  // bit position of the field's LSB inside that key word
};
struct FieldTable {
    Field f[kParamCols];
};

// Packed keys, MSB-first by word: keys[j][i] for key word j of row i.
__global__ void pack_keys(const int64_t* __restrict__ words, size_t n, int k, const ulonglong2* __restrict__ tables,
                          uint32_t slots, const Field* __restrict__ fields, FieldTable ft, int n_keys,
                          unsigned long long* __restrict__ keys) {
    // fields are laid out in word order, so the key words fill one after another
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned long long cur = 0;
        int ck = 0;
        for (int w = 0; w < k; ++w) {
            const unsigned long long v = (unsigned long long)words[i * k + w];
            const ulonglong2* T = tables + (size_t)w * slots;
            uint32_t s = (uint32_t)(mix64(v) & (slots - 1));
            while (T[s].x != v || T[s].y == 0) s = (s + 1) & (slots - 1);
            const unsigned long long r = T[s].y - 2;
            const Field f = fields ? fields[w] : ft.f[w];
            if (f.key != ck) {
                keys[(size_t)ck * n + i] = cur;
                cur = 0;
                ck = f.key;
            }
            cur |= r << f.shift;
        }
        keys[(size_t)ck * n + i] = cur;
        (void)n_keys;
    }
}

__global__ void iota32(uint32_t* p, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

__global__ void gather_u64(const unsigned long long* __restrict__ src, const uint32_t* __restrict__ perm, size_t n,
                           unsigned long long* __restrict__ dst) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[perm[i]];
}

__global__ void row_heads_k(const int64_t* __restrict__ rows, const uint32_t* __restrict__ perm, size_t n, int k,
                            uint8_t* __restrict__ head) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint8_t h = 1;
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

__global__ void gather_rows_u32(const int64_t* __restrict__ src, const uint32_t* __restrict__ idx, size_t m, int k,
                                int64_t* __restrict__ dst) {
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < m * k; q += (size_t)gridDim.x * blockDim.x)
        dst[q] = src[(size_t)idx[q / k] * k + q % k];
}

// Small sets (n <= kSmallSort): exact stable rank by counting, one launch.
// rank(i) = #{j : row_j < row_i} + #{j < i : row_j == row_i}; thread i keeps its
// row in registers and streams 128-row chunks of the j range through shared
// memory (warp-broadcast reads).  blockIdx.y splits the j range so that even a
// few thousand rows fill every SM; partial counts meet in rank[] by atomics.
constexpr uint32_t kSmallSort = 24576;
constexpr int kRankChunk = 128;
template <int KMAX>
__global__ void __launch_bounds__(kRankChunk)
rank_by_count(const int64_t* __restrict__ rows, uint32_t n, int k, uint32_t j_per_split, uint32_t* __restrict__ rank) {
    __shared__ unsigned long long sj[kRankChunk * KMAX];
    const uint32_t i = blockIdx.x * kRankChunk + threadIdx.x;
    unsigned long long r[KMAX];
#pragma unroll
    for (int w = 0; w < KMAX; ++w) r[w] = (i < n && w < k) ? (unsigned long long)rows[(size_t)i * k + w] : 0ull;
    const uint32_t jb = blockIdx.y * j_per_split, je = min(n, jb + j_per_split);
    uint32_t cnt = 0;
    for (uint32_t j0 = jb; j0 < je; j0 += kRankChunk) {
        const uint32_t m = min((uint32_t)kRankChunk, je - j0);
        __syncthreads();
        for (uint32_t q = threadIdx.x; q < m * (uint32_t)k; q += kRankChunk)
            sj[(q / k) * KMAX + q % k] = (unsigned long long)rows[(size_t)j0 * k + q];
        __syncthreads();
        for (uint32_t jj = 0; jj < m; ++jj) {
            const unsigned long long* b = sj + jj * KMAX;
            int cmp = 0;  // -1: row_j < row_i, 1: row_j > row_i
#pragma unroll
            for (int w = 0; w < KMAX; ++w) {
                if (w >= k) break;
                const unsigned long long x = b[w];
                if (x != r[w]) {
                    cmp = x < r[w] ? -1 : 1;
                    break;
                }
            }
            cnt += (cmp < 0 || (cmp == 0 && j0 + jj < i)) ? 1u : 0u;
        }
    }
    if (i < n) atomicAdd(rank + i, cnt);
}

__global__ void perm_from_rank(const uint32_t* __restrict__ rank, uint32_t n, uint32_t* __restrict__ perm) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) perm[rank[i]] = i;
}

__global__ void keys_to_rows(const unsigned long long* __restrict__ keys, size_t n, int n_keys,
                             int64_t* __restrict__ rows) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        for (int j = 0; j < n_keys; ++j) rows[i * n_keys + j] = (int64_t)keys[(size_t)j * n + i];
}

// perm = stable canonical order of n rows of k words (k <= 32) by counting
void count_sort_rows(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, uint32_t* d_perm) {
    DevBuf rank(n * 4, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(rank.p, 0, n * 4, ctx.stream));
    const uint32_t bx = (uint32_t)((n + kRankChunk - 1) / kRankChunk);
    // split j so that bx * by covers ~16 CTAs (64 warps) per SM, in whole
    // chunks: the compare loop is latency-bound (4 CTAs per SM: 80 us for
    // 7,000 rows at C3)
    uint32_t by = std::max<uint32_t>(1, (uint32_t)(16 * ctx.sm_count) / bx);
    uint32_t per = (uint32_t)((n + by - 1) / by);
    per = (per + kRankChunk - 1) / kRankChunk * kRankChunk;
    by = (uint32_t)((n + per - 1) / per);
    const dim3 grid(bx, by);
    if (k <= 8)
        IGB_LAUNCH(ctx, rank_by_count<8>, grid, kRankChunk, 0, d_rows, (uint32_t)n, (int)k, per, rank.as<uint32_t>());
    else if (k <= 16)
        IGB_LAUNCH(ctx, rank_by_count<16>, grid, kRankChunk, 0, d_rows, (uint32_t)n, (int)k, per, rank.as<uint32_t>());
    else
        IGB_LAUNCH(ctx, rank_by_count<32>, grid, kRankChunk, 0, d_rows, (uint32_t)n, (int)k, per, rank.as<uint32_t>());
    IGB_LAUNCH(ctx, perm_from_rank, grid_for(ctx, n, 256), 256, 0, rank.as<uint32_t>(), (uint32_t)n, d_perm);
}

uint32_t next_pow2_u32(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return (uint32_t)p;
}

}  // namespace

void sort_rows_canonical(Ctx& ctx, const int64_t* d_words, size_t n, size_t k, uint32_t* d_perm) {
    if (n == 0) return;
    if (n == 1 || k == 0) {
        IGB_LAUNCH(ctx, iota32, 1, 32, 0, d_perm, n);
        return;
    }
    Trace tr(ctx, "sort_rows", -1);
    // Per-column hash sets; start small (columns usually hold a few thousand
    // distinct words) and grow x16 when a column passes half load.
    uint32_t slots = next_pow2_u32(std::min<uint64_t>(2 * n + 16, 1ull << 16));
    DevBuf tables, counts((k + 2) * 4, ctx.stream);  // per column counts, then the full flag
    std::vector<unsigned int> hc(k + 2);
    for (;;) {
        if ((uint64_t)slots * k * 16 > (1ull << 31) || k > 512) {
            sort_rows_canonical_lsd(ctx, d_words, n, k, d_perm);
            return;
        }
        tables.alloc((size_t)slots * k * 16, ctx.stream);
        IGB_CUDA(cudaMemsetAsync(tables.p, 0, (size_t)slots * k * 16, ctx.stream));
        IGB_CUDA(cudaMemsetAsync(counts.p, 0, (k + 2) * 4, ctx.stream));
        IGB_LAUNCH(ctx, column_insert, grid_for(ctx, n * k, 256), 256, 0, d_words, n, (int)k, tables.as<ulonglong2>(),
                   slots, counts.as<unsigned int>(), reinterpret_cast<int*>(counts.as<unsigned int>() + k + 1));
        read_back(ctx, hc.data(), counts.p, (k + 2) * 4);  // counts and the full flag in one read-back
        const int hfull = (int)hc[k + 1];
        if (!hfull) break;
        if (slots >= (1u << 20) || slots >= 2 * n + 16) {
            sort_rows_canonical_lsd(ctx, d_words, n, k, d_perm);
            return;
        }
        slots *= 16;
    }
    // Field layout: ceil(log2 D_w) bits per word, MSB-first, never straddling a key word.
    std::vector<Field> fields(k);
    int n_keys = 1, used = 0;
    std::vector<int> used_bits;
    for (size_t w = 0; w < k; ++w) {
        int b = 1;
        while ((1ull << b) < hc[w]) ++b;
        if (used + b > 64) {
            used_bits.push_back(used);
            ++n_keys;
            used = 0;
        }
        fields[w].key = n_keys - 1;
        used += b;
        fields[w].shift = 64 - used;
    }
    used_bits.push_back(used);
    if (n_keys > 48 || n_keys >= (int)k) {
        sort_rows_canonical_lsd(ctx, d_words, n, k, d_perm);
        return;
    }
    tr.mark("column_hash");
    // Rank the distinct values of every column.
    uint64_t m = 0;
    uint32_t dmax = 0;
    for (size_t w = 0; w < k; ++w) {
        m += hc[w];
        dmax = std::max<uint32_t>(dmax, hc[w]);
    }
    if (dmax <= kRankSmall && k <= (size_t)kParamCols) {
        // no host->device copies here: they would queue behind a caller's
        // bulk prefetch on the copy engine
        Starts st{};
        for (size_t w = 0; w < k; ++w) st.v[w + 1] = st.v[w] + hc[w];
        DevBuf vals(m * 8, ctx.stream), where(m * 4, ctx.stream), cursor((k + 1) * 4, ctx.stream);
        IGB_LAUNCH(ctx, init_cursor, 1, 128, 0, st, (int)k, cursor.as<unsigned int>());
        IGB_LAUNCH(ctx, column_collect_seg, grid_for(ctx, (size_t)k * slots, 256), 256, 0, tables.as<ulonglong2>(),
                   (int)k, slots, cursor.as<unsigned int>(), vals.as<unsigned long long>(), where.as<uint32_t>());
        const dim3 grid((unsigned)k, (dmax + 255) / 256);
        IGB_LAUNCH(ctx, column_rank_small, grid, 256, 0, vals.as<unsigned long long>(), where.as<uint32_t>(), st,
                   tables.as<ulonglong2>());
    } else {
        DevBuf vals(m * 8, ctx.stream), vals2(m * 8, ctx.stream), where(m * 4, ctx.stream), where2(m * 4, ctx.stream),
            col(m * 4, ctx.stream), col2(m * 4, ctx.stream), nout(4, ctx.stream), cstart((k + 1) * 4, ctx.stream);
        IGB_CUDA(cudaMemsetAsync(nout.p, 0, 4, ctx.stream));
        IGB_LAUNCH(ctx, column_collect, grid_for(ctx, (size_t)k * slots, 256), 256, 0, tables.as<ulonglong2>(), (int)k,
                   slots, vals.as<unsigned long long>(), where.as<uint32_t>(), nout.as<unsigned int>());
        size_t tb1 = 0, tb2 = 0;
        IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb1, vals.as<unsigned long long>(),
                                                 vals2.as<unsigned long long>(), where.as<uint32_t>(),
                                                 where2.as<uint32_t>(), (int64_t)m, 0, 64, ctx.stream));
        IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, col.as<uint32_t>(), col2.as<uint32_t>(),
                                                 where2.as<uint32_t>(), where.as<uint32_t>(), (int64_t)m, 0, 32,
                                                 ctx.stream));
        DevBuf temp(std::max(tb1, tb2), ctx.stream);
        IGB_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, tb1, vals.as<unsigned long long>(),
                                                 vals2.as<unsigned long long>(), where.as<uint32_t>(),
                                                 where2.as<uint32_t>(), (int64_t)m, 0, 64, ctx.stream));
        IGB_LAUNCH(ctx, column_of, grid_for(ctx, m, 256), 256, 0, where2.as<uint32_t>(), m, slots, col.as<uint32_t>());
        int cbits = 1;
        while ((1ull << cbits) < k) ++cbits;
        IGB_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, tb2, col.as<uint32_t>(), col2.as<uint32_t>(),
                                                 where2.as<uint32_t>(), where.as<uint32_t>(), (int64_t)m, 0, cbits,
                                                 ctx.stream));
        std::vector<unsigned int> hstart(k + 1, 0);
        for (size_t w = 0; w < k; ++w) hstart[w + 1] = hstart[w] + hc[w];
        IGB_CUDA(cudaMemcpyAsync(cstart.p, hstart.data(), (k + 1) * 4, cudaMemcpyHostToDevice, ctx.stream));
        IGB_LAUNCH(ctx, write_ranks, grid_for(ctx, m, 256), 256, 0, where.as<uint32_t>(), m, slots,
                   cstart.as<unsigned int>(), tables.as<ulonglong2>());
    }
    tr.mark("column_ranks");
    // Packed keys and LSD over the key words (least significant word first).
    DevBuf dfields, keys((size_t)n_keys * n * 8, ctx.stream);
    FieldTable ft{};
    if (k <= (size_t)kParamCols) {
        for (size_t w = 0; w < k; ++w) ft.f[w] = fields[w];
    } else {
        dfields.alloc(k * sizeof(Field), ctx.stream);
        IGB_CUDA(cudaMemcpyAsync(dfields.p, fields.data(), k * sizeof(Field), cudaMemcpyHostToDevice, ctx.stream));
    }
    IGB_LAUNCH(ctx, pack_keys, grid_for(ctx, n, 128), 128, 0, d_words, n, (int)k, tables.as<ulonglong2>(), slots,
               dfields.p ? dfields.as<Field>() : nullptr, ft, n_keys, keys.as<unsigned long long>());
    if (n <= kSmallSort && n_keys <= 32) {
        // few rows: rank by counting on the packed keys (<= 8 words, most
        // comparisons end at the first) instead of ~B/8 launch-bound radix passes
        DevBuf krows(n * n_keys * 8, ctx.stream);
        IGB_LAUNCH(ctx, keys_to_rows, grid_for(ctx, n, 256), 256, 0, keys.as<unsigned long long>(), n, n_keys,
                   krows.as<int64_t>());
        count_sort_rows(ctx, krows.as<int64_t>(), n, (size_t)n_keys, d_perm);
        tr.mark("count_keys");
        return;
    }
    DevBuf k1(n * 8, ctx.stream), k2(n * 8, ctx.stream), p2(n * 4, ctx.stream);
    IGB_LAUNCH(ctx, iota32, grid_for(ctx, n, 256), 256, 0, d_perm, n);
    size_t tb3 = 0;
    IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb3, k1.as<unsigned long long>(), k2.as<unsigned long long>(),
                                             d_perm, p2.as<uint32_t>(), (int64_t)n, 0, 64, ctx.stream));
    DevBuf temp3(tb3, ctx.stream);
    uint32_t* cur = d_perm;
    uint32_t* alt = p2.as<uint32_t>();
    for (int j = n_keys - 1; j >= 0; --j) {
        const unsigned long long* kj = keys.as<unsigned long long>() + (size_t)j * n;
        if (j == n_keys - 1) {
            IGB_CUDA(cudaMemcpyAsync(k1.p, kj, n * 8, cudaMemcpyDeviceToDevice, ctx.stream));
        } else {
            IGB_LAUNCH(ctx, gather_u64, grid_for(ctx, n, 256), 256, 0, kj, cur, n, k1.as<unsigned long long>());
        }
        const int begin = 64 - used_bits[j];
        IGB_CUDA(cub::DeviceRadixSort::SortPairs(temp3.p, tb3, k1.as<unsigned long long>(),
                                                 k2.as<unsigned long long>(), cur, alt, (int64_t)n, begin, 64,
                                                 ctx.stream));
        std::swap(cur, alt);
    }
    if (cur != d_perm) IGB_CUDA(cudaMemcpyAsync(d_perm, cur, n * 4, cudaMemcpyDeviceToDevice, ctx.stream));
    if (tr.on) {
        int bits = 0;
        for (int b : used_bits) bits += b;
        fprintf(stderr, "[ig trace] sort_rows n=%zu k=%zu keys=%d bits=%d\n", n, k, n_keys, bits);
    }
    tr.mark("lsd");
}

size_t distinct_rows(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, DevBuf& out, const uint32_t* d_perm,
                     DevBuf* o_perm) {
    if (n == 0) {
        out.alloc(8, ctx.stream);
        return 0;
    }
    DevBuf perm(n * 4, ctx.stream), head(n, ctx.stream), rep(n * 4, ctx.stream), nsel(8, ctx.stream);
    if (d_perm)
        IGB_CUDA(cudaMemcpyAsync(perm.p, d_perm, n * 4, cudaMemcpyDeviceToDevice, ctx.stream));
    else
        sort_rows_canonical(ctx, d_rows, n, k, perm.as<uint32_t>());
    IGB_LAUNCH(ctx, row_heads_k, grid_for(ctx, n, 256), 256, 0, d_rows, perm.as<uint32_t>(), n, (int)k,
               head.as<uint8_t>());
    size_t tb = 0;
    IGB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, perm.as<uint32_t>(), head.as<uint8_t>(), rep.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)n, ctx.stream));
    DevBuf temp(tb, ctx.stream);
    IGB_CUDA(cub::DeviceSelect::Flagged(temp.p, tb, perm.as<uint32_t>(), head.as<uint8_t>(), rep.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)n, ctx.stream));
    int64_t m = 0;
    read_back(ctx, &m, nsel.p, 8);
    out.alloc(std::max<size_t>((size_t)m * k, 1) * 8, ctx.stream);
    IGB_LAUNCH(ctx, gather_rows_u32, grid_for(ctx, (size_t)m * k, 256), 256, 0, d_rows, rep.as<uint32_t>(), (size_t)m,
               (int)k, out.as<int64_t>());
    if (o_perm) *o_perm = std::move(perm);
    return (size_t)m;
}

}  // namespace igb
