// ingest.cu — device CSV ingest: CSV bytes -> the
// schema (kind, mean, population std over the training rows) and the typed
// train / test columns, resident in HBM; the same result as the host path
// read_csv -> slice -> infer_schema -> build_columns (csv.cpp:14-89,
// pipeline.cpp:35-49,107-193), which remains the path for inputs this one does
// not take (quoted fields, a header with quotes).
//
// Exactness, piece by piece:
// * records: '\n', "\r\n" and a lone '\r' end a record, a trailing terminator
//   adds none, a final unterminated record counts if non-empty; every record
//   must have the header's field count (the host reader's DataError).
// * numbers: a cell is parsed on the device only when the result is certainly
//   std::from_chars's: [-]digits[.digits][(e|E)[+|-]digits] with <= 15
//   significant digits and a decimal exponent within +-22 after dropping
//   trailing zeros, i.e. one correctly rounded IEEE multiply or divide of two
//   exact doubles (Clinger's fast path).  Any other cell that could still be a
//   number goes back to the host's from_chars; everything else is text.
// * statistics: one warp per numeric column streams the training rows and lane
//   0 adds them in row order (sum, then sum of squared deviations) with _rn
//   intrinsics, exactly the host's sequential double sums; the squared
//   deviations accumulate as fma(d, d, ss), the rounding of the reference's
//   -march=native build (GCC contracts pipeline.cpp:159); sqrt is _rn.
// * categorical ids and the label mapping follow first appearance in row
//   order (an exact-content hash table records each string's first row), as
//   build_columns assigns them.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "encode.cuh"
#include "host_pipeline.hpp"
#include "ig_internal.cuh"

namespace igb {
namespace {

enum : uint8_t { kEmpty = 0, kNum = 1, kHost = 2, kText = 3 };

unsigned grid_for(const Ctx& ctx, size_t work, int threads) {
    size_t g = (work + threads - 1) / threads;
    const size_t cap = (size_t)ctx.sm_count * 32;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}


// terminator positions in [from, n) (order-preserving compaction) + quote flag.
// Each thread takes 16 aligned bytes per step (one 16-byte load; the byte
// after them for a '\r' at the end); bit j of ends16 = byte j ends a record.
__device__ __forceinline__ uint32_t ends16(const char* __restrict__ b, size_t n, size_t from, size_t lo, size_t hi,
                                          size_t p, bool& quote) {
    // p: 16-aligned position; bytes outside [max(lo, from), min(hi, n)) do not count
    uint4 v = make_uint4(0, 0, 0, 0);
    if (p + 16 <= n) {
        v = *reinterpret_cast<const uint4*>(b + p);
    } else {
        unsigned char t[16] = {0};
        for (int j = 0; j < 16; ++j)
            if (p + j < n) t[j] = (unsigned char)b[p + j];
        memcpy(&v, t, 16);
    }
    const unsigned char* c = reinterpret_cast<const unsigned char*>(&v);
    const unsigned char next = p + 16 < n ? (unsigned char)b[p + 16] : 0;
    uint32_t m = 0;
    const size_t a0 = max(lo, from), a1 = min(hi, n);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const size_t i = p + j;
        if (i < a0 || i >= a1) continue;
        const unsigned char ch = c[j];
        const unsigned char nx = j + 1 < 16 ? c[j + 1] : next;
        const bool last = i + 1 == n;
        if (ch == '\n' || (ch == '\r' && (last || nx != '\n'))) m |= 1u << j;
        quote |= ch == '"';
    }
    return m;
}

__global__ void mark_ends(const char* __restrict__ b, size_t n, size_t from, uint32_t* __restrict__ cnt_block,
                          int* __restrict__ quote) {
    // pass 1: count per block
    __shared__ uint32_t sc;
    if (threadIdx.x == 0) sc = 0;
    __syncthreads();
    const size_t chunk = (((n - from) + gridDim.x - 1) / gridDim.x + 15) & ~size_t{15};
    const size_t lo = from + (size_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
    uint32_t c = 0;
    bool q = false;
    for (size_t p = (lo & ~size_t{15}) + 16 * threadIdx.x; p < hi; p += 16 * (size_t)blockDim.x)
        c += __popc(ends16(b, n, from, lo, hi, p, q));
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&sc, c);
    if (q) atomicOr(quote, 1);
    __syncthreads();
    if (threadIdx.x == 0) cnt_block[blockIdx.x] = sc;
}

__global__ void write_ends(const char* __restrict__ b, size_t n, size_t from, const uint32_t* __restrict__ off_block,
                           uint32_t* __restrict__ ends) {
    // pass 2: ordered positions inside each block chunk (block prefix of the
    // per-thread counts, serial over the chunk in 16-byte steps)
    const size_t chunk = (((n - from) + gridDim.x - 1) / gridDim.x + 15) & ~size_t{15};
    const size_t lo = from + (size_t)blockIdx.x * chunk, hi = min(n, lo + chunk);
    __shared__ uint32_t warp_cnt[32];
    __shared__ uint32_t base;
    if (threadIdx.x == 0) base = off_block[blockIdx.x];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    bool q = false;
    for (size_t p0 = lo & ~size_t{15}; p0 < hi; p0 += 16 * (size_t)blockDim.x) {
        const size_t p = p0 + 16 * threadIdx.x;
        const uint32_t m = p < hi ? ends16(b, n, from, lo, hi, p, q) : 0u;
        const uint32_t c = __popc(m);
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_cnt[wid] = incl;
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (int w = 0; w < nw; ++w) {
            if (w < wid) before += warp_cnt[w];
            total += warp_cnt[w];
        }
        uint32_t pos = base + before + incl - c;
        for (uint32_t mm = m; mm; mm &= mm - 1) ends[pos++] = (uint32_t)(p + __ffs(mm) - 1);
        __syncthreads();
        if (threadIdx.x == 0) base += total;
        __syncthreads();
    }
}

struct Records {
    const uint32_t* ends;
    uint32_t m;       // terminators
    uint32_t body;    // first byte after the header record
    uint32_t n_bytes;
    bool tail;        // a non-empty unterminated last record
};

__device__ __forceinline__ void record_span(const char* b, const Records& R, uint32_t r, uint32_t& s, uint32_t& e) {
    s = r == 0 ? R.body : R.ends[r - 1] + 1;
    e = r < R.m ? R.ends[r] : R.n_bytes;
    if (r < R.m && b[e] == '\n' && e > s && b[e - 1] == '\r') --e;  // CRLF
}

// Warp per record: field starts beg[r*(C+1)+f], beg[..+C] = end + 1.
__global__ void split_fields(const char* __restrict__ b, Records R, uint32_t n_rec, int C, uint32_t* __restrict__ beg,
                             unsigned long long* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    const size_t warps = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t r = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_rec; r += warps) {
        uint32_t s, e;
        record_span(b, R, (uint32_t)r, s, e);
        uint32_t* out = beg + r * (size_t)(C + 1);
        uint32_t f = 0;
        for (uint32_t base = s; base < e; base += 32) {
            const uint32_t i = base + lane;
            const bool comma = i < e && b[i] == ',';
            const uint32_t m = __ballot_sync(0xffffffffu, comma);
            if (comma) {
                const uint32_t k = f + 1 + __popc(m & ((1u << lane) - 1u));
                if (k < (uint32_t)C) out[k] = i + 1;
            }
            f += __popc(m);
        }
        if (lane == 0) {
            out[0] = s;
            out[C] = e + 1;
            if (f + 1 != (uint32_t)C) atomicMin(bad, ((unsigned long long)r << 32) | (f + 1));
        }
    }
}

__constant__ double kPow10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                  1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

__device__ uint8_t parse_cell(const char* s, int len, double* out) {
    if (len == 0) return kEmpty;
    int i = 0;
    bool neg = false;
    if (s[0] == '-') {
        neg = true;
        i = 1;
    }
    uint64_t w = 0;
    int sig = 0, dexp = 0;
    bool any = false, inexact = false;
    for (; i < len && s[i] >= '0' && s[i] <= '9'; ++i) {
        const int d = s[i] - '0';
        any = true;
        if (w == 0 && d == 0) continue;  // leading zero
        if (sig < 19) {
            w = w * 10 + d;
            ++sig;
        } else {
            ++dexp;
            inexact |= d != 0;
        }
    }
    if (i < len && s[i] == '.') {
        ++i;
        for (; i < len && s[i] >= '0' && s[i] <= '9'; ++i) {
            const int d = s[i] - '0';
            any = true;
            if (w == 0 && d == 0) {
                --dexp;
                continue;
            }
            if (sig < 19) {
                w = w * 10 + d;
                ++sig;
                --dexp;
            } else {
                inexact |= d != 0;
            }
        }
    }
    if (!any) return kText;  // "", "-", ".", "inf", "nan", "+1", " 1", ... are not finite numbers
    if (i < len && (s[i] == 'e' || s[i] == 'E')) {
        int j = i + 1;
        bool eneg = false;
        if (j < len && (s[j] == '+' || s[j] == '-')) {
            eneg = s[j] == '-';
            ++j;
        }
        if (j >= len || s[j] < '0' || s[j] > '9') return kText;  // from_chars stops before 'e': trailing text
        int e10 = 0;
        for (; j < len && s[j] >= '0' && s[j] <= '9'; ++j) e10 = min(e10 * 10 + (s[j] - '0'), 100000);
        dexp += eneg ? -e10 : e10;
        i = j;
    }
    if (i != len) return kText;
    if (inexact) return kHost;
    if (w == 0) {
        *out = neg ? -0.0 : 0.0;
        return kNum;
    }
    while (w % 10 == 0) {
        w /= 10;
        ++dexp;
        --sig;
    }
    if (sig > 15 || dexp > 22 || dexp < -22) return kHost;
    const double m = (double)w;  // exact: w < 10^15 < 2^53
    double v = dexp >= 0 ? __dmul_rn(m, kPow10[dexp]) : __ddiv_rn(m, kPow10[-dexp]);
    *out = neg ? -v : v;
    return kNum;
}

// thread per (record, column): value + status, column-major [col][record]
__global__ void parse_cells(const char* __restrict__ b, const uint32_t* __restrict__ beg, uint32_t n_rec, int C,
                            int label, double* __restrict__ val, uint8_t* __restrict__ st) {
    const size_t total = (size_t)n_rec * C;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)(q / C);
        const int c = (int)(q % C);
        const size_t o = (size_t)c * n_rec + r;
        if (c == label) {
            st[o] = kText;
            continue;
        }
        const uint32_t s = beg[(size_t)r * (C + 1) + c], e = beg[(size_t)r * (C + 1) + c + 1] - 1;
        double v = 0.0;
        const uint8_t k = parse_cell(b + s, (int)(e - s), &v);
        st[o] = k;
        val[o] = k == kNum ? v : __longlong_as_double(0x7ff8000000000000ll);
    }
}

__global__ void list_host_cells(const uint8_t* __restrict__ st, size_t total, uint32_t* __restrict__ list,
                                unsigned int* __restrict__ cnt, uint32_t cap) {
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x)
        if (st[q] == kHost) {
            const unsigned int o = atomicAdd(cnt, 1u);
            if (o < cap) list[o] = (uint32_t)q;
        }
}

__global__ void patch_cells(const uint32_t* __restrict__ list, const double* __restrict__ v,
                            const uint8_t* __restrict__ k, uint32_t n, double* __restrict__ val,
                            uint8_t* __restrict__ st) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        val[list[i]] = v[i];
        st[list[i]] = k[i];
    }
}

// per column over the training records: text seen (-> categorical) and
// parsed count
// per column: any text cell / how many numeric cells among the training rows;
// a block per (column, row chunk), one atomic per block and column
__global__ void column_kinds(const uint8_t* __restrict__ st, uint32_t n_rec, uint32_t ntr, int C,
                             int* __restrict__ text, unsigned int* __restrict__ parsed) {
    const int c = blockIdx.y;
    const uint8_t* k = st + (size_t)c * n_rec;
    unsigned int cnt = 0;
    int any_text = 0;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < ntr; r += gridDim.x * blockDim.x) {
        const uint8_t x = k[r];
        any_text |= x == kText;
        cnt += x == kNum;
    }
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        any_text |= __shfl_xor_sync(0xffffffffu, any_text, o);
    }
    __shared__ unsigned int s_cnt;
    __shared__ int s_text;
    if (threadIdx.x == 0) {
        s_cnt = 0;
        s_text = 0;
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_cnt, cnt);
        if (any_text) s_text = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_cnt) atomicAdd(parsed + c, s_cnt);
        if (s_text) text[c] = 1;
    }
}

// A block per numeric column: the training values staged through shared
// memory in row order, one thread adds them sequentially (the reference's
// left-to-right double sums, pipeline.cpp:107-129) — the add chain is the
// only serial part; the staging loads run ahead of it.
constexpr int kStatChunk = 2048;
__global__ void __launch_bounds__(256)
column_stats(const double* __restrict__ val, const uint8_t* __restrict__ st, uint32_t n_rec,
             uint32_t ntr, const int* __restrict__ cols, int n_cols, double* __restrict__ mean,
             double* __restrict__ sd) {
    __shared__ double s_v[kStatChunk];
    __shared__ uint32_t s_wc[8];
    const int wc = blockIdx.x;
    if (wc >= n_cols) return;
    const int c = cols[wc];
    const double* v = val + (size_t)c * n_rec;
    const uint8_t* k = st + (size_t)c * n_rec;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double sum = 0.0, mu = 0.0, ss = 0.0;
    uint32_t cnt = 0;
    for (int pass = 0; pass < 2; ++pass) {
        for (uint32_t r0 = 0; r0 < ntr; r0 += kStatChunk) {
            const uint32_t m = min((uint32_t)kStatChunk, ntr - r0);
            // the chunk's numeric values, compacted in row order (the add
            // chain then runs over a dense array, no per-row branch)
            uint32_t base = 0;
            for (uint32_t i0 = 0; i0 < m; i0 += blockDim.x) {
                const uint32_t i = i0 + threadIdx.x;
                const bool ok = i < m && k[r0 + i] == kNum;
                const double x = ok ? v[r0 + i] : 0.0;
                const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                if (lane == 0) s_wc[wid] = __popc(bal);
                __syncthreads();
                uint32_t before = 0, tot = 0;
                for (int w = 0; w < 8; ++w) {
                    before += w < wid ? s_wc[w] : 0u;
                    tot += s_wc[w];
                }
                if (ok) s_v[base + before + __popc(bal & ((1u << lane) - 1u))] = x;
                base += tot;
                __syncthreads();
            }
            if (threadIdx.x == 0) {
                if (pass == 0) {
                    for (uint32_t i = 0; i < base; ++i) sum = __dadd_rn(sum, s_v[i]);
                    cnt += base;
                } else {
                    for (uint32_t i = 0; i < base; ++i) {
                        const double d = __dsub_rn(s_v[i], mu);
                        ss = __fma_rn(d, d, ss);  // the reference's contracted ss += d * d (host_pipeline.cpp)
                    }
                }
            }
            __syncthreads();  // s_v is refilled next chunk
        }
        if (pass == 0 && threadIdx.x == 0) mu = __ddiv_rn(sum, (double)cnt);
    }
    if (threadIdx.x == 0) {
        mean[wc] = mu;
        sd[wc] = __dsqrt_rn(__ddiv_rn(ss, (double)cnt));
    }
}

// First-error cell of a numeric column outside the training rows: text where
// a number is required (build_columns' DataError, column-major order).
__global__ void first_text(const uint8_t* __restrict__ st, uint32_t n_rec, uint32_t r0, uint32_t r1,
                           const int* __restrict__ cols, int n_cols, unsigned long long* __restrict__ bad) {
    const size_t span = r1 - r0, total = span * (size_t)n_cols;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const int c = cols[q / span];
        const uint32_t r = r0 + (uint32_t)(q % span);
        if (st[(size_t)c * n_rec + r] == kText) atomicMin(bad, ((unsigned long long)c << 32) | (r - r0));
    }
}

// ---------------------------------------------------------------- interning
// Slot = {hash | 1, representative record + 1}; first[slot] = min record.
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

struct Intern {
    ulonglong2* slots;
    unsigned int* first;
    uint32_t mask;
};

// cells of `cols` (interned per table: records [0,ntr) and [ntr,n) separately)
__global__ void intern_cells(const char* __restrict__ b, const uint32_t* __restrict__ beg, uint32_t n_rec,
                             uint32_t ntr, int C, const int* __restrict__ cols, int n_cols, Intern H,
                             uint32_t* __restrict__ cell_slot, int* __restrict__ full) {
    const size_t total = (size_t)n_rec * n_cols;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const int ci = (int)(q / n_rec);
        const uint32_t r = (uint32_t)(q % n_rec);
        const int c = cols[ci];
        const uint32_t s = beg[(size_t)r * (C + 1) + c], e = beg[(size_t)r * (C + 1) + c + 1] - 1;
        if (e == s) {
            cell_slot[q] = 0xffffffffu;  // empty cell
            continue;
        }
        const uint64_t table = r < ntr ? 0 : 1;
        uint64_t h = mix64(0x9e3779b97f4a7c15ull ^ ((uint64_t)ci << 1 | table) ^ ((uint64_t)(e - s) << 40));
        for (uint32_t i = s; i < e; ++i) h = mix64(h ^ (uint8_t)b[i]);
        h |= 1ull;
        uint32_t slot = (uint32_t)(h >> 7) & H.mask;
        uint32_t probes = 0;
        for (;; slot = (slot + 1) & H.mask) {
            if (++probes > H.mask) {
                atomicOr(full, 1);
                cell_slot[q] = 0xffffffffu;
                break;
            }
            const uint64_t tag = ((uint64_t)ci << 40) | ((uint64_t)r + 1);  // column index | record + 1
            ulonglong2 cur = H.slots[slot];
            if (cur.x == 0ull) {
                cur = cas128(H.slots + slot, make_ulonglong2(0ull, 0ull), make_ulonglong2(h, tag));
                if (cur.x == 0ull) {
                    atomicMin(H.first + slot, r);
                    cell_slot[q] = slot;
                    break;
                }
            }
            if (cur.x != h) continue;
            while (cur.y == 0ull) cur.y = *reinterpret_cast<volatile unsigned long long*>(&H.slots[slot].y);
            if ((int)(cur.y >> 40) != ci) continue;  // another column's string (hash collision)
            const uint32_t r2 = (uint32_t)((cur.y & ((1ull << 40) - 1)) - 1);
            if ((r2 < ntr) != (r < ntr)) continue;  // the other table's string (hash collision)
            const uint32_t s2 = beg[(size_t)r2 * (C + 1) + c], e2 = beg[(size_t)r2 * (C + 1) + c + 1] - 1;
            bool same = e2 - s2 == e - s;
            for (uint32_t i = 0; same && i < e - s; ++i) same = b[s + i] == b[s2 + i];
            if (!same) continue;
            atomicMin(H.first + slot, r);
            cell_slot[q] = slot;
            break;
        }
    }
}

// occupied slots -> (column index, table, first record) keys for ordering
__global__ void collect_slots(const ulonglong2* __restrict__ slots, const unsigned int* __restrict__ first,
                              uint32_t n_slots, uint32_t ntr, const uint32_t* __restrict__ owner_col,
                              unsigned long long* __restrict__ key, uint32_t* __restrict__ sid,
                              unsigned int* __restrict__ cnt) {
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_slots; s += gridDim.x * blockDim.x)
        if (slots[s].x != 0ull) {
            const uint32_t fr = first[s];
            const uint64_t table = fr < ntr ? 0 : 1;
            const unsigned int o = atomicAdd(cnt, 1u);
            key[o] = ((uint64_t)owner_col[s] << 40) | (table << 39) | fr;
            sid[o] = s;
        }
}

// the column of a slot: from any cell that maps to it
__global__ void slot_columns(const uint32_t* __restrict__ cell_slot, uint32_t n_rec, int n_cols,
                             uint32_t* __restrict__ owner_col) {
    const size_t total = (size_t)n_rec * n_cols;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const uint32_t s = cell_slot[q];
        if (s != 0xffffffffu) owner_col[s] = (uint32_t)(q / n_rec);
    }
}

__global__ void assign_ids(const unsigned long long* __restrict__ key, const uint32_t* __restrict__ sid, uint32_t n,
                           int32_t* __restrict__ slot_id) {
    // keys sorted by (column, table, first record): id = rank inside its (column, table) run
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long grp = key[i] >> 39;
        uint32_t lo = 0, hi = i;  // first index of this group (binary search: keys sorted)
        while (lo < hi) {
            const uint32_t mid = (lo + hi) / 2;
            if ((key[mid] >> 39) < grp)
                lo = mid + 1;
            else
                hi = mid;
        }
        slot_id[sid[i]] = (int32_t)(i - lo);
    }
}

// cat ids into the two tables' [slot][row] blocks
__global__ void write_cat(const uint32_t* __restrict__ cell_slot, const int32_t* __restrict__ slot_id, uint32_t n_rec,
                          uint32_t ntr, int n_cols, const int* __restrict__ out_slot, int32_t* __restrict__ tr,
                          int32_t* __restrict__ te) {
    const size_t total = (size_t)n_rec * n_cols;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const int ci = (int)(q / n_rec);
        const uint32_t r = (uint32_t)(q % n_rec);
        const uint32_t s = cell_slot[q];
        const int32_t id = s == 0xffffffffu ? -1 : slot_id[s];
        const int o = out_slot[ci];
        if (o < 0) continue;
        if (r < ntr)
            tr[(size_t)o * ntr + r] = id;
        else
            te[(size_t)o * (n_rec - ntr) + (r - ntr)] = id;
    }
}

__global__ void write_labels(const uint32_t* __restrict__ cell_slot, const int32_t* __restrict__ slot_id,
                             const uint8_t* __restrict__ id_attack, uint32_t ntr, uint8_t* __restrict__ out) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < ntr; r += gridDim.x * blockDim.x) {
        const uint32_t s = cell_slot[r];
        out[r] = s == 0xffffffffu ? id_attack[0] : id_attack[1 + slot_id[s]];
    }
}

// numeric columns into the two tables' [slot][row] blocks
__global__ void write_num(const double* __restrict__ val, uint32_t n_rec, uint32_t ntr, const int* __restrict__ cols,
                          int n_cols, double* __restrict__ tr, double* __restrict__ te) {
    const size_t total = (size_t)n_rec * n_cols;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(q / n_rec);
        const uint32_t r = (uint32_t)(q % n_rec);
        const double v = val[(size_t)cols[i] * n_rec + r];
        if (r < ntr)
            tr[(size_t)i * ntr + r] = v;
        else
            te[(size_t)i * (n_rec - ntr) + (r - ntr)] = v;
    }
}

__global__ void gather_spans(const uint32_t* __restrict__ beg, int C, const uint32_t* __restrict__ rc, uint32_t n,
                             uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t r = rc[2 * i], c = rc[2 * i + 1];
        out[2 * i] = beg[(size_t)r * (C + 1) + c];
        out[2 * i + 1] = beg[(size_t)r * (C + 1) + c + 1] - 1;
    }
}

__global__ void any_empty(const uint32_t* __restrict__ cell_slot, uint32_t n, int* __restrict__ flag) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (cell_slot[i] == 0xffffffffu) *flag = 1;
}

std::shared_ptr<void> dev_owned(DevBuf&& b) {
    // long-lived column arrays: released with cudaFree like ig_columns_upload's
    void* p = b.p;
    b.p = nullptr;
    b.bytes = 0;
    return std::shared_ptr<void>(p, [](void* q) { cudaFree(q); });
}

template <class T>
std::vector<T> to_host(const Ctx& ctx, const DevBuf& d, size_t n) {
    std::vector<T> h(n);
    if (n) read_back(ctx, h.data(), d.p, n * sizeof(T));
    return h;
}

}  // namespace

bool ingest_csv(Ctx& ctx, const char* bytes, size_t len, const std::string& label,
                const std::vector<std::string>& attack, const std::vector<std::string>& normal, int decimals,
                long long train_rows, int ratio_k, ig_schema& S, ig_columns& TR, ig_columns& TE) {
    Trace tr(ctx, "ingest", -1);
    if (decimals < 0 || decimals > 12)
        fail(IG_E_CONFIG, "decimals must be in [0, 12], got " + std::to_string(decimals));
    if (len >= 0xffffffffull) return false;  // 32-bit offsets
    // header on the host (one record; quotes anywhere -> the host path)
    size_t p = 0;
    if (len >= 3 && (unsigned char)bytes[0] == 0xEF && (unsigned char)bytes[1] == 0xBB &&
        (unsigned char)bytes[2] == 0xBF)
        p = 3;
    size_t h_end = p;
    while (h_end < len && bytes[h_end] != '\n' && bytes[h_end] != '\r') ++h_end;
    std::vector<std::string> header;
    {
        size_t a = p;
        for (size_t i = p; i <= h_end; ++i)
            if (i == h_end || bytes[i] == ',') {
                header.emplace_back(bytes + a, i - a);
                a = i + 1;
            }
        for (auto& h : header)
            if (h.find('"') != std::string::npos) return false;
    }
    if (h_end == len && p == len) fail(IG_E_DATA, "<csv>: empty input, no header row");
    size_t body = h_end;
    if (body < len) body += (bytes[body] == '\r' && body + 1 < len && bytes[body + 1] == '\n') ? 2 : 1;
    const int C = (int)header.size();
    auto it = std::find(header.begin(), header.end(), label);
    if (it == header.end()) fail(IG_E_CONFIG, "label column '" + label + "' not found in header");
    const int label_index = (int)(it - header.begin());

    DevBuf d_b(std::max<size_t>(len, 1), ctx.stream);
    IGB_CUDA(cudaMemcpyAsync(d_b.p, bytes, len, cudaMemcpyHostToDevice, ctx.stream));
    const char* db = d_b.as<char>();
    // record terminators of the body
    const unsigned blocks = (unsigned)std::max<size_t>(1, std::min<size_t>((len - body + 65535) / 65536,
                                                                            (size_t)ctx.sm_count * 8));
    DevBuf cnt_block((blocks + 1) * 4, ctx.stream), off_block((blocks + 1) * 4, ctx.stream), quote(4, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(quote.p, 0, 4, ctx.stream));
    uint32_t m = 0;
    if (len > body) {
        IGB_LAUNCH(ctx, mark_ends, blocks, 256, 0, db, len, body, cnt_block.as<uint32_t>(), quote.as<int>());
        IGB_CUDA(cudaMemsetAsync(cnt_block.as<uint32_t>() + blocks, 0, 4, ctx.stream));
        size_t tb = 0;
        IGB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt_block.as<uint32_t>(), off_block.as<uint32_t>(),
                                               (int64_t)blocks + 1, ctx.stream));
        DevBuf temp(tb, ctx.stream);
        IGB_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, tb, cnt_block.as<uint32_t>(), off_block.as<uint32_t>(),
                                               (int64_t)blocks + 1, ctx.stream));
        struct {
            uint32_t m;
            int q;
        } h{};
        read_back(ctx, &h.m, off_block.as<uint32_t>() + blocks, 4);
        read_back(ctx, &h.q, quote.p, 4);
        if (h.q) return false;  // quoted fields: the host reader
        m = h.m;
    }
    DevBuf ends(std::max<size_t>(m, 1) * 4, ctx.stream);
    if (m) IGB_LAUNCH(ctx, write_ends, blocks, 256, 0, db, len, body, off_block.as<uint32_t>(), ends.as<uint32_t>());
    // records: m terminated ones, plus a non-empty tail
    uint32_t tail_start = (uint32_t)body;
    if (m) {
        uint32_t e_last = 0;
        read_back(ctx, &e_last, ends.as<uint32_t>() + m - 1, 4);
        tail_start = e_last + 1;
    }
    const bool tail = tail_start < len;
    const uint32_t n_rec = m + (tail ? 1 : 0);
    if (n_rec == 0) fail(IG_E_DATA, "empty table: no data rows to train on");
    const uint32_t ntr = train_rows >= 0 ? (uint32_t)std::min<long long>(train_rows, n_rec)
                                         : (uint32_t)((uint64_t)ratio_k * n_rec / 10);
    if (ntr == 0) fail(IG_E_DATA, "empty table: no data rows to train on");
    const uint32_t nte = n_rec - ntr;
    Records R{ends.as<uint32_t>(), m, (uint32_t)body, (uint32_t)len, tail};
    // fields
    DevBuf beg((size_t)n_rec * (C + 1) * 4, ctx.stream), bad(8, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, ctx.stream));
    IGB_LAUNCH(ctx, split_fields, grid_for(ctx, (size_t)n_rec * 32, 256), 256, 0, db, R, n_rec, C,
               beg.as<uint32_t>(), bad.as<unsigned long long>());
    unsigned long long hbad = 0;
    read_back(ctx, &hbad, bad.p, 8);
    if (hbad != ~0ull)
        fail(IG_E_DATA, "<csv>: line " + std::to_string((hbad >> 32) + 2) + ": expected " + std::to_string(C) +
                            " fields, got " + std::to_string(hbad & 0xffffffffu));
    tr.mark("records");
    // numbers
    const size_t cells = (size_t)n_rec * C;
    DevBuf val(cells * 8, ctx.stream), st(cells, ctx.stream);
    IGB_LAUNCH(ctx, parse_cells, grid_for(ctx, cells, 256), 256, 0, db, beg.as<uint32_t>(), n_rec, C, label_index,
               val.as<double>(), st.as<uint8_t>());
    {
        // cells outside the device fast path: std::from_chars on the host
        DevBuf hcnt(4, ctx.stream);
        IGB_CUDA(cudaMemsetAsync(hcnt.p, 0, 4, ctx.stream));
        const uint32_t cap = 1u << 20;
        DevBuf list((size_t)cap * 4, ctx.stream);
        IGB_LAUNCH(ctx, list_host_cells, grid_for(ctx, cells, 256), 256, 0, st.as<uint8_t>(), cells,
                   list.as<uint32_t>(), hcnt.as<unsigned int>(), cap);
        unsigned int nh = 0;
        read_back(ctx, &nh, hcnt.p, 4);
        if (nh > cap) return false;  // too many slow-path cells: the host path is as fast
        if (nh) {
            std::vector<uint32_t> hl = to_host<uint32_t>(ctx, list, nh);
            std::vector<uint32_t> hb = to_host<uint32_t>(ctx, beg, (size_t)n_rec * (C + 1));
            std::vector<double> hv(nh);
            std::vector<uint8_t> hk(nh);
            for (unsigned int i = 0; i < nh; ++i) {
                const uint32_t c = hl[i] / n_rec, r = hl[i] % n_rec;
                const uint32_t s = hb[(size_t)r * (C + 1) + c], e = hb[(size_t)r * (C + 1) + c + 1] - 1;
                auto v = parse_double_strict(std::string_view(bytes + s, e - s));
                hk[i] = v ? kNum : kText;
                hv[i] = v ? *v : std::numeric_limits<double>::quiet_NaN();
            }
            DevBuf dv(nh * 8, ctx.stream), dk(nh, ctx.stream);
            IGB_CUDA(cudaMemcpyAsync(dv.p, hv.data(), nh * 8, cudaMemcpyHostToDevice, ctx.stream));
            IGB_CUDA(cudaMemcpyAsync(dk.p, hk.data(), nh, cudaMemcpyHostToDevice, ctx.stream));
            IGB_LAUNCH(ctx, patch_cells, grid_for(ctx, nh, 256), 256, 0, list.as<uint32_t>(), dv.as<double>(),
                       dk.as<uint8_t>(), nh, val.as<double>(), st.as<uint8_t>());
            IGB_CUDA(cudaStreamSynchronize(ctx.stream));
        }
    }
    // kinds (training rows)
    DevBuf text(C * 4, ctx.stream), parsed(C * 4, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(text.p, 0, C * 4, ctx.stream));
    IGB_CUDA(cudaMemsetAsync(parsed.p, 0, C * 4, ctx.stream));
    {
        const dim3 grid((unsigned)std::max<size_t>(1, std::min<size_t>((ntr + 255) / 256, 32)), (unsigned)C);
        IGB_LAUNCH(ctx, column_kinds, grid, 256, 0, st.as<uint8_t>(), n_rec, ntr, C, text.as<int>(),
                   parsed.as<unsigned int>());
    }
    std::vector<int> htext = to_host<int>(ctx, text, C);
    std::vector<unsigned int> hparsed = to_host<unsigned int>(ctx, parsed, C);
    S = ig_schema{};
    S.names = header;
    S.label_index = label_index;
    S.label_column = label;
    S.attack_values = attack;
    S.normal_values = normal;
    S.decimals = decimals;
    S.kind.assign(C, 1);
    S.mean.assign(C, 0.0);
    S.sd.assign(C, 0.0);
    std::vector<int> num_cols, cat_cols;
    for (int c = 0; c < C; ++c) {
        if (c == label_index) continue;
        if (!htext[c] && hparsed[c] > 0) {
            S.kind[c] = 0;
            num_cols.push_back(c);
        } else {
            cat_cols.push_back(c);
        }
    }
    const int n_num = (int)num_cols.size(), n_cat = (int)cat_cols.size();
    DevBuf d_num(std::max(n_num, 1) * 4, ctx.stream), d_cat_cols(std::max(n_cat + 1, 1) * 4, ctx.stream);
    if (n_num) IGB_CUDA(cudaMemcpyAsync(d_num.p, num_cols.data(), n_num * 4, cudaMemcpyHostToDevice, ctx.stream));
    if (n_num) {
        DevBuf mean(n_num * 8, ctx.stream), sd(n_num * 8, ctx.stream);
        IGB_LAUNCH(ctx, column_stats, n_num, 256, 0, val.as<double>(), st.as<uint8_t>(), n_rec, ntr,
                   d_num.as<int>(), n_num, mean.as<double>(), sd.as<double>());
        std::vector<double> hm = to_host<double>(ctx, mean, n_num), hs = to_host<double>(ctx, sd, n_num);
        for (int i = 0; i < n_num; ++i) {
            S.mean[num_cols[i]] = hm[i];
            S.sd[num_cols[i]] = hs[i];
        }
        if (nte) {  // test cells must parse in numeric columns (build_columns)
            IGB_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, ctx.stream));
            IGB_LAUNCH(ctx, first_text, grid_for(ctx, (size_t)nte * n_num, 256), 256, 0, st.as<uint8_t>(), n_rec,
                       ntr, n_rec, d_num.as<int>(), n_num, bad.as<unsigned long long>());
            read_back(ctx, &hbad, bad.p, 8);
            if (hbad != ~0ull) {
                const uint32_t c = (uint32_t)(hbad >> 32), r = (uint32_t)hbad;
                std::vector<uint32_t> hb(C + 1);
                read_back(ctx, hb.data(), beg.as<uint32_t>() + (size_t)(ntr + r) * (C + 1), (C + 1) * 4);
                fail(IG_E_DATA, "row " + std::to_string(r) + ", column " + std::to_string(c) + " (" + header[c] +
                                    "): cannot parse '" + std::string(bytes + hb[c], hb[c + 1] - 1 - hb[c]) +
                                    "' as a number");
            }
        }
    }
    tr.mark("numbers");
    // categorical columns and the label: intern by exact content, ids by first appearance
    std::vector<int> icols = cat_cols;
    icols.push_back(label_index);  // last: labels (training rows only are used)
    const int n_icol = (int)icols.size();
    IGB_CUDA(cudaMemcpyAsync(d_cat_cols.p, icols.data(), n_icol * 4, cudaMemcpyHostToDevice, ctx.stream));
    const size_t icells = (size_t)n_rec * n_icol;
    uint32_t n_slots = 1024;
    while (n_slots < 2 * icells + 16) n_slots <<= 1;
    DevBuf slots((size_t)n_slots * 16, ctx.stream), first((size_t)n_slots * 4, ctx.stream),
        cell_slot(icells * 4, ctx.stream), full(4, ctx.stream), owner((size_t)n_slots * 4, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(slots.p, 0, (size_t)n_slots * 16, ctx.stream));
    IGB_CUDA(cudaMemsetAsync(first.p, 0xff, (size_t)n_slots * 4, ctx.stream));
    IGB_CUDA(cudaMemsetAsync(full.p, 0, 4, ctx.stream));
    Intern H{slots.as<ulonglong2>(), first.as<unsigned int>(), n_slots - 1};
    IGB_LAUNCH(ctx, intern_cells, grid_for(ctx, icells, 256), 256, 0, db, beg.as<uint32_t>(), n_rec, ntr, C,
               d_cat_cols.as<int>(), n_icol, H, cell_slot.as<uint32_t>(), full.as<int>());
    IGB_LAUNCH(ctx, slot_columns, grid_for(ctx, icells, 256), 256, 0, cell_slot.as<uint32_t>(), n_rec, n_icol,
               owner.as<uint32_t>());
    DevBuf key((size_t)n_slots * 8, ctx.stream), key2((size_t)n_slots * 8, ctx.stream), sid((size_t)n_slots * 4, ctx.stream),
        sid2((size_t)n_slots * 4, ctx.stream), dcnt(4, ctx.stream), slot_id((size_t)n_slots * 4, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(dcnt.p, 0, 4, ctx.stream));
    IGB_LAUNCH(ctx, collect_slots, grid_for(ctx, n_slots, 256), 256, 0, slots.as<ulonglong2>(),
               first.as<unsigned int>(), n_slots, ntr, owner.as<uint32_t>(), key.as<unsigned long long>(),
               sid.as<uint32_t>(), dcnt.as<unsigned int>());
    struct {
        unsigned int d;
        int f;
    } hd{};
    read_back(ctx, &hd.d, dcnt.p, 4);
    read_back(ctx, &hd.f, full.p, 4);
    if (hd.f) return false;
    const uint32_t nd = hd.d;
    if (nd) {
        int cbits = 1;
        while ((1 << cbits) <= n_icol) ++cbits;
        size_t tb = 0;
        IGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<unsigned long long>(),
                                                 key2.as<unsigned long long>(), sid.as<uint32_t>(),
                                                 sid2.as<uint32_t>(), (int64_t)nd, 0, 40 + cbits, ctx.stream));
        DevBuf temp(tb, ctx.stream);
        IGB_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, tb, key.as<unsigned long long>(),
                                                 key2.as<unsigned long long>(), sid.as<uint32_t>(),
                                                 sid2.as<uint32_t>(), (int64_t)nd, 0, 40 + cbits, ctx.stream));
        IGB_LAUNCH(ctx, assign_ids, grid_for(ctx, nd, 256), 256, 0, key2.as<unsigned long long>(),
                   sid2.as<uint32_t>(), nd, slot_id.as<int32_t>());
    }
    // dictionaries (id order) from the sorted keys; strings from the host bytes
    std::vector<unsigned long long> hkey = to_host<unsigned long long>(ctx, key2, nd);
    std::vector<std::vector<std::string>> dict_tr(C), dict_te(C);
    std::vector<std::string> train_labels;  // distinct training labels in id order
    if (nd) {
        std::vector<uint32_t> rc(2 * (size_t)nd);
        for (uint32_t i = 0; i < nd; ++i) {
            rc[2 * i] = (uint32_t)(hkey[i] & ((1ull << 39) - 1));
            rc[2 * i + 1] = (uint32_t)icols[(int)(hkey[i] >> 40)];
        }
        DevBuf d_rc(rc.size() * 4, ctx.stream), d_sp(rc.size() * 4, ctx.stream);
        IGB_CUDA(cudaMemcpyAsync(d_rc.p, rc.data(), rc.size() * 4, cudaMemcpyHostToDevice, ctx.stream));
        IGB_LAUNCH(ctx, gather_spans, grid_for(ctx, nd, 256), 256, 0, beg.as<uint32_t>(), C, d_rc.as<uint32_t>(), nd,
                   d_sp.as<uint32_t>());
        std::vector<uint32_t> sp = to_host<uint32_t>(ctx, d_sp, rc.size());
        for (uint32_t i = 0; i < nd; ++i) {
            const bool test = (hkey[i] >> 39) & 1ull;
            const int c = (int)rc[2 * i + 1];
            std::string str(bytes + sp[2 * i], sp[2 * i + 1] - sp[2 * i]);
            if (c == label_index) {
                if (!test) train_labels.push_back(std::move(str));
            } else {
                (test ? dict_te : dict_tr)[c].push_back(std::move(str));
            }
        }
    }
    // labels -> attack flags (every training label must be covered, as infer_schema checks)
    std::vector<uint8_t> id_attack(1 + train_labels.size());
    {
        DevBuf fe(4, ctx.stream);
        IGB_CUDA(cudaMemsetAsync(fe.p, 0, 4, ctx.stream));
        IGB_LAUNCH(ctx, any_empty, grid_for(ctx, ntr, 256), 256, 0,
                   cell_slot.as<uint32_t>() + (size_t)(n_icol - 1) * n_rec, ntr, fe.as<int>());
        int he = 0;
        read_back(ctx, &he, fe.p, 4);
        if (he) id_attack[0] = is_attack(S, std::string_view()) ? 1 : 0;  // an empty label cell
    }
    for (size_t i = 0; i < train_labels.size(); ++i) id_attack[1 + i] = is_attack(S, train_labels[i]) ? 1 : 0;
    tr.mark("dictionaries");
    // typed columns
    auto columns = [&](ig_columns& c, uint32_t rows, bool labels, std::vector<std::vector<std::string>>& dict) {
        c = ig_columns{};
        c.n_rows = rows;
        c.n_cols = C;
        c.label_index = label_index;
        c.decimals = decimals;
        c.scale = std::pow(10.0, decimals);
        c.kind = S.kind;
        c.mean = S.mean;
        c.sd = S.sd;
        c.slot.assign(C, -1);
        c.dict.assign(C, {});
        for (int j = 0; j < C; ++j) {
            if (j == label_index) continue;
            c.slot[j] = S.kind[j] == 0 ? (int)c.n_num++ : (int)c.n_cat++;
            if (S.kind[j] == 1) c.dict[j] = std::move(dict[j]);
        }
        c.device = ctx.device;
        (void)labels;
    };
    columns(TR, ntr, true, dict_tr);
    columns(TE, nte, false, dict_te);
    DevBuf v_tr(std::max<size_t>((size_t)n_num * ntr, 1) * 8, ctx.stream),
        v_te(std::max<size_t>((size_t)n_num * nte, 1) * 8, ctx.stream),
        c_tr(std::max<size_t>((size_t)n_cat * ntr, 1) * 4, ctx.stream),
        c_te(std::max<size_t>((size_t)n_cat * nte, 1) * 4, ctx.stream), a_tr(std::max<size_t>(ntr, 1), ctx.stream),
        out_slot(std::max(n_icol, 1) * 4, ctx.stream), ida(id_attack.size(), ctx.stream);
    if (n_num)
        IGB_LAUNCH(ctx, write_num, grid_for(ctx, (size_t)n_rec * n_num, 256), 256, 0, val.as<double>(), n_rec, ntr,
                   d_num.as<int>(), n_num, v_tr.as<double>(), v_te.as<double>());
    std::vector<int> oslot(n_icol, -1);
    for (int i = 0; i < n_cat; ++i) oslot[i] = i;  // cat_cols are in table order = slot order
    IGB_CUDA(cudaMemcpyAsync(out_slot.p, oslot.data(), n_icol * 4, cudaMemcpyHostToDevice, ctx.stream));
    IGB_CUDA(cudaMemcpyAsync(ida.p, id_attack.data(), id_attack.size(), cudaMemcpyHostToDevice, ctx.stream));
    if (n_cat)
        IGB_LAUNCH(ctx, write_cat, grid_for(ctx, (size_t)n_rec * n_icol, 256), 256, 0, cell_slot.as<uint32_t>(),
                   slot_id.as<int32_t>(), n_rec, ntr, n_icol, out_slot.as<int>(), c_tr.as<int32_t>(),
                   c_te.as<int32_t>());
    IGB_LAUNCH(ctx, write_labels, grid_for(ctx, ntr, 256), 256, 0,
               cell_slot.as<uint32_t>() + (size_t)(n_icol - 1) * n_rec, slot_id.as<int32_t>(), ida.as<uint8_t>(),
               ntr, a_tr.as<uint8_t>());
    IGB_CUDA(cudaStreamSynchronize(ctx.stream));
    TR.d_values = dev_owned(std::move(v_tr));
    TR.d_cat = dev_owned(std::move(c_tr));
    TR.is_attack = to_host<uint8_t>(ctx, a_tr, ntr);  // class counts are checked on the host
    TR.d_attack = dev_owned(std::move(a_tr));
    TE.d_values = dev_owned(std::move(v_te));
    TE.d_cat = dev_owned(std::move(c_te));
    tr.mark("columns");
    return true;
}

}  // namespace igb
