// encode.cu — kernel (1): tokenise → vocabulary → anti-contradiction → pack.
//
// Reference: tokenize_row / format_zscore proj/src/pipeline.cpp:77-105,171-202;
// TokenVocabulary::build :62-69 (std::set byte order, built from ALL training
// rows before filtering, :294 vs :314); anti_contradiction_filter :204-235;
// encode_training :273-328; encode_rows :330-339 (unseen tokens dropped, :254);
// PackedRow bit layout proj/src/bitpack.cpp:17-28.
//
// Split of work: the host owns CSV parsing, schema statistics and the string
// order of the vocabulary (bit-exactness, SURVEY.md §7 hard part 3).  The
// device owns every per-cell operation: the z-score units
// llround(((v-mean)/std)·10^p) in IEEE double with explicit _rn intrinsics (no
// contraction, no fast-math), the distinct (column, units) set, the
// (column, units) → bit lookup and the packed rows; the anti-contradiction
// filter runs on the device as a canonical row sort + run scan.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <mutex>
#include <thread>
#include <exception>

#include "encode.cuh"
#include "host_pipeline.hpp"
#include "subset.cuh"

namespace igb {

namespace {

constexpr int64_t kEmptyCode = INT64_MIN;       // the bare "j:" token (pipeline.cpp:185-186)
constexpr int64_t kFreeSlot = INT64_MIN + 1;    // shared-memory hash: unused slot
constexpr int64_t kCap = 9000000000000000000ll; // pipeline.cpp:81-87 clamp

unsigned grid_for(const Ctx& ctx, size_t work, int threads) {
    size_t g = (work + threads - 1) / threads;
    const size_t cap = (size_t)ctx.sm_count * 32;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

// Per feature column f: numeric source slot (>=0) or categorical slot (<0: ~slot).
struct ColDesc {
    int src;        // >= 0: values block index; < 0: ~cat block index
    double mean, sd;
};

// codes[f][r]: numeric → units or kEmptyCode; categorical → id or kEmptyCode.
__global__ void cell_codes(const double* __restrict__ values, const int32_t* __restrict__ cat,
                           const ColDesc* __restrict__ cols, int n_feat, size_t n, double scale,
                           int64_t* __restrict__ codes) {
    const size_t total = (size_t)n_feat * n;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const int f = (int)(q / n);
        const size_t r = q % n;
        const ColDesc c = cols[f];
        int64_t code;
        if (c.src >= 0) {
            const double v = values[(size_t)c.src * n + r];
            if (isnan(v)) {
                code = kEmptyCode;
            } else {
                const double z = (c.sd == 0.0) ? 0.0 : __ddiv_rn(__dsub_rn(v, c.mean), c.sd);
                const double scaled = __dmul_rn(z, scale);
                if (fabs(scaled) >= 9.0e18)
                    code = scaled < 0 ? -kCap : kCap;
                else
                    code = llround(scaled);  // halfway cases away from zero, as std::llround
            }
        } else {
            const int32_t id = cat[(size_t)(~c.src) * n + r];
            code = id < 0 ? kEmptyCode : (int64_t)id;
        }
        codes[q] = code;
    }
}

// Block-level distinct codes of one column chunk (shared-memory hash), appended
// to a global (column, code) list.  grid = (chunks, n_feat).
// 8,192-row chunks (128 KB of slots, dynamic shared memory): fewer chunks,
// fewer repeats of a column's codes across chunks for the host to merge.
constexpr int kDistinctRows = 8192;
constexpr int kDistinctSlots = 16384;
__global__ void __launch_bounds__(256)
distinct_codes(const int64_t* __restrict__ codes, size_t n, int64_t* __restrict__ out_code,
               int32_t* __restrict__ out_col, unsigned long long* __restrict__ out_count) {
    extern __shared__ int64_t slots[];
    const int f = blockIdx.y;
    const size_t r0 = (size_t)blockIdx.x * kDistinctRows;
    for (int i = threadIdx.x; i < kDistinctSlots; i += blockDim.x) slots[i] = kFreeSlot;
    __syncthreads();
    const size_t r1 = min(n, r0 + kDistinctRows);
    for (size_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        const int64_t c = codes[(size_t)f * n + r];
        unsigned s = (unsigned)(mix64((uint64_t)c) & (kDistinctSlots - 1));
        for (;;) {
            const unsigned long long prev =
                atomicCAS(reinterpret_cast<unsigned long long*>(&slots[s]), (unsigned long long)kFreeSlot,
                          (unsigned long long)c);
            if (prev == (unsigned long long)kFreeSlot) {
                const unsigned long long o = atomicAdd(out_count, 1ull);
                out_code[o] = c;
                out_col[o] = f;
                break;
            }
            if ((int64_t)prev == c) break;
            s = (s + 1) & (kDistinctSlots - 1);
        }
    }
}

struct Lut {
    int kind;      // 0 numeric (sorted codes + bits), 1 categorical (id -> bit)
    int off, len;  // numeric: into lcodes/lbits; categorical: into cbits
    int empty_bit; // bit of the "j:" token or -1
};

__device__ __forceinline__ int lookup(const Lut& L, int64_t code, const int64_t* __restrict__ lcodes,
                                      const int32_t* __restrict__ lbits, const int32_t* __restrict__ cbits) {
    if (code == kEmptyCode) return L.empty_bit;
    if (L.kind == 1) return (code >= 0 && code < L.len) ? cbits[L.off + code] : -1;
    int lo = 0, hi = L.len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (lcodes[L.off + mid] < code)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < L.len && lcodes[L.off + lo] == code) ? lbits[L.off + lo] : -1;
}

// Set each cell's token bit in its packed row (bitpack.cpp:25-26); tokens not
// in the vocabulary are dropped (pipeline.cpp:254).
__global__ void pack_cells(const int64_t* __restrict__ codes, size_t n, int n_feat, const Lut* __restrict__ luts,
                           const int64_t* __restrict__ lcodes, const int32_t* __restrict__ lbits,
                           const int32_t* __restrict__ cbits, int k, unsigned long long* __restrict__ rows) {
    const size_t total = (size_t)n_feat * n;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const int f = (int)(q / n);
        const size_t r = q % n;
        const int bit = lookup(luts[f], codes[q], lcodes, lbits, cbits);
        if (bit >= 0) atomicOr(rows + r * k + (bit >> 6), 1ull << (bit & 63));
    }
}

// ------------------------------------------------------------------ device vocabulary
// TokenVocabulary::build (pipeline.cpp:62-69: std::set<std::string>, byte order)
// and the bit assignment of encode_training (:294-304) on the device, for up
// to kVocabMax tokens (else the host builds it, as before).  A token is
// "<j>:<value>"; its byte order is reproduced by a 128-bit key:
//   [127:120] rank of the "<j>:" prefix among the feature columns (host, byte
//             order: no prefix is a prefix of another, they all end in ':')
//   [119:118] group: 0 the empty value, 1 a '-' value, 2 any other
//   numeric:  19 nibbles, the integer part's decimal digits + 1, left aligned,
//             0 after the last one ('.' and the end of the string sort below
//             every digit), then the p fractional digits as an integer (they
//             have a fixed width, so numeric order is byte order)
//   categorical: the value's byte-order rank within its column's dictionary
//             (host, computed with the columns)
// The value text is format_zscore's (pipeline.cpp:77-105): sign only for
// non-zero negatives, whole = |units| / 10^p, frac = |units| % 10^p.
constexpr int kVocabMax = 8192;
constexpr int kVocabSlots = 1 << 15;

struct FeatDesc {
    int kind;      // 0 numeric, 1 categorical
    int col_rank;  // byte-order rank of "<j>:" among the features
    int cat_off;   // categorical: offset into cbits / crank
    int cat_len;   // categorical: dictionary size
};

__device__ __forceinline__ ulonglong2 cas128_enc(ulonglong2* addr, ulonglong2 cmp, ulonglong2 val) {
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

// exact distinct (feature, code) of the per-chunk lists (distinct_codes repeats
// a value once per 8,192-row chunk); slot = {code, feature + 1}, {0, 0} empty
__global__ void vocab_unique(const int64_t* __restrict__ raw_code, const int32_t* __restrict__ raw_col,
                             const unsigned long long* __restrict__ raw_count, ulonglong2* __restrict__ slots,
                             int64_t* __restrict__ u_code, int32_t* __restrict__ u_feat,
                             unsigned int* __restrict__ u_count) {
    const unsigned long long m = *raw_count;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const int64_t c = raw_code[i];
        const int f = raw_col[i];
        const ulonglong2 me = make_ulonglong2((unsigned long long)c, (unsigned long long)f + 1ull);
        unsigned s = (unsigned)(mix64((uint64_t)c ^ (0x9e3779b97f4a7c15ull * (uint64_t)(f + 1))) & (kVocabSlots - 1));
        for (unsigned probe = 0; probe < (unsigned)kVocabSlots; ++probe, s = (s + 1) & (kVocabSlots - 1)) {
            const ulonglong2 old = cas128_enc(slots + s, make_ulonglong2(0ull, 0ull), me);
            if (old.x == 0ull && old.y == 0ull) {
                const unsigned idx = atomicAdd(u_count, 1u);
                if (idx < (unsigned)kVocabMax) {
                    u_code[idx] = c;
                    u_feat[idx] = f;
                }
                break;
            }
            if (old.x == me.x && old.y == me.y) break;
        }
    }
}

__device__ __forceinline__ void token_key(const FeatDesc& d, int64_t code, const int32_t* __restrict__ crank,
                                          uint64_t pow10p, unsigned long long& hi, unsigned long long& lo) {
    hi = (unsigned long long)d.col_rank << 56;
    lo = 0;
    if (code == kEmptyCode) return;  // group 0
    if (d.kind == 1) {
        hi |= (1ull << 54) | (unsigned long long)(uint32_t)crank[d.cat_off + code];
        return;
    }
    const bool neg = code < 0;
    const uint64_t mag = neg ? (uint64_t)0 - (uint64_t)code : (uint64_t)code;
    const uint64_t whole = mag / pow10p, frac = mag % pow10p;
    hi |= (unsigned long long)((neg && mag != 0) ? 1 : 2) << 54;
    // decimal digits of whole, most significant first (at least one digit)
    int nd = 0;
    uint8_t dig[20];
    uint64_t w = whole;
    do {
        dig[nd++] = (uint8_t)(w % 10);
        w /= 10;
    } while (w);
    // nibble i (0-based, left aligned) = digit i + 1; 13 nibbles in hi[53:2], 6 in lo[63:40]
    for (int i = 0; i < nd; ++i) {
        const unsigned long long nib = (unsigned long long)dig[nd - 1 - i] + 1ull;
        if (i < 13)
            hi |= nib << (50 - 4 * i);
        else
            lo |= nib << (60 - 4 * (i - 13));
    }
    lo |= (unsigned long long)frac;  // < 10^12 < 2^40
}

__device__ __forceinline__ bool key_gt(unsigned long long ah, unsigned long long al, unsigned long long bh,
                                       unsigned long long bl) {
    return ah > bh || (ah == bh && al > bl);
}

// ascending bitonic sort of (hi, lo, idx) in shared memory; n2 a power of two
__device__ void block_bitonic(unsigned long long* hi, unsigned long long* lo, uint16_t* idx, int n2) {
    for (int k = 2; k <= n2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    if (key_gt(hi[i], lo[i], hi[ixj], lo[ixj]) == up) {
                        unsigned long long t = hi[i];
                        hi[i] = hi[ixj];
                        hi[ixj] = t;
                        t = lo[i];
                        lo[i] = lo[ixj];
                        lo[ixj] = t;
                        const uint16_t u = idx[i];
                        idx[i] = idx[ixj];
                        idx[ixj] = u;
                    }
                }
            }
            __syncthreads();
        }
}

// The same for n2 <= 1024 with a 1024-thread block, one element per thread
// (padded with all-ones keys): the exchanges with partners in the same warp
// (j < 32, 40 of the 55 stages) go through shuffles, the rest through shared
// memory — 15 block barriers instead of 55.
__device__ void block_bitonic_1024(unsigned long long* hi, unsigned long long* lo, uint16_t* idx, int n2) {
    const int i = threadIdx.x;
    unsigned long long h = i < n2 ? hi[i] : ~0ull, l = i < n2 ? lo[i] : ~0ull;
    uint32_t x = i < n2 ? idx[i] : 0xffffu;
    __syncthreads();
    for (int k = 2; k <= 1024; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            unsigned long long ph, pl;
            uint32_t px;
            if (j < 32) {
                ph = __shfl_xor_sync(0xffffffffu, h, j);
                pl = __shfl_xor_sync(0xffffffffu, l, j);
                px = __shfl_xor_sync(0xffffffffu, x, j);
            } else {
                hi[i] = h;
                lo[i] = l;
                idx[i] = (uint16_t)x;
                __syncthreads();
                ph = hi[i ^ j];
                pl = lo[i ^ j];
                px = idx[i ^ j];
                __syncthreads();
            }
            // ascending where (i & k) == 0: the lower index keeps the smaller key
            const bool up = (i & k) == 0, lower = (i & j) == 0;
            const bool mine_gt = key_gt(h, l, ph, pl);
            if (mine_gt == (up == lower)) {
                h = ph;
                l = pl;
                x = px;
            }
        }
    hi[i] = h;
    lo[i] = l;
    idx[i] = (uint16_t)x;
    __syncthreads();
}

// One block: rank the distinct tokens in byte order (bit = rank), then the pack
// tables — numeric (feature, code) sorted with their bits, categorical id ->
// bit, the empty token's bit per feature — and the token list in bit order for
// the host text.  out_L = number of tokens (> kVocabMax: the host builds it).
__global__ void __launch_bounds__(1024)
vocab_build(const int64_t* __restrict__ u_code, const int32_t* __restrict__ u_feat,
            const unsigned int* __restrict__ u_count, const FeatDesc* __restrict__ desc, int n_feat,
            const int32_t* __restrict__ crank, int cat_total, uint64_t pow10p, Lut* __restrict__ lut,
            int64_t* __restrict__ lcodes, int32_t* __restrict__ lbits, int32_t* __restrict__ cbits,
            int32_t* __restrict__ ubits, int64_t* __restrict__ list_code, int32_t* __restrict__ list_feat,
            unsigned int* __restrict__ out_L) {
    extern __shared__ unsigned long long vsm[];
    const unsigned U = *u_count;
    if (threadIdx.x == 0) *out_L = U;
    if (U > (unsigned)kVocabMax) return;
    int n2 = 1;
    while (n2 < (int)U) n2 <<= 1;
    unsigned long long* hi = vsm;
    unsigned long long* lo = vsm + kVocabMax;
    uint16_t* idx = reinterpret_cast<uint16_t*>(vsm + 2 * kVocabMax);
    for (int f = threadIdx.x; f < n_feat; f += blockDim.x) {
        const FeatDesc d = desc[f];
        lut[f] = Lut{d.kind, d.kind == 1 ? d.cat_off : 0, d.kind == 1 ? d.cat_len : 0, -1};
    }
    for (int i = threadIdx.x; i < cat_total; i += blockDim.x) cbits[i] = -1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        if (i < (int)U) {
            token_key(desc[u_feat[i]], u_code[i], crank, pow10p, hi[i], lo[i]);
        } else {
            hi[i] = ~0ull;
            lo[i] = ~0ull;
        }
        idx[i] = (uint16_t)i;
    }
    __syncthreads();
    if (n2 <= 1024 && blockDim.x == 1024)
        block_bitonic_1024(hi, lo, idx, n2);
    else
        block_bitonic(hi, lo, idx, n2);
    for (int pos = threadIdx.x; pos < (int)U; pos += blockDim.x) {
        const int i = idx[pos];
        const int f = u_feat[i];
        const int64_t c = u_code[i];
        ubits[i] = pos;
        list_code[pos] = c;
        list_feat[pos] = f;
        if (c == kEmptyCode)
            lut[f].empty_bit = pos;
        else if (desc[f].kind == 1)
            cbits[desc[f].cat_off + c] = pos;
    }
    __syncthreads();
    // numeric tables: (feature, code) order
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        if (i < (int)U) {
            hi[i] = (unsigned long long)u_feat[i];
            lo[i] = (unsigned long long)u_code[i] ^ (1ull << 63);
        } else {
            hi[i] = ~0ull;
            lo[i] = ~0ull;
        }
        idx[i] = (uint16_t)i;
    }
    __syncthreads();
    if (n2 <= 1024 && blockDim.x == 1024)
        block_bitonic_1024(hi, lo, idx, n2);
    else
        block_bitonic(hi, lo, idx, n2);
    for (int pos = threadIdx.x; pos < (int)U; pos += blockDim.x) {
        const int i = idx[pos];
        lcodes[pos] = u_code[i];
        lbits[pos] = ubits[i];
        const int f = (int)hi[pos];
        if (desc[f].kind == 0 && (pos == 0 || (int)hi[pos - 1] != f)) lut[f].off = pos;
    }
    __syncthreads();
    for (int pos = threadIdx.x; pos < (int)U; pos += blockDim.x) {
        const int f = (int)hi[pos];
        if (desc[f].kind == 0 && (pos + 1 == (int)U || (int)hi[pos + 1] != f)) lut[f].len = pos + 1 - lut[f].off;
    }
}

// categorical features of a test table: their Lut points at its remapped table
// (triples feature, offset, length)
__global__ void patch_cat_lut(const int32_t* __restrict__ fol, int n, Lut* __restrict__ lut) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        lut[fol[3 * i]].off = fol[3 * i + 1];
        lut[fol[3 * i]].len = fol[3 * i + 2];
    }
}

// categorical test ids -> the training dictionary's bits (remap: test id ->
// training id or -1, built on the host from the two dictionaries' strings)
__global__ void remap_cat(const int32_t* __restrict__ remap, int n, const int32_t* __restrict__ train_cbits,
                          const int32_t* __restrict__ train_off_of, int32_t* __restrict__ out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int r = remap[i];
        out[i] = r >= 0 ? train_cbits[train_off_of[i] + r] : -1;
    }
}

// Run heads of the canonically sorted rows: head[i] = rows differ from i-1.



// Anti-contradiction grouping without sorting: every row joins the hash slot
// of its exact content (open addressing; a slot holds the first row's index + 1,
// equality is checked on all K words), and ORs its class into the slot.
__global__ void group_insert(const int64_t* __restrict__ rows, size_t n, int k, unsigned int* __restrict__ slot_row,
                             uint32_t mask, const uint8_t* __restrict__ attack, unsigned int* __restrict__ slot_cls,
                             uint32_t* __restrict__ grp) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const int64_t* a = rows + i * k;
        uint64_t h = 0x9e3779b97f4a7c15ull;
        for (int w = 0; w < k; ++w) h = mix64(h ^ (uint64_t)a[w]);
        uint32_t s = (uint32_t)h & mask;
        for (;; s = (s + 1) & mask) {
            unsigned int cur = slot_row[s];
            if (cur == 0u) {
                cur = atomicCAS(slot_row + s, 0u, (unsigned int)i + 1u);
                if (cur == 0u) break;  // first row of this content
            }
            const int64_t* b = rows + (size_t)(cur - 1u) * k;
            bool same = true;
            for (int w = 0; w < k && same; ++w) same = a[w] == b[w];
            if (same) break;
        }
        grp[i] = s;
        atomicOr(slot_cls + s, attack[i] ? 1u : 2u);
    }
}

__global__ void group_flags(const uint32_t* __restrict__ grp, const unsigned int* __restrict__ slot_cls,
                            const uint8_t* __restrict__ attack, size_t n, uint8_t* __restrict__ keep_a,
                            uint8_t* __restrict__ keep_n, uint8_t* __restrict__ removed) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const bool contra = slot_cls[grp[i]] == 3u;
        const bool a = attack[i] != 0;
        keep_a[i] = (!contra && a) ? 1 : 0;
        keep_n[i] = (!contra && !a) ? 1 : 0;
        removed[i] = contra ? 1 : 0;
    }
}

__global__ void iota32(uint32_t* p, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)i;
}

__global__ void gather_rows_idx(const int64_t* __restrict__ src, const uint32_t* __restrict__ idx, size_t m, int k,
                                int64_t* __restrict__ dst) {
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < m * k; q += (size_t)gridDim.x * blockDim.x)
        dst[q] = src[(size_t)idx[q / k] * k + q % k];
}

// Stable selection of row indices whose flag is set.
// Stable selection of row indices whose flag is set, for several flag arrays
// at once: the counts come back in one read-back.
void select_flagged_n(Ctx& ctx, const uint8_t* const* d_flags, int nsets, size_t n, DevBuf* idx_out, size_t* counts) {
    DevBuf iota(std::max<size_t>(n, 1) * 4, ctx.stream), nsel(8 * nsets, ctx.stream);
    IGB_LAUNCH(ctx, iota32, grid_for(ctx, n, 256), 256, 0, iota.as<uint32_t>(), n);
    size_t tb = 0;
    IGB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.as<uint32_t>(), d_flags[0], iota.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)n, ctx.stream));
    DevBuf temp(tb, ctx.stream);
    for (int s = 0; s < nsets; ++s) {
        idx_out[s].alloc(std::max<size_t>(n, 1) * 4, ctx.stream);
        IGB_CUDA(cub::DeviceSelect::Flagged(temp.p, tb, iota.as<uint32_t>(), d_flags[s], idx_out[s].as<uint32_t>(),
                                            nsel.as<int64_t>() + s, (int64_t)n, ctx.stream));
    }
    std::vector<int64_t> h(nsets);
    read_back(ctx, h.data(), nsel.p, 8 * nsets);
    for (int s = 0; s < nsets; ++s) counts[s] = (size_t)h[s];
}

struct DeviceCols {
    DevBuf values, cat, cols, codes, attack;
    const uint8_t* attack_ptr = nullptr;
    size_t n = 0;
    int n_feat = 0;
    std::vector<int> feat_col;  // feature index -> table column
};

// H2D of the parsed columns + kernel (1a): per-cell codes.
namespace {
// the numeric block from its narrow copy form (host_pipeline.hpp): one
// column per blockIdx.y; value = code / scale (IEEE division, the host checked
// it reproduces every parsed value), the type's minimum = empty cell (NaN)
__global__ void narrow_decode(const unsigned char* __restrict__ blob, size_t n, double* __restrict__ out) {
    const NarrowHead h = reinterpret_cast<const NarrowHead*>(blob)[blockIdx.y];
    const unsigned char* src = blob + h.off;
    double* dst = out + (size_t)blockIdx.y * n;
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    for (size_t r = (size_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (size_t)gridDim.x * blockDim.x) {
        double v;
        if (h.type == 0) {
            v = reinterpret_cast<const double*>(src)[r];
        } else if (h.type == 1) {
            const int8_t q = reinterpret_cast<const int8_t*>(src)[r];
            v = q == INT8_MIN ? nan : __ddiv_rn((double)q, h.scale);
        } else if (h.type == 2) {
            const int16_t q = reinterpret_cast<const int16_t*>(src)[r];
            v = q == INT16_MIN ? nan : __ddiv_rn((double)q, h.scale);
        } else {
            const int32_t q = reinterpret_cast<const int32_t*>(src)[r];
            v = q == INT32_MIN ? nan : __ddiv_rn((double)q, h.scale);
        }
        dst[r] = v;
    }
}

struct PrefetchCols {
    DevBuf values, cat, attack;
    cudaEvent_t ready = nullptr;
    int device = -1;
    ~PrefetchCols() {
        if (ready) cudaEventDestroy(ready);
    }
};
}  // namespace

// returns true when it queued copies that read the columns' host memory
bool upload_and_code(Ctx& ctx, const ig_columns& c, DeviceCols& d) {
    d.n = c.n_rows;
    std::vector<ColDesc> desc;
    for (size_t j = 0; j < c.n_cols; ++j) {
        if (j == c.label_index) continue;
        ColDesc cd;
        cd.src = c.kind[j] == 0 ? c.slot[j] : ~c.slot[j];
        cd.mean = c.mean[j];
        cd.sd = c.sd[j];
        desc.push_back(cd);
        d.feat_col.push_back((int)j);
    }
    d.n_feat = (int)desc.size();
    d.cols.alloc(std::max<size_t>(desc.size(), 1) * sizeof(ColDesc), ctx.stream);
    if (!desc.empty())
        IGB_CUDA(cudaMemcpyAsync(d.cols.p, desc.data(), desc.size() * sizeof(ColDesc), cudaMemcpyHostToDevice,
                                 ctx.stream));
    const double* vals;
    const int32_t* cats;
    bool host_read = false;
    auto* pf = static_cast<PrefetchCols*>(c.prefetch.get());
    if (pf && pf->device == ctx.device) {
        // a prefetch is in flight: order after it, then own its buffers
        // (freed on this stream once the encode kernels are done)
        IGB_CUDA(cudaStreamWaitEvent(ctx.stream, pf->ready, 0));
        d.values = std::move(pf->values);
        d.cat = std::move(pf->cat);
        d.attack = std::move(pf->attack);
        d.values.s = d.cat.s = d.attack.s = ctx.stream;
        c.prefetch.reset();
        vals = d.values.as<double>();
        cats = d.cat.as<int32_t>();
        d.attack_ptr = d.attack.as<uint8_t>();
    } else if (c.d_values && c.device == ctx.device) {
        // resident columns (ig_columns_upload): no host traffic
        vals = static_cast<const double*>(c.d_values.get());
        cats = static_cast<const int32_t*>(c.d_cat.get());
        d.attack_ptr = static_cast<const uint8_t*>(c.d_attack.get());
    } else {
        host_read = true;
        d.values.alloc(c.values.size() * 8, ctx.stream);
        d.cat.alloc(c.cat.size() * 4, ctx.stream);
        if (!c.values.empty())
            IGB_CUDA(cudaMemcpyAsync(d.values.p, c.values.data(), c.values.size() * 8, cudaMemcpyHostToDevice,
                                     ctx.stream));
        if (!c.cat.empty())
            IGB_CUDA(cudaMemcpyAsync(d.cat.p, c.cat.data(), c.cat.size() * 4, cudaMemcpyHostToDevice, ctx.stream));
        if (!c.is_attack.empty()) {
            d.attack.alloc(c.n_rows, ctx.stream);
            IGB_CUDA(cudaMemcpyAsync(d.attack.p, c.is_attack.data(), c.n_rows, cudaMemcpyHostToDevice, ctx.stream));
        }
        vals = d.values.as<double>();
        cats = d.cat.as<int32_t>();
        d.attack_ptr = d.attack.as<uint8_t>();
    }
    const size_t cells = (size_t)d.n_feat * d.n;
    d.codes.alloc(std::max<size_t>(cells, 1) * 8, ctx.stream);
    if (cells)
        IGB_LAUNCH(ctx, cell_codes, grid_for(ctx, cells, 256), 256, 0, vals, cats, d.cols.as<ColDesc>(), d.n_feat,
                   d.n, c.scale, d.codes.as<int64_t>());
    return host_read;
}

// Pack `d`'s cells into rows with lookup tables already on the device.
void pack_tables(Ctx& ctx, uint32_t L, const DeviceCols& d, const Lut* luts, const int64_t* lcodes,
                 const int32_t* lbits, const int32_t* cbits, DevRows& out) {
    out.L = L;
    out.k = words_for(L);
    out.n = d.n;
    out.buf.alloc(std::max<size_t>(out.n * out.k, 1) * 8, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(out.buf.p, 0, std::max<size_t>(out.n * out.k, 1) * 8, ctx.stream));
    const size_t cells = (size_t)d.n_feat * d.n;
    if (cells && out.k)
        IGB_LAUNCH(ctx, pack_cells, grid_for(ctx, cells, 256), 256, 0, d.codes.as<int64_t>(), d.n, d.n_feat, luts,
                   lcodes, lbits, cbits, (int)out.k, reinterpret_cast<unsigned long long*>(out.data()));
}

// Upload a host vocabulary's lookup tables and pack `d`'s cells into rows.
void pack_with(Ctx& ctx, const ig_encoding& e, const DeviceCols& d,
               const std::vector<std::vector<int32_t>>& cat_id_to_bit, DevRows& out) {
    std::vector<Lut> luts(d.n_feat);
    std::vector<int64_t> lcodes;
    std::vector<int32_t> lbits, cbits;
    for (int f = 0; f < d.n_feat; ++f) {
        const int j = d.feat_col[f];
        Lut& L = luts[f];
        L.empty_bit = e.empty_bit[j];
        if (e.kind[j] == 0) {
            L.kind = 0;
            L.off = (int)lbits.size();
            L.len = (int)e.num_codes[j].size();
            lcodes.insert(lcodes.end(), e.num_codes[j].begin(), e.num_codes[j].end());
            lbits.insert(lbits.end(), e.num_bits[j].begin(), e.num_bits[j].end());
        } else {
            L.kind = 1;
            L.off = (int)cbits.size();
            L.len = (int)cat_id_to_bit[j].size();
            cbits.insert(cbits.end(), cat_id_to_bit[j].begin(), cat_id_to_bit[j].end());
        }
    }
    DevBuf dl(std::max<size_t>(luts.size(), 1) * sizeof(Lut), ctx.stream);
    DevBuf dc(std::max<size_t>(lcodes.size(), 1) * 8, ctx.stream), db(std::max<size_t>(lbits.size(), 1) * 4, ctx.stream),
        dcb(std::max<size_t>(cbits.size(), 1) * 4, ctx.stream);
    if (!luts.empty())
        IGB_CUDA(cudaMemcpyAsync(dl.p, luts.data(), luts.size() * sizeof(Lut), cudaMemcpyHostToDevice, ctx.stream));
    if (!lcodes.empty())
        IGB_CUDA(cudaMemcpyAsync(dc.p, lcodes.data(), lcodes.size() * 8, cudaMemcpyHostToDevice, ctx.stream));
    if (!lbits.empty())
        IGB_CUDA(cudaMemcpyAsync(db.p, lbits.data(), lbits.size() * 4, cudaMemcpyHostToDevice, ctx.stream));
    if (!cbits.empty())
        IGB_CUDA(cudaMemcpyAsync(dcb.p, cbits.data(), cbits.size() * 4, cudaMemcpyHostToDevice, ctx.stream));
    pack_tables(ctx, e.L, d, dl.as<Lut>(), dc.as<int64_t>(), db.as<int32_t>(), dcb.as<int32_t>(), out);
    // Lookup tables are freed stream-ordered after the kernel.
}

// The vocabulary on the host (more than kVocabMax tokens, or IG_HOST_VOCAB=1):
// read the distinct (column, code) list back, token text, byte-order sort.
void host_vocab_build(Ctx& ctx, const ig_columns& c, const DeviceCols& d, const DevBuf& lcode, const DevBuf& lcol,
                      const DevBuf& lcnt, ig_encoding& e, DevRows& all) {
    unsigned long long m = 0;
    read_back(ctx, &m, lcnt.p, 8);
    std::vector<int64_t> hcode(m);
    std::vector<int32_t> hcol(m);
    if (m) {
        read_back(ctx, hcode.data(), lcode.p, m * 8);
        read_back(ctx, hcol.data(), lcol.p, m * 4);
    }

    // Host: token text for each distinct (column, code), byte-order sort → bits.
    std::vector<std::unordered_set<int64_t>> seen(c.n_cols);
    struct Tok {
        std::string text;
        int col;
        int64_t code;
    };
    std::vector<Tok> toks;
    for (size_t i = 0; i < m; ++i) {
        const int j = d.feat_col[hcol[i]];
        if (!seen[j].insert(hcode[i]).second) continue;
        std::string value;
        if (hcode[i] == kEmptyCode)
            value.clear();
        else if (c.kind[j] == 0)
            value = format_units(hcode[i], c.decimals);
        else
            value = c.dict[j][(size_t)hcode[i]];
        toks.push_back({std::to_string(j) + ":" + value, j, hcode[i]});
    }
    std::sort(toks.begin(), toks.end(), [](const Tok& a, const Tok& b) { return a.text < b.text; });
    e.L = (uint32_t)toks.size();
    e.num_codes.assign(c.n_cols, {});
    e.num_bits.assign(c.n_cols, {});
    e.cat_bits.assign(c.n_cols, {});
    e.empty_bit.assign(c.n_cols, -1);
    std::vector<std::vector<int32_t>> cat_id_to_bit(c.n_cols);
    for (size_t j = 0; j < c.n_cols; ++j) cat_id_to_bit[j].assign(c.dict[j].size(), -1);
    std::vector<std::vector<std::pair<int64_t, int32_t>>> num(c.n_cols);
    for (size_t b = 0; b < toks.size(); ++b) {
        const Tok& t = toks[b];
        e.vocab_blob += t.text;
        e.vocab_blob += '\n';
        if (t.code == kEmptyCode) {
            e.empty_bit[t.col] = (int)b;
        } else if (c.kind[t.col] == 0) {
            num[t.col].push_back({t.code, (int32_t)b});
        } else {
            cat_id_to_bit[t.col][(size_t)t.code] = (int32_t)b;
            e.cat_bits[t.col].emplace(c.dict[t.col][(size_t)t.code], (int32_t)b);
        }
    }
    for (size_t j = 0; j < c.n_cols; ++j) {
        std::sort(num[j].begin(), num[j].end());
        for (auto& [code, bit] : num[j]) {
            e.num_codes[j].push_back(code);
            e.num_bits[j].push_back(bit);
        }
    }

    // (1c) pack every training row.
    pack_with(ctx, e, d, cat_id_to_bit, all);
}

}  // namespace
}  // namespace igb

// Host text of a device-built vocabulary (ig_encoding::hv): the tokens in bit
// order are copied to page-locked memory on the encode stream; a host thread
// waits for them and fills the host fields.  It also checks that the tokens'
// text is strictly increasing in byte order — the device keys' contract.
struct HostVocabJob {
    igb::BgTask task;
    std::mutex mu;
    bool joined = false;
    std::exception_ptr err;
    void* pinned = nullptr;  // codes [kVocabMax] int64, features [kVocabMax] int32, L (the library's pool)
    ~HostVocabJob() {
        task.join();
        if (pinned) ig_host_free(pinned);
    }
};

const ig_encoding& ig_encoding::host_vocab() const {
    if (hv) {
        std::lock_guard<std::mutex> lock(hv->mu);
        if (!hv->joined) {
            hv->task.join();
            hv->joined = true;
        }
        if (hv->err) std::rethrow_exception(hv->err);
    }
    return *this;
}

namespace igb {
namespace {

// Host descriptors of the device vocabulary, prepared before the encode
// kernels are queued so that the host work overlaps them: byte-order rank of
// each "<j>:" prefix, categorical dictionary offsets and each value's
// byte-order rank in its dictionary; staged in page-locked memory.
struct VocabPrep {
    bool ok = false;
    int nf = 0, cat_total = 0;
    std::vector<int> cat_off;
    void* pinned = nullptr;  // FeatDesc[nf] then int32 crank[cat_total] (the library's page-locked pool)
    ~VocabPrep() {
        if (pinned) ig_host_free(pinned);
    }
};

void vocab_prepare(const ig_columns& c, VocabPrep& vp) {
    static const bool host_only = getenv("IG_HOST_VOCAB") != nullptr;  // A/B and fallback tests
    std::vector<int> feat_col;
    for (size_t j = 0; j < c.n_cols; ++j)
        if (j != c.label_index) feat_col.push_back((int)j);
    const int nf = (int)feat_col.size();
    if (host_only || nf == 0 || nf > 255 || c.decimals > 12) return;
    std::vector<int> order(nf);
    for (int f = 0; f < nf; ++f) order[f] = f;
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        return std::to_string(feat_col[a]) + ":" < std::to_string(feat_col[b]) + ":";
    });
    std::vector<FeatDesc> desc(nf);
    for (int r = 0; r < nf; ++r) desc[order[r]].col_rank = r;
    std::vector<int32_t> crank;
    vp.cat_off.assign(nf, 0);
    for (int f = 0; f < nf; ++f) {
        const int j = feat_col[f];
        desc[f].kind = c.kind[j];
        desc[f].cat_off = 0;
        desc[f].cat_len = 0;
        if (c.kind[j] != 1) continue;
        const auto& dict = c.dict[j];
        desc[f].cat_off = (int)crank.size();
        desc[f].cat_len = (int)dict.size();
        vp.cat_off[f] = desc[f].cat_off;
        std::vector<int> ids(dict.size());
        for (size_t i = 0; i < ids.size(); ++i) ids[i] = (int)i;
        std::sort(ids.begin(), ids.end(), [&](int a, int b) { return dict[a] < dict[b]; });
        crank.resize(crank.size() + dict.size());
        for (size_t r = 0; r < ids.size(); ++r) crank[desc[f].cat_off + ids[r]] = (int32_t)r;
    }
    vp.nf = nf;
    vp.cat_total = (int)crank.size();
    const size_t bytes = nf * sizeof(FeatDesc) + crank.size() * 4;
    if (ig_host_alloc(bytes, &vp.pinned) != IG_OK) return;
    std::memcpy(vp.pinned, desc.data(), nf * sizeof(FeatDesc));
    if (!crank.empty()) std::memcpy(static_cast<char*>(vp.pinned) + nf * sizeof(FeatDesc), crank.data(), crank.size() * 4);
    vp.ok = true;
}

bool device_vocab(Ctx& ctx, const ig_columns& c, const DeviceCols& d, const VocabPrep& vp, const DevBuf& lcode,
                  const DevBuf& lcol, const DevBuf& lcnt, ig_encoding& e) {
    const int nf = d.n_feat;
    if (!vp.ok || vp.nf != nf) return false;
    const int cat_total = vp.cat_total;
    e.dv.cat_off = vp.cat_off;
    // scratch in one block: descriptors, crank | dedup slots, counter | unique
    // (code, feature) | their bits | token list in bit order + L
    auto up16 = [](size_t b) { return (b + 15) & ~size_t{15}; };
    const size_t o_desc = 0, o_crank = o_desc + up16(nf * sizeof(FeatDesc)),
                 o_slots = o_crank + up16(std::max(cat_total, 1) * 4),
                 o_ucount = o_slots + (size_t)kVocabSlots * sizeof(ulonglong2), o_ucode = o_ucount + 16,
                 o_ufeat = o_ucode + kVocabMax * 8, o_ubits = o_ufeat + kVocabMax * 4, o_list = o_ubits + kVocabMax * 4,
                 list_bytes = (size_t)kVocabMax * 12 + 8, total = o_list + list_bytes;
    DevBuf scratch(total, ctx.stream);
    char* sp = scratch.as<char>();
    IGB_CUDA(cudaMemcpyAsync(sp + o_desc, vp.pinned, nf * sizeof(FeatDesc), cudaMemcpyHostToDevice, ctx.stream));
    if (cat_total)
        IGB_CUDA(cudaMemcpyAsync(sp + o_crank, static_cast<const char*>(vp.pinned) + nf * sizeof(FeatDesc),
                                 (size_t)cat_total * 4, cudaMemcpyHostToDevice, ctx.stream));
    IGB_CUDA(cudaMemsetAsync(sp + o_slots, 0, o_ucode - o_slots, ctx.stream));  // slots + counter
    unsigned int* u_count = reinterpret_cast<unsigned int*>(sp + o_ucount);
    int64_t* u_code = reinterpret_cast<int64_t*>(sp + o_ucode);
    int32_t* u_feat = reinterpret_cast<int32_t*>(sp + o_ufeat);
    IGB_LAUNCH(ctx, vocab_unique, (unsigned)ctx.sm_count, 256, 0, lcode.as<int64_t>(), lcol.as<int32_t>(),
               lcnt.as<unsigned long long>(), reinterpret_cast<ulonglong2*>(sp + o_slots), u_code, u_feat, u_count);
    DeviceVocab& dv = e.dv;
    dv.n_feat = nf;
    dv.feat_col = d.feat_col;
    const size_t p_lut = 0, p_lcodes = up16(nf * sizeof(Lut)), p_lbits = p_lcodes + kVocabMax * 8,
                 p_cbits = p_lbits + kVocabMax * 4;
    dv.mem.alloc(p_cbits + std::max(cat_total, 1) * 4, ctx.stream);
    char* mp = dv.mem.as<char>();
    dv.lut = mp + p_lut;
    dv.lcodes = reinterpret_cast<int64_t*>(mp + p_lcodes);
    dv.lbits = reinterpret_cast<int32_t*>(mp + p_lbits);
    dv.cbits = reinterpret_cast<int32_t*>(mp + p_cbits);
    int64_t* list_code = reinterpret_cast<int64_t*>(sp + o_list);
    int32_t* list_feat = reinterpret_cast<int32_t*>(sp + o_list + kVocabMax * 8);
    unsigned int* out_L = reinterpret_cast<unsigned int*>(sp + o_list + kVocabMax * 12);
    uint64_t pow10p = 1;
    for (int i = 0; i < c.decimals; ++i) pow10p *= 10;
    const int smem = kVocabMax * 18;
    IGB_SMEM_ATTR(ctx, vocab_build, smem);
    IGB_LAUNCH(ctx, vocab_build, 1, 1024, smem, u_code, u_feat, u_count,
               reinterpret_cast<const FeatDesc*>(sp + o_desc), nf, reinterpret_cast<const int32_t*>(sp + o_crank),
               cat_total, pow10p, static_cast<Lut*>(dv.lut), dv.lcodes, dv.lbits, dv.cbits,
               reinterpret_cast<int32_t*>(sp + o_ubits), list_code, list_feat, out_L);
    // the token list (for the host text) and L come back in one copy
    auto job = std::make_shared<HostVocabJob>();
    if (ig_host_alloc(list_bytes, &job->pinned) != IG_OK) fail(IG_E_OOM, "page-locked host memory");
    IGB_CUDA(cudaMemcpyAsync(job->pinned, list_code, list_bytes, cudaMemcpyDeviceToHost, ctx.stream));
    IGB_CUDA(cudaStreamSynchronize(ctx.stream));
    const unsigned int L = *reinterpret_cast<const unsigned int*>(static_cast<const char*>(job->pinned) +
                                                                  (size_t)kVocabMax * 12);
    if (L > (unsigned)kVocabMax) {
        dv = DeviceVocab{};
        return false;
    }
    e.L = L;
    dv.valid = true;
    dv.mem.persist();
    e.hv = job;  // text built by start_host_vocab once the rows are queued
    return true;
}

// The host fields of a device-built vocabulary, on a host thread (the token
// list is already in page-locked memory).
void start_host_vocab(Ctx& ctx, const ig_columns& c, const DeviceCols& d, ig_encoding& e) {
    HostVocabJob* jp = e.hv.get();
    if (!jp) return;
    const uint32_t L = e.L;
    const int ncols = (int)c.n_cols, decimals = c.decimals;
    std::vector<int> kind = c.kind, fcol = d.feat_col;
    ig_encoding* ep = &e;
    const auto* dict = &e.dict;  // e.dict = c.dict (copied before this call)
    jp->task.start(ctx.vocab_worker, [jp, ep, dict, ncols, decimals, kind, fcol, L] {
        try {
            const int64_t* code = static_cast<const int64_t*>(jp->pinned);
            const int32_t* feat =
                reinterpret_cast<const int32_t*>(static_cast<const char*>(jp->pinned) + (size_t)kVocabMax * 8);
            ig_encoding& E = *ep;
            E.num_codes.assign(ncols, {});
            E.num_bits.assign(ncols, {});
            E.cat_bits.assign(ncols, {});
            E.empty_bit.assign(ncols, -1);
            std::vector<std::vector<std::pair<int64_t, int32_t>>> num(ncols);
            std::string prev, blob;
            for (uint32_t b = 0; b < L; ++b) {
                const int j = fcol[feat[b]];
                std::string value;
                if (code[b] == kEmptyCode)
                    value.clear();
                else if (kind[j] == 0)
                    value = format_units(code[b], decimals);
                else
                    value = (*dict)[j][(size_t)code[b]];
                std::string text = std::to_string(j) + ":" + value;
                if (b && !(prev < text)) fail(IG_E_CUDA, "device vocabulary order differs from byte order at bit " +
                                                             std::to_string(b) + " ('" + prev + "', '" + text + "')");
                blob += text;
                blob += '\n';
                if (code[b] == kEmptyCode)
                    E.empty_bit[j] = (int)b;
                else if (kind[j] == 0)
                    num[j].push_back({code[b], (int32_t)b});
                else
                    E.cat_bits[j].emplace(value, (int32_t)b);
                prev = std::move(text);
            }
            for (int j = 0; j < ncols; ++j) {
                std::sort(num[j].begin(), num[j].end());
                for (auto& [cd, bit] : num[j]) {
                    E.num_codes[j].push_back(cd);
                    E.num_bits[j].push_back(bit);
                }
            }
            E.vocab_blob = std::move(blob);
        } catch (...) {
            jp->err = std::current_exception();
        }
    });
}

}  // namespace

void prefetch_columns(Ctx& ctx, ig_columns& c) {
    if (c.d_values && c.device == ctx.device) return;  // already resident
    auto pf = std::make_shared<PrefetchCols>();
    pf->device = ctx.device;
    pf->values.alloc(std::max<size_t>(c.values.size(), 1) * 8, ctx.copy);
    pf->cat.alloc(std::max<size_t>(c.cat.size(), 1) * 4, ctx.copy);
    pf->attack.alloc(std::max<size_t>(c.is_attack.size(), 1), ctx.copy);
    static const bool raw = getenv("IG_COLUMNS_RAW_COPY") != nullptr;  // A/B
    if (!c.narrow.empty() && !raw) {
        // the narrow form (C3 test columns: 14 MB instead of 42 MB), decoded
        // on the copy stream
        DevBuf blob(c.narrow.size(), ctx.copy);
        IGB_CUDA(cudaMemcpyAsync(blob.p, c.narrow.data(), c.narrow.size(), cudaMemcpyHostToDevice, ctx.copy));
        const dim3 grid((unsigned)std::min<size_t>((c.n_rows + 255) / 256, 64), (unsigned)c.n_num);
        Ctx cc = ctx;
        cc.stream = ctx.copy;
        IGB_LAUNCH(cc, narrow_decode, grid, 256, 0, blob.as<unsigned char>(), c.n_rows, pf->values.as<double>());
        ctx.launches += cc.launches - ctx.launches;
    } else if (!c.values.empty()) {
        IGB_CUDA(cudaMemcpyAsync(pf->values.p, c.values.data(), c.values.size() * 8, cudaMemcpyHostToDevice, ctx.copy));
    }
    if (!c.cat.empty())
        IGB_CUDA(cudaMemcpyAsync(pf->cat.p, c.cat.data(), c.cat.size() * 4, cudaMemcpyHostToDevice, ctx.copy));
    if (!c.is_attack.empty())
        IGB_CUDA(cudaMemcpyAsync(pf->attack.p, c.is_attack.data(), c.is_attack.size(), cudaMemcpyHostToDevice,
                                 ctx.copy));
    IGB_CUDA(cudaEventCreateWithFlags(&pf->ready, cudaEventDisableTiming));
    IGB_CUDA(cudaEventRecord(pf->ready, ctx.copy));
    c.prefetch = pf;
}

void drop_prefetch(ig_columns& c) {
    if (auto* pf = static_cast<PrefetchCols*>(c.prefetch.get())) cudaEventSynchronize(pf->ready);
    c.prefetch.reset();
}

void encode_training_dev(Ctx& ctx, const ig_columns& c, ig_encoding& e) {
    if (c.is_attack.size() != c.n_rows) fail(IG_E_INVALID_ARG, "encode_training: columns built without labels");
    e = ig_encoding{};
    e.n_cols = c.n_cols;
    e.label_index = c.label_index;
    e.decimals = c.decimals;
    e.kind = c.kind;
    e.dict = c.dict;
    VocabPrep vp;
    vocab_prepare(c, vp);
    DeviceCols d;
    upload_and_code(ctx, c, d);

    // (1b) distinct (column, code) over ALL training rows (vocabulary precedes the filter).
    const size_t chunks = (d.n + kDistinctRows - 1) / kDistinctRows;
    const size_t cap = std::max<size_t>((size_t)d.n_feat * d.n, 1);
    DevBuf lcode(cap * 8, ctx.stream), lcol(cap * 4, ctx.stream), lcnt(8, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(lcnt.p, 0, 8, ctx.stream));
    if (d.n && d.n_feat)
        IGB_SMEM_ATTR(ctx, distinct_codes, kDistinctSlots * (int)sizeof(int64_t));
    if (d.n && d.n_feat)
        IGB_LAUNCH(ctx, distinct_codes, dim3((unsigned)chunks, (unsigned)d.n_feat), 256,
                   kDistinctSlots * sizeof(int64_t), d.codes.as<int64_t>(), d.n,
                   lcode.as<int64_t>(), lcol.as<int32_t>(), lcnt.as<unsigned long long>());
    DevRows all;
    if (device_vocab(ctx, c, d, vp, lcode, lcol, lcnt, e)) {
        // (1c) pack every training row with the device tables, then the host text
        pack_tables(ctx, e.L, d, static_cast<const Lut*>(e.dv.lut), e.dv.lcodes, e.dv.lbits, e.dv.cbits, all);
        start_host_vocab(ctx, c, d, e);
    } else {
        host_vocab_build(ctx, c, d, lcode, lcol, lcnt, e, all);
    }
    const size_t n = all.n, k = all.k;

    // Class checks + anti-contradiction filter (pipeline.cpp:306-318) on the device.
    size_t n_att = 0;
    for (uint8_t a : c.is_attack) n_att += a;
    if (n_att == 0 || n_att == n) fail(IG_E_DATA, "training data must contain both attack and normal instances");
    uint32_t slots = 1024;
    while (slots < 2 * n) slots <<= 1;
    DevBuf slot_row((size_t)slots * 4, ctx.stream), slot_cls((size_t)slots * 4, ctx.stream), grp(n * 4, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(slot_row.p, 0, (size_t)slots * 4, ctx.stream));
    IGB_CUDA(cudaMemsetAsync(slot_cls.p, 0, (size_t)slots * 4, ctx.stream));
    IGB_LAUNCH(ctx, group_insert, grid_for(ctx, n, 256), 256, 0, all.data(), n, (int)k, slot_row.as<unsigned int>(),
               slots - 1, d.attack_ptr, slot_cls.as<unsigned int>(), grp.as<uint32_t>());
    DevBuf keep_a(n, ctx.stream), keep_n(n, ctx.stream), removed(n, ctx.stream);
    IGB_LAUNCH(ctx, group_flags, grid_for(ctx, n, 256), 256, 0, grp.as<uint32_t>(), slot_cls.as<unsigned int>(),
               d.attack_ptr, n, keep_a.as<uint8_t>(), keep_n.as<uint8_t>(), removed.as<uint8_t>());
    DevBuf idx[3];
    size_t cnt[3];
    const uint8_t* flags[3] = {keep_a.as<uint8_t>(), keep_n.as<uint8_t>(), removed.as<uint8_t>()};
    select_flagged_n(ctx, flags, 3, n, idx, cnt);
    DevBuf &idx_a = idx[0], &idx_n = idx[1], &idx_r = idx[2];
    const size_t na = cnt[0], nn = cnt[1], nr = cnt[2];
    if (na == 0 || nn == 0) fail(IG_E_DATA, "anti-contradiction filtering emptied a class; training impossible");
    if (nr) {
        std::vector<uint32_t> h(nr);
        read_back(ctx, h.data(), idx_r.p, nr * 4);
        e.removed.assign(h.begin(), h.end());
    }
    for (int cls = 0; cls < 2; ++cls) {
        DevRows& dst = cls == 0 ? e.attack : e.normal;
        const size_t mrows = cls == 0 ? na : nn;
        dst.n = mrows;
        dst.k = k;
        dst.L = e.L;
        dst.buf.alloc(std::max<size_t>(mrows * k, 1) * 8, ctx.stream);
        if (mrows * k)
            IGB_LAUNCH(ctx, gather_rows_idx, grid_for(ctx, mrows * k, 256), 256, 0, all.data(),
                       (cls == 0 ? idx_a : idx_n).as<uint32_t>(), mrows, (int)k, dst.data());
    }
    // no final synchronisation: every consumer of the rows is ordered on this
    // stream (or waits for an event recorded on it), and the queued work reads
    // no host memory (the columns' copies finished before the read-backs
    // above), so the caller's next host work overlaps the gathers
}

void encode_rows_dev(Ctx& ctx, const ig_columns& c, const ig_encoding& train, ig_encoding& e, bool queue_only) {
    if (c.n_cols != train.n_cols || c.label_index != train.label_index)
        fail(IG_E_DATA, "encode_rows: columns do not match the training schema");
    e = ig_encoding{};
    e.L = train.L;
    e.n_cols = train.n_cols;
    e.label_index = train.label_index;
    e.decimals = train.decimals;
    DeviceCols d;
    const bool host_read = upload_and_code(ctx, c, d);
    if (train.dv.valid && train.dv.n_feat == d.n_feat && train.dv.feat_col == d.feat_col) {
        // the training vocabulary's device tables: numeric codes and empty
        // tokens as they are; categorical ids of this table -> training ids
        // through the value text (host, from the two dictionaries) -> bits
        const DeviceVocab& dv = train.dv;
        std::vector<int32_t> remap, train_off;
        std::vector<int> cfeat, coff, clen;
        for (int f = 0; f < d.n_feat; ++f) {
            const int j = d.feat_col[f];
            if (c.kind[j] != 1) continue;
            std::unordered_map<std::string, int32_t> tid;
            for (size_t i = 0; i < train.dict[j].size(); ++i) tid.emplace(train.dict[j][i], (int32_t)i);
            cfeat.push_back(f);
            coff.push_back((int)remap.size());
            clen.push_back((int)c.dict[j].size());
            for (const auto& v : c.dict[j]) {
                auto it = tid.find(v);
                remap.push_back(it == tid.end() ? -1 : it->second);
                train_off.push_back(dv.cat_off[f]);
            }
        }
        DevBuf lut(d.n_feat * sizeof(Lut), ctx.stream), cb(std::max<size_t>(remap.size(), 1) * 4, ctx.stream);
        IGB_CUDA(cudaMemcpyAsync(lut.p, dv.lut, d.n_feat * sizeof(Lut), cudaMemcpyDeviceToDevice, ctx.stream));
        if (!cfeat.empty()) {
            DevBuf rm(remap.size() * 4 + train_off.size() * 4 + cfeat.size() * 12, ctx.stream);
            std::vector<int32_t> host(remap);
            host.insert(host.end(), train_off.begin(), train_off.end());
            for (size_t i = 0; i < cfeat.size(); ++i) {
                host.push_back(cfeat[i]);
                host.push_back(coff[i]);
                host.push_back(clen[i]);
            }
            IGB_CUDA(cudaMemcpyAsync(rm.p, host.data(), host.size() * 4, cudaMemcpyHostToDevice, ctx.stream));
            const int32_t* rmp = rm.as<int32_t>();
            if (!remap.empty())
                IGB_LAUNCH(ctx, remap_cat, grid_for(ctx, remap.size(), 256), 256, 0, rmp, (int)remap.size(),
                           dv.cbits, rmp + remap.size(), cb.as<int32_t>());
            IGB_LAUNCH(ctx, patch_cat_lut, 1, 256, 0, rmp + 2 * remap.size(), (int)cfeat.size(), lut.as<Lut>());
        }
        pack_tables(ctx, train.L, d, lut.as<Lut>(), dv.lcodes, dv.lbits, cb.as<int32_t>(), e.all);
        if (host_read || !queue_only) IGB_CUDA(cudaStreamSynchronize(ctx.stream));
        return;
    }
    train.host_vocab();
    // Categorical ids of this table → training bits through the token text.
    std::vector<std::vector<int32_t>> cat_id_to_bit(c.n_cols);
    for (size_t j = 0; j < c.n_cols; ++j) {
        if (j == c.label_index || c.kind[j] != 1) continue;
        cat_id_to_bit[j].assign(c.dict[j].size(), -1);
        for (size_t id = 0; id < c.dict[j].size(); ++id) {
            auto it = train.cat_bits[j].find(c.dict[j][id]);
            if (it != train.cat_bits[j].end()) cat_id_to_bit[j][id] = it->second;
        }
    }
    pack_with(ctx, train, d, cat_id_to_bit, e.all);
    // copies from the caller's host columns must finish before we return; with
    // resident or prefetched columns the work stays queued on the stream
    if (host_read || !queue_only) IGB_CUDA(cudaStreamSynchronize(ctx.stream));
}

void upload_columns(Ctx& ctx, ig_columns& c) {
    if (c.d_values && c.device == ctx.device) return;  // already resident (uploaded or device-ingested)
    auto up = [&](const void* src, size_t bytes) {
        void* p = nullptr;
        IGB_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 8)));
        if (bytes) IGB_CUDA(cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, ctx.stream));
        return std::shared_ptr<void>(p, [](void* q) { cudaFree(q); });
    };
    c.d_values = up(c.values.data(), c.values.size() * 8);
    c.d_cat = up(c.cat.data(), c.cat.size() * 4);
    c.d_attack = up(c.is_attack.data(), c.is_attack.size());
    c.device = ctx.device;
    IGB_CUDA(cudaStreamSynchronize(ctx.stream));
}

}  // namespace igb
