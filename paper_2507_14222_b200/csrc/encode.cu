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
#include <limits>
#include <string>
#include <unordered_map>
#include <unordered_set>

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
    int kind;      // 0 numeric (sorted codes + bits), 1 categorical (id → bit)
    int off, len;  // into codes/bits arrays
    int empty_bit; // bit of the "j:" token or -1
};

__device__ __forceinline__ int lookup(const Lut& L, int64_t code, const int64_t* __restrict__ lcodes,
                                      const int32_t* __restrict__ lbits) {
    if (code == kEmptyCode) return L.empty_bit;
    if (L.kind == 1) return (code >= 0 && code < L.len) ? lbits[L.off + code] : -1;
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
                           const int64_t* __restrict__ lcodes, const int32_t* __restrict__ lbits, int k,
                           unsigned long long* __restrict__ rows) {
    const size_t total = (size_t)n_feat * n;
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (size_t)gridDim.x * blockDim.x) {
        const int f = (int)(q / n);
        const size_t r = q % n;
        const int bit = lookup(luts[f], codes[q], lcodes, lbits);
        if (bit >= 0) atomicOr(rows + r * k + (bit >> 6), 1ull << (bit & 63));
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
size_t select_flagged(Ctx& ctx, const uint8_t* d_flags, size_t n, DevBuf& idx_out) {
    DevBuf iota(n * 4, ctx.stream), nsel(8, ctx.stream);
    idx_out.alloc(std::max<size_t>(n, 1) * 4, ctx.stream);
    IGB_LAUNCH(ctx, iota32, grid_for(ctx, n, 256), 256, 0, iota.as<uint32_t>(), n);
    size_t tb = 0;
    IGB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.as<uint32_t>(), d_flags, idx_out.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)n, ctx.stream));
    DevBuf temp(tb, ctx.stream);
    IGB_CUDA(cub::DeviceSelect::Flagged(temp.p, tb, iota.as<uint32_t>(), d_flags, idx_out.as<uint32_t>(),
                                        nsel.as<int64_t>(), (int64_t)n, ctx.stream));
    int64_t m = 0;
    read_back(ctx, &m, nsel.p, 8);
    return (size_t)m;
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

// Upload a vocabulary's lookup tables and pack `d`'s cells into rows.
void pack_with(Ctx& ctx, const ig_encoding& e, const DeviceCols& d,
               const std::vector<std::vector<int32_t>>& cat_id_to_bit, DevRows& out) {
    std::vector<Lut> luts(d.n_feat);
    std::vector<int64_t> lcodes;
    std::vector<int32_t> lbits;
    for (int f = 0; f < d.n_feat; ++f) {
        const int j = d.feat_col[f];
        Lut& L = luts[f];
        L.empty_bit = e.empty_bit[j];
        L.off = (int)lbits.size();
        if (e.kind[j] == 0) {
            L.kind = 0;
            L.len = (int)e.num_codes[j].size();
            lcodes.insert(lcodes.end(), e.num_codes[j].begin(), e.num_codes[j].end());
            lbits.insert(lbits.end(), e.num_bits[j].begin(), e.num_bits[j].end());
        } else {
            L.kind = 1;
            L.len = (int)cat_id_to_bit[j].size();
            lcodes.resize(lcodes.size() + cat_id_to_bit[j].size(), 0);
            lbits.insert(lbits.end(), cat_id_to_bit[j].begin(), cat_id_to_bit[j].end());
        }
    }
    DevBuf dl(std::max<size_t>(luts.size(), 1) * sizeof(Lut), ctx.stream);
    DevBuf dc(std::max<size_t>(lcodes.size(), 1) * 8, ctx.stream), db(std::max<size_t>(lbits.size(), 1) * 4, ctx.stream);
    if (!luts.empty())
        IGB_CUDA(cudaMemcpyAsync(dl.p, luts.data(), luts.size() * sizeof(Lut), cudaMemcpyHostToDevice, ctx.stream));
    if (!lcodes.empty())
        IGB_CUDA(cudaMemcpyAsync(dc.p, lcodes.data(), lcodes.size() * 8, cudaMemcpyHostToDevice, ctx.stream));
    if (!lbits.empty())
        IGB_CUDA(cudaMemcpyAsync(db.p, lbits.data(), lbits.size() * 4, cudaMemcpyHostToDevice, ctx.stream));
    out.L = e.L;
    out.k = words_for(e.L);
    out.n = d.n;
    out.buf.alloc(std::max<size_t>(out.n * out.k, 1) * 8, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(out.buf.p, 0, std::max<size_t>(out.n * out.k, 1) * 8, ctx.stream));
    const size_t cells = (size_t)d.n_feat * d.n;
    if (cells && out.k)
        IGB_LAUNCH(ctx, pack_cells, grid_for(ctx, cells, 256), 256, 0, d.codes.as<int64_t>(), d.n, d.n_feat,
                   dl.as<Lut>(), dc.as<int64_t>(), db.as<int32_t>(), (int)out.k,
                   reinterpret_cast<unsigned long long*>(out.data()));
    // Lookup tables are freed stream-ordered after the kernel.
}

}  // namespace

void prefetch_columns(Ctx& ctx, ig_columns& c) {
    if (c.d_values && c.device == ctx.device) return;  // already resident
    auto pf = std::make_shared<PrefetchCols>();
    pf->device = ctx.device;
    pf->values.alloc(std::max<size_t>(c.values.size(), 1) * 8, ctx.copy);
    pf->cat.alloc(std::max<size_t>(c.cat.size(), 1) * 4, ctx.copy);
    pf->attack.alloc(std::max<size_t>(c.is_attack.size(), 1), ctx.copy);
    if (!c.values.empty())
        IGB_CUDA(cudaMemcpyAsync(pf->values.p, c.values.data(), c.values.size() * 8, cudaMemcpyHostToDevice, ctx.copy));
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
    DeviceCols d;
    upload_and_code(ctx, c, d);

    // (1b) distinct (column, code) over ALL training rows (vocabulary precedes the filter).
    const size_t chunks = (d.n + kDistinctRows - 1) / kDistinctRows;
    const size_t cap = std::max<size_t>((size_t)d.n_feat * d.n, 1);
    DevBuf lcode(cap * 8, ctx.stream), lcol(cap * 4, ctx.stream), lcnt(8, ctx.stream);
    IGB_CUDA(cudaMemsetAsync(lcnt.p, 0, 8, ctx.stream));
    if (d.n && d.n_feat)
        IGB_CUDA(cudaFuncSetAttribute(distinct_codes, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kDistinctSlots * (int)sizeof(int64_t)));
    if (d.n && d.n_feat)
        IGB_LAUNCH(ctx, distinct_codes, dim3((unsigned)chunks, (unsigned)d.n_feat), 256,
                   kDistinctSlots * sizeof(int64_t), d.codes.as<int64_t>(), d.n,
                   lcode.as<int64_t>(), lcol.as<int32_t>(), lcnt.as<unsigned long long>());
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
    DevRows all;
    pack_with(ctx, e, d, cat_id_to_bit, all);
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
    DevBuf idx_a, idx_n, idx_r;
    const size_t na = select_flagged(ctx, keep_a.as<uint8_t>(), n, idx_a);
    const size_t nn = select_flagged(ctx, keep_n.as<uint8_t>(), n, idx_n);
    const size_t nr = select_flagged(ctx, removed.as<uint8_t>(), n, idx_r);
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
    IGB_CUDA(cudaStreamSynchronize(ctx.stream));
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
