// subset.cuh — host entry points of the subset-test kernels (subset.cu) and the
// mining kernels (mine.cu).  Device pointers throughout; k = words per row.
#pragma once

#include <vector>

#include "ig_internal.cuh"

namespace igb {

void measure_int_peaks(Ctx& ctx, double* lop3_per_s, double* popc_per_s);

// mask[p] = 1 iff some opponent row ⊇ pattern p (kernels.cpp:59-65).
void coverage_any_dev(Ctx& ctx, const int64_t* d_pat, size_t np, const int64_t* d_opp, size_t no,
                      size_t k, uint8_t* d_mask);
// support[p] = #{i : pattern p ⊆ rows[i]}.
void count_support_dev(Ctx& ctx, const int64_t* d_pat, size_t np, const int64_t* d_rows, size_t n,
                       size_t k, int64_t* d_support);
// out[t] = Σ_p s_p [p ⊆ t] with the reference's overflow semantics; returns
// IG_OK or IG_E_OVERFLOW (kernels.cpp:40-46,67-77).
int fused_score_dev(Ctx& ctx, const int64_t* d_pat, size_t np, const int64_t* d_scores,
                    const int64_t* d_tests, size_t nt, size_t k, int64_t* d_out);

// out[t] = left & rows[t] (kernels.cpp:50-57), one launch for the window.
void pair_window_dev(Ctx& ctx, const int64_t* d_left, const int64_t* d_rows, size_t cnt, size_t k, int64_t* d_out);

// Distinct non-empty {X_u & X_v : u <= v} of one class (u == v gives the
// union term X^c), unordered.  Exact: fingerprints only pick the bucket.
struct EnumStats {
    uint64_t pairs = 0;       // unordered pairs of the input rows (i < j), as the reference counts them
    uint64_t distinct_rows = 0;  // rows actually paired (identical rows collapse)
    uint64_t table_slots = 0; // final hash capacity
    int retries = 0;          // capacity growths
    int levels = 0;           // collision levels used (1 = no fingerprint collision)
    uint64_t collisions = 0;  // inserts that met an equal fingerprint of different content
};
void enumerate_dev(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, uint32_t L, DevRows& out,
                   EnumStats* stats, const uint32_t* d_perm = nullptr);

// Which pairs of the (distinct, canonical) rows to insert: the tiles
// tile_begin, tile_begin + tile_step, ... of the u <= v triangle, or an explicit
// list of (u, v) row pairs (multi-GPU owner phase).
struct PairSource {
    uint64_t tile_begin = 0, tile_step = 1;
    const uint2* list = nullptr;
    uint64_t n_list = 0;
};
// Exact dedup of the non-empty pair intersections of `src`: one representative
// (u, v) per distinct content -> reps_out; returns the count.
uint64_t dedup_pairs(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, const PairSource& src, DevBuf& reps_out,
                     EnumStats* stats);
void materialize_pairs(Ctx& ctx, const int64_t* d_rows, size_t k, const uint2* d_reps, uint64_t count, uint32_t L,
                       DevRows& out);
// Multi-GPU: route representatives to their owner rank (fingerprint of the
// content mod world).  send gets the records grouped by destination; counts[world].
void bucket_by_owner(Ctx& ctx, const int64_t* d_rows, size_t k, const uint2* d_reps, uint64_t count, int world,
                     DevBuf& send, std::vector<uint64_t>& counts);

// score[p] = support[p] * popcount(p)^2 with overflow flag (mine.hpp:46-48).
// Returns IG_OK / IG_E_OVERFLOW.
int score_dev(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* d_support,
              int64_t* d_score);
// Checked Σ scores (mine.hpp:50-51) -> IG_OK / IG_E_OVERFLOW.
int total_score_dev(Ctx& ctx, const int64_t* d_score, size_t np, int64_t* total);
// both, with one read-back (IG_E_OVERFLOW if either overflows)
int score_total_dev(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* d_support, int64_t* d_score,
                    int64_t* total);
unsigned score_total_launch(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* d_support,
                            int64_t* d_score, DevBuf& buf);
int score_total_collect(Ctx& ctx, const DevBuf& buf, unsigned g, int64_t* total);

// Keep rows whose flag is 0 (stable), with their supports/scores.
size_t compact_unflagged(Ctx& ctx, const int64_t* d_words, const int64_t* d_sup, const int64_t* d_sc,
                         const uint8_t* d_flag, size_t n, size_t k, int64_t* o_words, int64_t* o_sup,
                         int64_t* o_sc, DevBuf* o_idx = nullptr);  // o_idx: kept position -> source index

// Reorder rows (+ optional per-row int64 payloads) into canonical words::less order.
// o_perm (optional): canonical position -> previous position (left empty when n < 2).
void canonical_order(Ctx& ctx, DevRows& rows, DevBuf* a, DevBuf* b, DevBuf* o_perm = nullptr);
// out[i] = a[b ? b[i] : i]
void compose_u32(Ctx& ctx, const uint32_t* a, const uint32_t* b, size_t n, uint32_t* out);

}  // namespace igb
