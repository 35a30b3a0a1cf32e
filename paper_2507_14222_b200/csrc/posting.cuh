// posting.cuh — posting-bitmap (vertical) subset tests; see posting.cu.
#pragma once

#include <memory>

#include "ig_internal.cuh"

namespace igb {

// Postings of a row set: bit r of post[t] set iff row r contains bit t, for all
// 64*K bit positions (padding bits included, so any input is handled exactly).
struct Postings {
    uint32_t L = 0;      // bit positions covered (64 * K)
    size_t n = 0;        // posting rows (distinct rows when built with distinct = true)
    size_t n_src = 0;    // source rows
    size_t W = 0;        // words per posting = ceil(n / 64)
    DevBuf dense;        // L x W u64
    DevBuf df;           // L u32: rows containing the bit
    DevBuf nz_off;       // L+1 u32: CSR offsets of non-zero words
    DevBuf nz_idx;       // non-zero word indices
    DevBuf perm;         // canonical position i = source row perm[i]; empty = identity
    DevBuf group;        // canonical position i -> posting row (distinct builds only)
    DevBuf rep;          // posting row -> source row (distinct builds only)
};

// Token rank space: tokens ordered by (document frequency, id), rarest first.
struct RankSpace {
    uint32_t L = 0;
    DevBuf df;      // L u32
    DevBuf rank;    // L u16: token -> rank
    DevBuf byrank;  // L u16: rank -> token
};

// A pattern set's scan index, independent of the postings it is scanned
// against: CSR token lists (rarest first in a rank space) and the patterns
// grouped by their three rarest tokens (t1, t2, t3) under (t1, t2) parents.
struct PatternIndex {
    size_t np = 0;   // patterns
    size_t G = 0;    // groups
    DevBuf beg;      // np u32: start of each pattern's token list in *toks
    DevBuf len;      // np u32: its length
    std::shared_ptr<DevBuf> toks;  // u16 tokens (shared by subset indexes)
    DevBuf order;    // np u32: patterns in group-key order
    DevBuf gid;      // np u32: group of each ordered position
    DevBuf gkey;     // G u64: (t1 << 32) | (t2 << 16) | t3
    size_t G2 = 0;   // parent groups (t1, t2)
    DevBuf pid;      // G u32: parent of each group
    DevBuf pkey;     // G2 u32: (t1 << 16) | t2
    // Optional: scan only these positions (of the group order), nsel of them —
    // a subset of the patterns (the pure ones among the candidates) without a
    // re-built index; pattern ids (and scores) stay the full set's.
    DevBuf sel;
    size_t nsel = 0;
};

// descending: most frequent first (default: rarest first)
void make_rank_space(Ctx& ctx, const uint32_t* d_df, uint32_t L, RankSpace& R, bool descending = false);
// Clustering order of rows for postings and pair tiles: lexicographic in
// reflected-Gray order over the tokens ranked most frequent first.  Rows
// containing the same frequent tokens become contiguous, so a pattern's hits
// form fewer, longer runs (C3 matcher -18% vs words::less); identical rows are
// adjacent.  Not the canonical order (that one is only needed for output).
void cluster_order(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, uint32_t* d_perm);
// df = A.df + B.df (postings of the two training classes)
void combined_rank_space(Ctx& ctx, const Postings& A, const Postings& B, RankSpace& R);
// max_tokens: an upper bound on a pattern's token count (0: unknown)
void build_pattern_index(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const RankSpace& R, PatternIndex& I,
                         uint32_t max_tokens = 0);
void group_ids(Ctx& ctx, const unsigned long long* d_sorted_key, size_t np, PatternIndex& I);
// index of the patterns S.pattern[d_src_of[i]], i < n (a subset, e.g. the pure
// patterns among the candidates), without re-ranking or re-sorting
void subset_pattern_index(Ctx& ctx, const PatternIndex& S, const uint32_t* d_src_of, size_t n, PatternIndex& I);
// I.sel = the positions (group order) whose pattern is not flagged, in order
// (count: how many there are, known to the caller)
size_t select_unflagged_positions(Ctx& ctx, PatternIndex& I, const uint8_t* d_flag, size_t count);

bool postings_supported(uint32_t L, size_t n);
// canonical: index rows in words::less order (clusters rows that share tokens).
// distinct: one posting row per distinct row (for coverage / evidence, where
// multiplicity does not matter or is restored by `group`); never for support.
void build_postings(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, uint32_t L, Postings& P,
                    bool canonical = true, bool distinct = false, const uint32_t* d_perm = nullptr);
// I: the patterns' scan index (nullptr: built here, ranked by P's frequencies)
void posting_support(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, int64_t* d_support,
                     const PatternIndex* I = nullptr);
void posting_cover(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, uint8_t* d_mask,
                   const PatternIndex* I = nullptr);
// d_out[source row] (P.n int64) is zeroed and accumulated; requires all scores >= 0.
// sum_fits: caller proved Σ scores <= INT64_MAX (no overflow check needed).
void posting_match(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* d_scores, const Postings& P,
                   int64_t* d_out, int* d_overflow, bool sum_fits, const PatternIndex* I = nullptr);

}  // namespace igb
