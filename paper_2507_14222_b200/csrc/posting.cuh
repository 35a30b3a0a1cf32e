// posting.cuh — posting-bitmap (vertical) subset tests; see posting.cu.
#pragma once

#include "ig_internal.cuh"

namespace igb {

// Postings of a row set: bit r of post[t] set iff row r contains bit t, for all
// 64*K bit positions (padding bits included, so any input is handled exactly).
struct Postings {
    uint32_t L = 0;      // bit positions covered (64 * K)
    size_t n = 0;        // posting rows (distinct rows when built with distinct = true)
    size_t n_src = 0;    // source rows
    size_t W = 0;        // words per posting = ceil(n / 64)
    uint32_t nz_total = 0;
    DevBuf dense;        // L x W u64
    DevBuf df;           // L u32: rows containing the bit
    DevBuf nz_off;       // L+1 u32: CSR offsets of non-zero words
    DevBuf nz_idx;       // non-zero word indices
    DevBuf perm;         // canonical position i = source row perm[i]; empty = identity
    DevBuf group;        // canonical position i -> posting row (distinct builds only)
    DevBuf rep;          // posting row -> source row (distinct builds only)
};

bool postings_supported(uint32_t L, size_t n);
// canonical: index rows in words::less order (clusters rows that share tokens).
// distinct: one posting row per distinct row (for coverage / evidence, where
// multiplicity does not matter or is restored by `group`); never for support.
void build_postings(Ctx& ctx, const int64_t* d_rows, size_t n, size_t k, uint32_t L, Postings& P,
                    bool canonical = true, bool distinct = false, const uint32_t* d_perm = nullptr);
void posting_support(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, int64_t* d_support);
void posting_cover(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const Postings& P, uint8_t* d_mask);
// d_out[source row] (P.n int64) is zeroed and accumulated; requires all scores >= 0.
// sum_fits: caller proved Σ scores <= INT64_MAX (no overflow check needed).
void posting_match(Ctx& ctx, const int64_t* d_pat, size_t np, size_t k, const int64_t* d_scores, const Postings& P,
                   int64_t* d_out, int* d_overflow, bool sum_fits);

}  // namespace igb
