/* oracle/ig_oracle.c — TEST INFRASTRUCTURE ONLY: the plain-C CPU restatement
 * of the IG hot path that tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg use as the CHECKER of the CUDA path.  Never linked into,
 * loaded by, or called from the product library.
 *
 * Each function restates the reference semantics it cites:
 *   words::is_subset / popcount / less     proj/include/ig/bitpack.hpp:31-68
 *   pair window AND                       proj/src/kernels.cpp:50-57
 *   coverage_any (first-hit early exit)    proj/src/kernels.cpp:59-65,89-103
 *   fused_score (checked int64, p order)   proj/src/kernels.cpp:40-46,67-77,105-118
 *   enumerate_candidates                  proj/include/ig/mine.hpp:35-40
 *   count_support                         proj/include/ig/mine.hpp:42-44
 *   score_patterns / total_score          proj/include/ig/mine.hpp:46-51
 *   reject_covered
 *
 * Pinned against: the SPEC known answers (tests/golden/spec_examples.json) and
 * fixtures produced by the reference itself (oracle/_ref, tests/golden/*.npz,
 * made by tests/golden/make_golden.py).
 *
 * Status codes follow include/ig_b200.h: 0 ok, 1 invalid argument, 5 data,
 * 6 arithmetic overflow.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef int64_t i64;
typedef uint64_t u64;

static inline int is_subset(const i64* p, const i64* x, size_t k) {
    for (size_t w = 0; w < k; ++w)
        if ((p[w] & x[w]) != p[w]) return 0;
    return 1;
}
static inline int popcount_k(const i64* a, size_t k) {
    int n = 0;
    for (size_t w = 0; w < k; ++w) n += __builtin_popcountll((u64)a[w]);
    return n;
}
static inline int any_k(const i64* a, size_t k) {
    for (size_t w = 0; w < k; ++w)
        if (a[w]) return 1;
    return 0;
}
/* canonical order: lexicographic on words viewed unsigned (bitpack.hpp:59-68) */
static inline int cmp_k(const i64* a, const i64* b, size_t k) {
    for (size_t w = 0; w < k; ++w) {
        u64 ua = (u64)a[w], ub = (u64)b[w];
        if (ua != ub) return ua < ub ? -1 : 1;
    }
    return 0;
}
static inline u64 mix(const i64* a, size_t k) {
    u64 h = 0x243f6a8885a308d3ull;
    for (size_t w = 0; w < k; ++w) {
        h += (u64)a[w] + 0x9e3779b97f4a7c15ull;
        h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ull;
        h = (h ^ (h >> 27)) * 0x94d049bb133111ebull;
        h ^= h >> 31;
    }
    return h;
}

/* ---------------- exact K-word set (open addressing, full compare) ---------------- */
typedef struct {
    size_t k, count, cap;
    uint32_t* slot;
    u64* hash;
    i64* arena;
    size_t arena_cap;
} wset;

static void ws_init(wset* s, size_t k) {
    s->k = k;
    s->count = 0;
    s->cap = 1u << 12;
    s->slot = (uint32_t*)malloc(s->cap * sizeof(uint32_t));
    memset(s->slot, 0xff, s->cap * sizeof(uint32_t));
    s->arena_cap = 1024;
    s->hash = (u64*)malloc(s->arena_cap * sizeof(u64));
    s->arena = (i64*)malloc(s->arena_cap * k * sizeof(i64));
}
static void ws_free(wset* s) {
    free(s->slot);
    free(s->hash);
    free(s->arena);
}
static void ws_grow(wset* s) {
    size_t cap = s->cap * 2;
    uint32_t* slot = (uint32_t*)malloc(cap * sizeof(uint32_t));
    memset(slot, 0xff, cap * sizeof(uint32_t));
    for (size_t id = 0; id < s->count; ++id) {
        size_t p = s->hash[id] & (cap - 1);
        while (slot[p] != 0xffffffffu) p = (p + 1) & (cap - 1);
        slot[p] = (uint32_t)id;
    }
    free(s->slot);
    s->slot = slot;
    s->cap = cap;
}
static void ws_insert(wset* s, const i64* w) {
    if ((s->count + 1) * 2 > s->cap) ws_grow(s);
    u64 h = mix(w, s->k);
    size_t p = h & (s->cap - 1);
    for (;;) {
        uint32_t id = s->slot[p];
        if (id == 0xffffffffu) break;
        if (s->hash[id] == h && cmp_k(s->arena + (size_t)id * s->k, w, s->k) == 0) return;
        p = (p + 1) & (s->cap - 1);
    }
    if (s->count == s->arena_cap) {
        s->arena_cap *= 2;
        s->hash = (u64*)realloc(s->hash, s->arena_cap * sizeof(u64));
        s->arena = (i64*)realloc(s->arena, s->arena_cap * s->k * sizeof(i64));
    }
    s->slot[p] = (uint32_t)s->count;
    s->hash[s->count] = h;
    memcpy(s->arena + s->count * s->k, w, s->k * sizeof(i64));
    s->count++;
}

/* ---------------- merge sort of row pointers in canonical order ---------------- */
static void msort(const i64** a, const i64** tmp, size_t n, size_t k) {
    if (n < 2) return;
    if (n <= 16) {
        for (size_t i = 1; i < n; ++i) {
            const i64* v = a[i];
            size_t j = i;
            while (j > 0 && cmp_k(a[j - 1], v, k) > 0) {
                a[j] = a[j - 1];
                --j;
            }
            a[j] = v;
        }
        return;
    }
    size_t h = n / 2;
    if (n > 65536) {
#pragma omp task shared(a, tmp)
        msort(a, tmp, h, k);
        msort(a + h, tmp + h, n - h, k);
#pragma omp taskwait
    } else {
        msort(a, tmp, h, k);
        msort(a + h, tmp + h, n - h, k);
    }
    size_t i = 0, j = h, o = 0;
    while (i < h && j < n) tmp[o++] = (cmp_k(a[j], a[i], k) < 0) ? a[j++] : a[i++];
    while (i < h) tmp[o++] = a[i++];
    while (j < n) tmp[o++] = a[j++];
    memcpy(a, tmp, n * sizeof(*a));
}

/* ---------------- public (ctypes) surface ---------------- */
typedef struct {
    size_t n, k;
    i64* words;
} igo_set;

size_t igo_set_count(const igo_set* s) { return s->n; }
const i64* igo_set_words(const igo_set* s) { return s->words; }
void igo_set_free(igo_set* s) {
    if (!s) return;
    free(s->words);
    free(s);
}

/* enumerate_candidates: {X_i & X_j : i<j, non-empty} ∪ {X_i non-empty}, dedup,
 * canonical order. */
int igo_enumerate(const i64* rows, size_t n, size_t k, int threads, igo_set** out) {
    if (n == 0) return 5;
    int T = threads > 0 ? threads : omp_get_max_threads();
    wset* sets = (wset*)malloc(sizeof(wset) * T);
    for (int t = 0; t < T; ++t) ws_init(&sets[t], k);
#pragma omp parallel num_threads(T)
    {
        wset* s = &sets[omp_get_thread_num()];
        i64* tmp = (i64*)malloc(k * sizeof(i64));
#pragma omp for schedule(dynamic, 1)
        for (size_t i = 0; i < n; ++i) {
            const i64* xi = rows + i * k;
            if (any_k(xi, k)) ws_insert(s, xi);
            for (size_t j = i + 1; j < n; ++j) {
                const i64* xj = rows + j * k;
                int nz = 0;
                for (size_t w = 0; w < k; ++w) nz |= ((tmp[w] = xi[w] & xj[w]) != 0);
                if (nz) ws_insert(s, tmp);
            }
        }
        free(tmp);
    }
    size_t total = 0;
    for (int t = 0; t < T; ++t) total += sets[t].count;
    const i64** ptr = (const i64**)malloc((total ? total : 1) * sizeof(*ptr));
    const i64** tmpp = (const i64**)malloc((total ? total : 1) * sizeof(*ptr));
    size_t o = 0;
    for (int t = 0; t < T; ++t)
        for (size_t i = 0; i < sets[t].count; ++i) ptr[o++] = sets[t].arena + i * k;
#pragma omp parallel num_threads(T)
#pragma omp single
    msort(ptr, tmpp, total, k);
    igo_set* res = (igo_set*)malloc(sizeof(igo_set));
    res->k = k;
    res->words = (i64*)malloc((total ? total : 1) * k * sizeof(i64));
    size_t m = 0;
    for (size_t i = 0; i < total; ++i) {
        if (i > 0 && cmp_k(ptr[i - 1], ptr[i], k) == 0) continue;
        memcpy(res->words + m * k, ptr[i], k * sizeof(i64));
        ++m;
    }
    res->n = m;
    free(ptr);
    free(tmpp);
    for (int t = 0; t < T; ++t) ws_free(&sets[t]);
    free(sets);
    *out = res;
    return 0;
}

/* support[p] = #{i : P_p ⊆ X_i} over all class rows, duplicates included. */
int igo_count_support(const i64* pat, size_t np, const i64* rows, size_t n, size_t k, int threads,
                      i64* support) {
    int T = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(T)
    for (size_t p = 0; p < np; ++p) {
        i64 f = 0;
        const i64* pw = pat + p * k;
        for (size_t i = 0; i < n; ++i) f += is_subset(pw, rows + i * k, k);
        support[p] = f;
    }
    return 0;
}

/* score = support * size^2, checked (mine.hpp:46-48). */
int igo_score(const i64* pat, const i64* support, size_t np, size_t k, i64* score) {
    for (size_t p = 0; p < np; ++p) {
        i64 sz = popcount_k(pat + p * k, k), sq, s;
        if (__builtin_mul_overflow(sz, sz, &sq) || __builtin_mul_overflow(support[p], sq, &s)) return 6;
        score[p] = s;
    }
    return 0;
}

int igo_total_score(const i64* s, size_t n, i64* out) {
    i64 acc = 0;
    for (size_t i = 0; i < n; ++i)
        if (__builtin_add_overflow(acc, s[i], &acc)) return 6;
    *out = acc;
    return 0;
}

/* mask[p] = 1 iff some opponent row ⊇ P_p (kernels.cpp:59-65). */
int igo_coverage_any(const i64* pat, size_t np, const i64* opp, size_t no, size_t k, int threads,
                     uint8_t* mask) {
    int T = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(T)
    for (size_t p = 0; p < np; ++p) {
        uint8_t c = 0;
        for (size_t t = 0; t < no && !c; ++t) c = (uint8_t)is_subset(pat + p * k, opp + t * k, k);
        mask[p] = c;
    }
    return 0;
}

/* out[t] = Σ_p s_p [P_p ⊆ T_t], checked_add in pattern order (kernels.cpp:40-46,67-77). */
int igo_fused_score(const i64* pat, const i64* s, size_t np, const i64* tests, size_t nt, size_t k,
                    int threads, i64* out) {
    int T = threads > 0 ? threads : omp_get_max_threads();
    int overflow = 0;
#pragma omp parallel for schedule(dynamic, 16) num_threads(T) reduction(| : overflow)
    for (size_t t = 0; t < nt; ++t) {
        i64 acc = 0;
        const i64* tw = tests + t * k;
        for (size_t p = 0; p < np; ++p) {
            if (is_subset(pat + p * k, tw, k) && __builtin_add_overflow(acc, s[p], &acc)) {
                overflow = 1;
                break;
            }
        }
        out[t] = acc;
    }
    return overflow ? 6 : 0;
}

/* reject_covered: keep uncovered rows of (pat, support, score) in place; returns kept count. */
size_t igo_reject_covered(i64* pat, i64* support, i64* score, size_t np, const i64* opp, size_t no,
                          size_t k, int threads) {
    uint8_t* mask = (uint8_t*)malloc(np ? np : 1);
    igo_coverage_any(pat, np, opp, no, k, threads, mask);
    size_t m = 0;
    for (size_t p = 0; p < np; ++p) {
        if (mask[p]) continue;
        if (m != p) {
            memmove(pat + m * k, pat + p * k, k * sizeof(i64));
            support[m] = support[p];
            score[m] = score[p];
        }
        ++m;
    }
    free(mask);
    return m;
}
