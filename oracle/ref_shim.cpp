// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (checker / CPU baseline, never the product).
//
// Compiled together with the reference's own four translation units
// (/root/reference/proj/src/{bitpack,csv,kernels,pipeline}.cpp) into
// oracle/_ref/libigref.so by oracle/Makefile.  It does two things:
//
//  1. Supplies the modules the reference snapshot declares but does not ship:
//     `mine` (proj/include/ig/mine.hpp:35-51, semantics SPEC.md:281-354),
//     `purify`, `infer` and the `eval`
//     split/metrics.  They are restated here strictly on top of
//     the reference's own types and primitives (`words::*`, `PackedMatrix`,
//     `KernelBackend` from make_backend()), so the CPU arithmetic *is* the
//     reference's.
//  2. Exposes the reference pipeline and these modules through a flat
//     extern "C" surface so Python tests / bench.py's reference arm can drive
//     them with ctypes.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
// reference) load this library.

#include <algorithm>
#include <atomic>
#include <mutex>
#include <thread>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <omp.h>

#include "ig/bitpack.hpp"
#include "ig/csv.hpp"
#include "ig/errors.hpp"
#include "ig/kernels.hpp"
#include "ig/mine.hpp"
#include "ig/pipeline.hpp"
#include "ig/version.hpp"

#ifdef IG_WITH_B200
#include "ig_b200_backend.hpp"  // integration/: the reference-side binding of libig_b200.so
#endif

namespace ig {

// ---------------------------------------------------------------------------
// mine (mine.hpp:35-51)
// ---------------------------------------------------------------------------
namespace {

// Per-worker exact set of K-word keys: open addressing on words::hash
// (bitpack.hpp:70-78) with full words::equal compare, so the fingerprint is
// only a bucket hint and collisions never merge distinct contents.
class WordSet {
public:
    explicit WordSet(std::size_t k) : k_(k) { rehash(1u << 12); }

    void insert(const std::int64_t* w) {
        if ((count_ + 1) * 2 > slots_.size()) rehash(slots_.size() * 2);
        std::uint64_t h = words::hash(w, k_);
        std::size_t mask = slots_.size() - 1;
        std::size_t s = h & mask;
        while (true) {
            std::uint32_t id = slots_[s];
            if (id == kEmpty) {
                slots_[s] = static_cast<std::uint32_t>(count_);
                hashes_.push_back(h);
                arena_.insert(arena_.end(), w, w + k_);
                ++count_;
                return;
            }
            if (hashes_[id] == h && words::equal(arena_.data() + id * k_, w, k_)) return;
            s = (s + 1) & mask;
        }
    }
    std::size_t size() const { return count_; }
    const std::int64_t* row(std::size_t i) const { return arena_.data() + i * k_; }

private:
    static constexpr std::uint32_t kEmpty = 0xffffffffu;
    void rehash(std::size_t cap) {
        slots_.assign(cap, kEmpty);
        std::size_t mask = cap - 1;
        for (std::size_t id = 0; id < count_; ++id) {
            std::size_t s = hashes_[id] & mask;
            while (slots_[s] != kEmpty) s = (s + 1) & mask;
            slots_[s] = static_cast<std::uint32_t>(id);
        }
    }
    std::size_t k_;
    std::size_t count_ = 0;
    std::vector<std::uint32_t> slots_;
    std::vector<std::uint64_t> hashes_;
    std::vector<std::int64_t> arena_;
};

int resolve_threads(int t) { return t > 0 ? t : omp_get_max_threads(); }

}  // namespace

CandidateSet enumerate_candidates(const PackedMatrix& rows, const KernelBackend& backend,
                                  const KernelConfig& config, const ProgressFn& progress) {
    config.validate();
    const std::size_t n = rows.rows();
    const std::size_t k = rows.word_count();
    if (n == 0) throw DataError("enumerate_candidates: empty class");
    const int workers = resolve_threads(config.threads);
    std::vector<std::unique_ptr<WordSet>> sets(workers);
    for (auto& s : sets) s = std::make_unique<WordSet>(k);
    const std::uint64_t pairs_total = static_cast<std::uint64_t>(n) * (n - 1) / 2;

    // left-index blocks over workers, private maps per worker.
#pragma omp parallel num_threads(workers)
    {
        WordSet& mine = *sets[omp_get_thread_num()];
        std::vector<std::int64_t> buf(config.pair_batch * k);
#pragma omp for schedule(dynamic, 1)
        for (std::size_t i = 0; i < n; ++i) {
            // union term X^c (Eq. 1); empty rows never stored
            if (words::any(rows.row(i), k)) mine.insert(rows.row(i));
            for (std::size_t jb = i + 1; jb < n; jb += config.pair_batch) {
                const std::size_t je = std::min(jb + config.pair_batch, n);
                backend.pair_intersect_batch(rows, i, jb, je, buf.data());
                for (std::size_t t = 0; t < je - jb; ++t) {
                    const std::int64_t* w = buf.data() + t * k;
                    if (words::any(w, k)) mine.insert(w);
                }
            }
        }
    }

    // Deterministic merge in canonical words::less order (mine.hpp:21-22).
    std::vector<const std::int64_t*> all;
    for (auto& s : sets)
        for (std::size_t i = 0; i < s->size(); ++i) all.push_back(s->row(i));
    std::sort(all.begin(), all.end(),
              [k](const std::int64_t* a, const std::int64_t* b) { return words::less(a, b, k); });
    CandidateSet out;
    out.class_tag = rows.class_tag();
    out.source_rows = n;
    out.patterns = PackedMatrix(rows.logical_len(), rows.class_tag());
    out.patterns.reserve_rows(all.size());
    for (std::size_t i = 0; i < all.size(); ++i) {
        if (i > 0 && words::equal(all[i - 1], all[i], k)) continue;
        out.patterns.append_words(all[i]);
    }
    if (progress) progress(pairs_total, pairs_total, out.patterns.rows());
    return out;
}

void count_support(CandidateSet& candidates, const PackedMatrix& rows, const KernelConfig& config) {
    config.validate();
    if (candidates.patterns.logical_len() != rows.logical_len()) {
        throw std::invalid_argument("count_support: logical length mismatch");
    }
    const std::size_t k = rows.word_count();
    const std::size_t np = candidates.patterns.rows();
    candidates.supports.assign(np, 0);
    // recount against all class rows (duplicates included).
#pragma omp parallel for schedule(dynamic, 64) num_threads(resolve_threads(config.threads))
    for (std::size_t p = 0; p < np; ++p) {
        const std::int64_t* pw = candidates.patterns.row(p);
        std::int64_t f = 0;
        for (std::size_t i = 0; i < rows.rows(); ++i) f += words::is_subset(pw, rows.row(i), k);
        candidates.supports[p] = f;
    }
}

void score_patterns(CandidateSet& candidates) {
    const std::size_t np = candidates.patterns.rows();
    if (candidates.supports.size() != np) {
        throw std::invalid_argument("score_patterns: supports not counted");
    }
    const std::size_t k = candidates.patterns.word_count();
    candidates.scores.assign(np, 0);
    for (std::size_t p = 0; p < np; ++p) {
        const std::int64_t size = words::popcount(candidates.patterns.row(p), k);
        std::int64_t sq = 0, s = 0;
        if (__builtin_mul_overflow(size, size, &sq) ||
            __builtin_mul_overflow(candidates.supports[p], sq, &s)) {
            throw ArithmeticError("pattern score overflows int64");
        }
        candidates.scores[p] = s;
    }
}

std::int64_t total_score(const std::vector<std::int64_t>& scores) {
    std::int64_t acc = 0;
    for (std::int64_t s : scores) {
        if (__builtin_add_overflow(acc, s, &acc)) throw ArithmeticError("total score overflows int64");
    }
    return acc;
}

}  // namespace ig

// ---------------------------------------------------------------------------
// purify / infer / eval, restated on the reference types.
// ---------------------------------------------------------------------------
namespace refx {
using namespace ig;

// keep candidates that coverage_any reports not covered.
CandidateSet reject_covered(const CandidateSet& c, const PackedMatrix& opposite,
                            const KernelBackend& backend, std::size_t coverage_block) {
    auto mask = backend.coverage_any(c.patterns, opposite, coverage_block);
    CandidateSet out;
    out.class_tag = c.class_tag;
    out.source_rows = c.source_rows;
    out.patterns = PackedMatrix(c.patterns.logical_len(), c.class_tag);
    for (std::size_t p = 0; p < mask.size(); ++p) {
        if (mask[p]) continue;
        out.patterns.append_words(c.patterns.row(p));
        if (!c.supports.empty()) out.supports.push_back(c.supports[p]);
        if (!c.scores.empty()) out.scores.push_back(c.scores[p]);
    }
    return out;
}

struct NormalStats {
    double mu = 0, sigma = 0;
};

// mean / population std over strictly positive N; <2 positives -> 0,0.
NormalStats fit_normal_stats(const std::vector<std::int64_t>& nvals) {
    std::vector<double> pos;
    for (auto v : nvals)
        if (v > 0) pos.push_back(static_cast<double>(v));
    NormalStats st;
    if (pos.size() < 2) return st;
    double sum = 0;
    for (double v : pos) sum += v;
    st.mu = sum / static_cast<double>(pos.size());
    double ss = 0;
    // Written as the FMA the -march=native build (proj/CMakeLists.txt:10-18)
    // contracts this loop to, so the rounding does not depend on compiler flags.
    for (double v : pos) ss = std::fma(v - st.mu, v - st.mu, ss);
    st.sigma = std::sqrt(ss / static_cast<double>(pos.size()));
    return st;
}

// SPEC.md:444-452. Returns label (1 attack) and regulation code:
// 1 = R1-attack, 2 = R1-normal, 3 = R2, 4 = R3.
inline void classify(std::int64_t a, std::int64_t n, const NormalStats& st, double r,
                     std::uint8_t* label, std::uint8_t* reg) {
    if (a == 0 && n == 0) {
        *label = 1;
        *reg = 3;
    } else if (a >= n) {
        *label = 1;
        *reg = 1;
    } else if (static_cast<double>(n) < std::fma(-r, st.sigma, st.mu)) {  // mu - r*sigma, contracted
        *label = 1;
        *reg = 4;
    } else {
        *label = 0;
        *reg = 2;
    }
}

}  // namespace refx

// ---------------------------------------------------------------------------
// extern "C" surface
// ---------------------------------------------------------------------------
namespace {

thread_local std::string g_err;

// make_backend (kernels.cpp:188-194) plus the "b200" registration a maintainer
// adds when this shim is linked against libig_b200.so.
std::unique_ptr<ig::KernelBackend> backend_for(const char* name, int threads) {
#ifdef IG_WITH_B200
    if (std::string(name) == "b200") return ig::make_b200_backend(0);
#endif
    return ig::make_backend(name, threads);
}

enum Status : int {
    OK = 0,
    E_INVALID = 1,
    E_RANGE = 2,
    E_CONFIG = 3,
    E_IO = 4,
    E_DATA = 5,
    E_ARITH = 6,
    E_OTHER = 7,
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return OK;
    } catch (const ig::ConfigError& e) {
        g_err = e.what();
        return E_CONFIG;
    } catch (const ig::IoError& e) {
        g_err = e.what();
        return E_IO;
    } catch (const ig::DataError& e) {
        g_err = e.what();
        return E_DATA;
    } catch (const ig::ArithmeticError& e) {
        g_err = e.what();
        return E_ARITH;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return E_INVALID;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return E_RANGE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return E_OTHER;
    }
}

ig::PackedMatrix to_matrix(const std::int64_t* w, std::size_t n, std::uint32_t L,
                           ig::ClassTag tag = ig::ClassTag::unlabeled) {
    ig::PackedMatrix m(L, tag);
    m.reserve_rows(n);
    const std::size_t k = ig::words::count_for(L);
    for (std::size_t i = 0; i < n; ++i) m.append_words(w + i * k);
    return m;
}

std::vector<std::string> split_list(const char* s) {
    std::vector<std::string> out;
    if (!s || !*s) return out;
    std::string cur;
    for (const char* p = s; *p; ++p) {
        if (*p == ',') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += *p;
        }
    }
    out.push_back(cur);
    return out;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Cand {
    ig::CandidateSet c;
};

// One full IG run (fit + predict) on a CSV, driven through the reference pipeline.
struct Run {
    ig::Table train, test;
    ig::DatasetSchema schema;
    ig::TrainingEncoding enc;
    ig::PackedMatrix tests;
    std::vector<std::uint8_t> truth;
    ig::CandidateSet cand[2];  // 0 attack, 1 normal
    ig::CandidateSet pure[2];
    std::vector<std::int64_t> A, N;
    std::vector<std::uint8_t> label, reg;
    refx::NormalStats stats;
    std::string vocab_blob;  // tokens joined by '\n'
    std::vector<std::uint64_t> removed_rows;
    double t[8] = {0};  // parse, encode, enumerate, support(+score), purify, match, test_encode, total
};

}  // namespace

extern "C" {

const char* igref_last_error() { return g_err.c_str(); }
const char* igref_version() { return ig::version_string; }
int igref_max_threads() { return omp_get_max_threads(); }

int igref_format_zscore(double z, int decimals, char* buf, std::size_t cap) {
    return guard([&] {
        std::string s = ig::format_zscore(z, decimals);
        std::snprintf(buf, cap, "%s", s.c_str());
    });
}

// ---- KernelBackend primitives (kernels.hpp:27-58) ----
int igref_pair_intersect_batch(const char* backend, int threads, const std::int64_t* rows,
                               std::size_t n, std::uint32_t L, std::size_t left, std::size_t jb,
                               std::size_t je, std::int64_t* out) {
    return guard([&] {
        auto be = backend_for(backend, threads);
        be->pair_intersect_batch(to_matrix(rows, n, L), left, jb, je, out);
    });
}

int igref_coverage_any(const char* backend, int threads, const std::int64_t* pat, std::size_t np,
                       std::uint32_t Lp, const std::int64_t* opp, std::size_t no, std::uint32_t Lo,
                       std::size_t block, std::uint8_t* mask) {
    return guard([&] {
        auto be = backend_for(backend, threads);
        auto m = be->coverage_any(to_matrix(pat, np, Lp), to_matrix(opp, no, Lo), block);
        std::memcpy(mask, m.data(), m.size());
    });
}

int igref_fused_score(const char* backend, int threads, const std::int64_t* pat, std::size_t np,
                      std::uint32_t Lp, const std::int64_t* scores, std::size_t ns,
                      const std::int64_t* tests, std::size_t nt, std::uint32_t Lt,
                      std::int64_t* out) {
    return guard([&] {
        auto be = backend_for(backend, threads);
        auto v = be->fused_score(to_matrix(pat, np, Lp), std::span<const std::int64_t>(scores, ns),
                                 to_matrix(tests, nt, Lt));
        std::memcpy(out, v.data(), v.size() * sizeof(std::int64_t));
    });
}

// ---- mine (mine.hpp:35-51) ----
int igref_enumerate(const char* backend, int threads, std::size_t pair_batch,
                    const std::int64_t* rows, std::size_t n, std::uint32_t L, void** out) {
    return guard([&] {
        auto be = backend_for(backend, threads);
        ig::KernelConfig cfg;
        cfg.pair_batch = pair_batch;
        cfg.threads = threads;
        auto c = std::make_unique<Cand>();
        c->c = ig::enumerate_candidates(to_matrix(rows, n, L), *be, cfg);
        *out = c.release();
    });
}
void igref_cand_free(void* c) { delete static_cast<Cand*>(c); }
std::size_t igref_cand_count(void* c) { return static_cast<Cand*>(c)->c.patterns.rows(); }
const std::int64_t* igref_cand_words(void* c) { return static_cast<Cand*>(c)->c.patterns.data(); }
const std::int64_t* igref_cand_supports(void* c) { return static_cast<Cand*>(c)->c.supports.data(); }
const std::int64_t* igref_cand_scores(void* c) { return static_cast<Cand*>(c)->c.scores.data(); }
int igref_count_support(void* c, int threads, const std::int64_t* rows, std::size_t n,
                        std::uint32_t L) {
    return guard([&] {
        ig::KernelConfig cfg;
        cfg.threads = threads;
        ig::count_support(static_cast<Cand*>(c)->c, to_matrix(rows, n, L), cfg);
    });
}
int igref_score_patterns(void* c) {
    return guard([&] { ig::score_patterns(static_cast<Cand*>(c)->c); });
}
int igref_total_score(const std::int64_t* s, std::size_t n, std::int64_t* out) {
    return guard([&] { *out = ig::total_score(std::vector<std::int64_t>(s, s + n)); });
}

// ---- pipeline (pipeline.hpp) ----
// Encode a CSV (bytes) as the training table: returns L and the packed class
// matrices plus the vocabulary as '\n'-joined tokens.
int igref_run_create(const char* csv, std::size_t len, const char* label_col,
                     const char* attack_values, const char* normal_values, int decimals,
                     int ratio_k, std::size_t train_rows_override, const char* backend,
                     int threads, std::size_t pair_batch, std::size_t coverage_block,
                     std::size_t test_offset, std::size_t test_limit, int stages, double r, void** out) {
    return guard([&] {
        auto run = std::make_unique<Run>();
        double t0 = now_s();
        std::istringstream in(std::string(csv, len));
        ig::Table all = ig::read_csv(in, "<csv>");
        // positional split, first floor(k/10 * n) rows train.
        std::size_t n = all.rows.size();
        std::size_t ntr = train_rows_override ? train_rows_override
                                              : static_cast<std::size_t>(ratio_k) * n / 10;
        if (ratio_k < 0 || ratio_k > 10 || ntr > n) throw ig::ConfigError("bad ratio");
        run->train.header = all.header;
        run->test.header = all.header;
        run->train.rows.assign(all.rows.begin(), all.rows.begin() + ntr);
        run->test.rows.assign(all.rows.begin() + ntr, all.rows.end());
        // a bounded sample of the test rows: [test_offset, test_offset + test_limit)
        // (bench.py's reference arm rotates the offset across steps)
        if (test_offset) {
            const std::size_t off = std::min(test_offset, run->test.rows.size());
            run->test.rows.erase(run->test.rows.begin(), run->test.rows.begin() + off);
        }
        if (test_limit < run->test.rows.size()) run->test.rows.resize(test_limit);
        double t1 = now_s();
        run->t[0] = t1 - t0;

        run->schema = ig::infer_schema(run->train, label_col, split_list(attack_values),
                                       split_list(normal_values), decimals);
        run->enc = ig::encode_training(run->train, run->schema);
        double t2 = now_s();
        run->t[1] = t2 - t1;
        for (const auto& tok : run->enc.vocabulary.tokens()) {
            run->vocab_blob += tok;
            run->vocab_blob += '\n';
        }
        for (auto r0 : run->enc.filter_report.removed_rows) run->removed_rows.push_back(r0);
        if (stages <= 0) {
            *out = run.release();
            return;
        }

        auto be = backend_for(backend, threads);
        ig::KernelConfig cfg;
        cfg.pair_batch = pair_batch;
        cfg.coverage_block = coverage_block;
        cfg.threads = threads;
        const ig::PackedMatrix* X[2] = {&run->enc.attack, &run->enc.normal};
        double ta = now_s();
        for (int c = 0; c < 2; ++c) run->cand[c] = ig::enumerate_candidates(*X[c], *be, cfg);
        double tb = now_s();
        run->t[2] = tb - ta;
        for (int c = 0; c < 2; ++c) {
            ig::count_support(run->cand[c], *X[c], cfg);
            ig::score_patterns(run->cand[c]);
            ig::total_score(run->cand[c].scores);
        }
        double tc = now_s();
        run->t[3] = tc - tb;
        for (int c = 0; c < 2; ++c)
            run->pure[c] = refx::reject_covered(run->cand[c], *X[1 - c], *be, cfg.coverage_block);
        double td = now_s();
        run->t[4] = td - tc;
        if (stages <= 1) {
            *out = run.release();
            return;
        }

        double te0 = now_s();
        ig::check_schema_compatible(run->test, run->schema);
        run->tests = ig::encode_rows(run->test, run->schema, run->enc.vocabulary);
        run->truth = ig::truth_labels(run->test, run->schema);
        double te1 = now_s();
        run->t[6] = te1 - te0;
        // SPEC.md:424-428 evidence_scores
        run->A = be->fused_score(run->pure[0].patterns, run->pure[0].scores, run->tests);
        run->N = be->fused_score(run->pure[1].patterns, run->pure[1].scores, run->tests);
        double tf = now_s();
        run->t[5] = tf - te1;
        run->stats = refx::fit_normal_stats(run->N);
        run->label.resize(run->A.size());
        run->reg.resize(run->A.size());
        for (std::size_t i = 0; i < run->A.size(); ++i)
            refx::classify(run->A[i], run->N[i], run->stats, r, &run->label[i], &run->reg[i]);
        run->t[7] = now_s() - t0;
        *out = run.release();
    });
}

void igref_run_free(void* r) { delete static_cast<Run*>(r); }
std::uint32_t igref_run_L(void* r) { return static_cast<Run*>(r)->enc.vocabulary.size(); }
const char* igref_run_vocab(void* r) { return static_cast<Run*>(r)->vocab_blob.c_str(); }
std::size_t igref_run_rows(void* r, int which) {
    Run* R = static_cast<Run*>(r);
    switch (which) {
        case 0: return R->enc.attack.rows();
        case 1: return R->enc.normal.rows();
        case 2: return R->tests.rows();
        case 3: return R->removed_rows.size();
        case 4: return R->train.rows.size();
        case 5: return R->test.rows.size();
    }
    return 0;
}
const std::int64_t* igref_run_matrix(void* r, int which) {
    Run* R = static_cast<Run*>(r);
    switch (which) {
        case 0: return R->enc.attack.data();
        case 1: return R->enc.normal.data();
        case 2: return R->tests.data();
    }
    return nullptr;
}
const std::uint64_t* igref_run_removed(void* r) { return static_cast<Run*>(r)->removed_rows.data(); }
// which: 0/1 candidates attack/normal, 2/3 pure attack/normal; field 0 words,1 supports,2 scores
std::size_t igref_run_dict_count(void* r, int which) {
    Run* R = static_cast<Run*>(r);
    return which < 2 ? R->cand[which].patterns.rows() : R->pure[which - 2].patterns.rows();
}
const std::int64_t* igref_run_dict(void* r, int which, int field) {
    Run* R = static_cast<Run*>(r);
    const ig::CandidateSet& c = which < 2 ? R->cand[which] : R->pure[which - 2];
    if (field == 0) return c.patterns.data();
    if (field == 1) return c.supports.data();
    return c.scores.data();
}
const std::int64_t* igref_run_evidence(void* r, int which) {
    Run* R = static_cast<Run*>(r);
    return which == 0 ? R->A.data() : R->N.data();
}
const std::uint8_t* igref_run_labels(void* r, int which) {
    Run* R = static_cast<Run*>(r);
    return which == 0 ? R->label.data() : which == 1 ? R->reg.data() : R->truth.data();
}
void igref_run_stats(void* r, double* mu, double* sigma) {
    Run* R = static_cast<Run*>(r);
    *mu = R->stats.mu;
    *sigma = R->stats.sigma;
}
const double* igref_run_times(void* r) { return static_cast<Run*>(r)->t; }
// schema: per column kind (0 numeric, 1 categorical), mean, std
void igref_run_schema(void* r, std::uint8_t* kind, double* mean, double* sd, std::size_t* label_index) {
    Run* R = static_cast<Run*>(r);
    for (std::size_t j = 0; j < R->schema.columns.size(); ++j) {
        kind[j] = R->schema.columns[j].kind == ig::ColumnKind::numeric ? 0 : 1;
        mean[j] = R->schema.columns[j].mean;
        sd[j] = R->schema.columns[j].stddev;
    }
    *label_index = R->schema.label_index;
}
std::size_t igref_run_cols(void* r) { return static_cast<Run*>(r)->schema.columns.size(); }


#ifdef IG_WITH_B200
// kernels.hpp:23-26 under concurrency: `threads` host threads share ONE "b200"
// backend object and call pair_intersect_batch / coverage_any / fused_score on
// shared read-only inputs, `iters` times each, with thread-dependent windows;
// every result is compared with ParallelCpuBackend's.  Returns the number of
// mismatching results in *mismatches.
int igref_b200_concurrency(const std::int64_t* rows, std::size_t n, std::uint32_t L, const std::int64_t* pats,
                           std::size_t np, const std::int64_t* scores, int threads, int iters,
                           std::uint64_t* mismatches, std::uint64_t* calls) {
    return guard([&] {
        ig::PackedMatrix X(L, ig::ClassTag::attack), P(L, ig::ClassTag::attack);
        const std::size_t k = X.word_count();
        for (std::size_t i = 0; i < n; ++i) X.append_words(rows + i * k);
        for (std::size_t i = 0; i < np; ++i) P.append_words(pats + i * k);
        std::vector<std::int64_t> sc(scores, scores + np);
        auto b200 = backend_for("b200", 0);
        auto cpu = ig::make_backend("parallel-cpu", 1);
        const auto cov_want = cpu->coverage_any(P, X, 4096);
        const auto fs_want = cpu->fused_score(P, sc, X);
        std::atomic<std::uint64_t> bad{0}, ncalls{0};
        std::atomic<bool> failed{false};
        std::string first_err;
        std::mutex err_mu;
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) {
            pool.emplace_back([&, t] {
                try {
                    for (int it = 0; it < iters; ++it) {
                        const std::size_t left = (std::size_t)(t * 7 + it * 3) % (n - 1);
                        const std::size_t jb = left + 1, je = std::min(n, jb + 1 + (std::size_t)(t * 13 + it) % 97);
                        std::vector<std::int64_t> got((je - jb) * k), want((je - jb) * k);
                        b200->pair_intersect_batch(X, left, jb, je, got.data());
                        cpu->pair_intersect_batch(X, left, jb, je, want.data());
                        bad += got != want;
                        const std::size_t block = 1 + (std::size_t)(t * 31 + it) % 5000;  // never changes results
                        bad += b200->coverage_any(P, X, block) != cov_want;
                        bad += b200->fused_score(P, sc, X) != fs_want;
                        ncalls += 3;
                    }
                } catch (const std::exception& e) {
                    std::lock_guard<std::mutex> lk(err_mu);
                    if (!failed.exchange(true)) first_err = e.what();
                }
            });
        }
        for (auto& th : pool) th.join();
        if (failed) throw std::runtime_error("b200 backend call failed under concurrency: " + first_err);
        *mismatches = bad;
        *calls = ncalls;
    });
}

// enumerate_candidates on the device with a ProgressFn (mine.hpp:31-40):
// records how often it was called, whether pairs_done and candidates_found
// never decreased, and the last triple; returns the candidates' words.
int igref_b200_enumerate_progress(const std::int64_t* rows, std::size_t n, std::uint32_t L, std::uint64_t* ncalls,
                                  int* monotone, std::uint64_t* last3, void** out) {
    return guard([&] {
        ig::PackedMatrix X(L, ig::ClassTag::attack);
        for (std::size_t i = 0; i < n; ++i) X.append_words(rows + i * X.word_count());
        std::uint64_t calls = 0, pd = 0, cf = 0;
        bool mono = true;
        std::uint64_t last[3] = {0, 0, 0};
        ig::ProgressFn fn = [&](std::uint64_t done, std::uint64_t total, std::uint64_t found) {
            ++calls;
            mono = mono && done >= pd && found >= cf && done <= total;
            pd = done;
            cf = found;
            last[0] = done;
            last[1] = total;
            last[2] = found;
        };
        ig::KernelConfig cfg;
        auto c = std::make_unique<Cand>();
        c->c = ig::b200_enumerate_candidates(X, cfg, fn);
        *ncalls = calls;
        *monotone = mono ? 1 : 0;
        std::copy(last, last + 3, last3);
        *out = c.release();
    });
}
#endif

}  // extern "C"
