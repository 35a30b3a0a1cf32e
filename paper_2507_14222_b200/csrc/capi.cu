// capi.cu — the extern "C" boundary (include/ig_b200.h) and the fit
// orchestration.  Every entry point validates like the reference does
// (kernels.cpp:12-36, 93, 110, 143, 160; bitpack.cpp:53-58), runs on the
// context stream, and converts internal errors into ig_status codes.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <unordered_map>
#include <map>
#include <mutex>
#include <exception>
#include <future>
#include <utility>
#include <string>
#include <thread>
#include <vector>

#include "encode.cuh"
#include "host_pipeline.hpp"
#include "ig_b200.h"
#include "ig_internal.cuh"
#include "posting.cuh"
#include "subset.cuh"

// A context serialises the ABI calls made on it (kernels.hpp:23-26: backend
// methods may be called concurrently; callers wanting parallelism use one
// context per thread, as integration/ig_b200_backend.cpp does).  Recursive:
// an entry point may call another.
struct ig_ctx : igb::Ctx {
    std::recursive_mutex mu;
    std::unique_ptr<igb::Worker> class_worker;  // igb::Ctx::worker
    std::unique_ptr<igb::Worker> index_bg, vocab_bg;  // igb::Ctx::index_worker, vocab_worker
};

struct ig_candidates {
    igb::DevRows rows;
    igb::DevBuf support, score;
    bool has_support = false, has_score = false;
    bool ordered = true;  // rows in canonical words::less order
    uint64_t pairs = 0;
};

struct ig_model {
    uint32_t L = 0;
    bool sum_fits = true;  // Σ scores of each dictionary <= INT64_MAX (fit: checked on the candidates)
    uint64_t partial_total[2] = {0, 0};  // Σ candidate scores per class (checked)
    ig_candidates cand[2];
    ig_candidates pure[2];
    // scan index of each pure dictionary, built by fit; evidence reuses it for
    // every test batch: the candidates' index (token lists ranked by the
    // training rows' frequencies, grouped by rarest pair) with the pure
    // patterns' positions selected (pidx[c].sel), and the candidates' scores
    // in that index's pattern ids (pscore: the candidate set itself may be
    // reordered on copy-out).  Absent for models assembled from dictionaries.
    igb::PatternIndex pidx[2];
    igb::DevBuf pscore[2];
    bool has_pidx = false;
    double ms[6] = {0, 0, 0, 0, 0, 0};
    igb::EnumStats stats[2];
};

// Background index of a test encoding: its rows are packed on the context's
// index stream (rows_ready) and a host thread builds their postings there
// (done), so a fit issued meanwhile on the other streams overlaps both.
struct RowIndexJob {
    igb::BgTask task;
    igb::Postings P;
    bool has_postings = false;
    cudaEvent_t rows_ready = nullptr, done = nullptr;
    std::exception_ptr err;
    uint64_t launches = 0;
    bool joined = false;
    std::mutex mu;  // an encoding may be used by several contexts / threads
    // join the builder (rethrows its error); launches are added to `ctx` once
    void wait(igb::Ctx* ctx) {
        std::lock_guard<std::mutex> lock(mu);
        if (!joined) {
            task.join();
            joined = true;
            if (ctx) ctx->launches += launches;
        }
        if (err) std::rethrow_exception(err);
    }
    ~RowIndexJob() {
        task.join();
        if (rows_ready) cudaEventDestroy(rows_ready);
        if (done) cudaEventDestroy(done);
    }
};

namespace {

thread_local std::string g_err;

using igb::DevBuf;
using igb::DevRows;
using igb::Error;
using igb::fail;

// Every entry point: the context's call lock, its device, and status codes
// instead of exceptions.  Error text is per calling thread (ig_last_error).
template <class F>
int guard(ig_ctx* ctx, F&& f) {
    std::unique_lock<std::recursive_mutex> lock;
    if (ctx) lock = std::unique_lock<std::recursive_mutex>(ctx->mu);
    try {
        if (ctx) IGB_CUDA(cudaSetDevice(ctx->device));
        f();
        return IG_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        return e.status;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return IG_E_OOM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return IG_E_CUDA;
    }
}

void check_cfg(const ig_kernel_config* cfg) {
    if (!cfg) return;
    // kernels.cpp:12-15
    if (cfg->pair_batch < 1) fail(IG_E_CONFIG, "pair-batch must be >= 1");
    if (cfg->coverage_block < 1) fail(IG_E_CONFIG, "coverage-block must be >= 1");
}

void upload_rows(igb::Ctx& ctx, const int64_t* h, size_t n, uint32_t L, DevRows& d) {
    d.n = n;
    d.k = igb::words_for(L);
    d.L = L;
    const size_t bytes = std::max<size_t>(n * d.k, 1) * 8;
    d.buf.alloc(bytes, ctx.stream);
    if (n * d.k) IGB_CUDA(cudaMemcpyAsync(d.buf.p, h, n * d.k * 8, cudaMemcpyHostToDevice, ctx.stream));
}

// Borrow resident device rows without copying.
struct View {
    const int64_t* p;
    size_t n, k;
};

struct Timer {
    cudaEvent_t e[8];
    int used = 0;
    cudaStream_t s;
    explicit Timer(cudaStream_t st) : s(st) {
        for (auto& x : e) cudaEventCreate(&x);
    }
    ~Timer() {
        for (auto& x : e) cudaEventDestroy(x);
    }
    void mark() { cudaEventRecord(e[used++], s); }
    double ms(int a, int b) {
        float f = 0;
        cudaEventSynchronize(e[b]);
        cudaEventElapsedTime(&f, e[a], e[b]);
        return f;
    }
};

// Run fn(ctx, cls) for the two classes concurrently: class 0 on the calling
// thread and the context stream, class 1 on a second host thread and the
// context's auxiliary stream (ordered after everything already queued on the
// main stream; the main stream waits for it afterwards).  The classes are
// independent within each phase, so their host-side syncs overlap with the
// other class's kernels.
constexpr size_t kConcurrentRows = 40000;        // training rows (C3: 14,851; C4: 118,813)
constexpr size_t kConcurrentCandidates = 12000000;  // shard finish (C4 per rank: ~8.4 M at world 4, ~4.2 M at 8)
constexpr size_t kConcurrentPatterns = 8u << 20; // pure patterns (C3: 2.2 M; C4: 32 M)

template <class F>
void for_both_classes(igb::Ctx& ctx, F&& fn, bool concurrent = true) {
    static const bool serial = getenv("IG_SERIAL_CLASSES") != nullptr;  // profiling: one class at a time
    // diagnostics time each hot kernel alone: the classes run one after the other
    if (!concurrent || serial || ctx.diag) {
        fn(ctx, 0);
        fn(ctx, 1);
        return;
    }
    cudaEvent_t fork, join;
    IGB_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    IGB_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    IGB_CUDA(cudaEventRecord(fork, ctx.stream));
    IGB_CUDA(cudaStreamWaitEvent(ctx.aux, fork, 0));
    igb::Ctx c1 = ctx;
    c1.stream = ctx.aux;
    c1.launches = 0;
    for (auto& d : c1.diag_k) d = igb::DiagStat{};
    std::exception_ptr e0, e1;
    auto run1 = [&] {
        try {
            IGB_CUDA(cudaSetDevice(ctx.device));
            fn(c1, 1);
        } catch (...) {
            e1 = std::current_exception();
        }
    };
    std::thread th;
    std::future<void> done;
    if (ctx.worker)
        done = ctx.worker->submit(run1);
    else
        th = std::thread(run1);
    try {
        fn(ctx, 0);
    } catch (...) {
        e0 = std::current_exception();
    }
    if (ctx.worker)
        done.wait();
    else
        th.join();
    cudaEventRecord(join, c1.stream);
    cudaStreamWaitEvent(ctx.stream, join, 0);
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
    ctx.launches += c1.launches;
    ctx.diag_merge(c1);
    if (e0) std::rethrow_exception(e0);
    if (e1) std::rethrow_exception(e1);
}

// The mining half of cmd_train: for both classes enumerate →
// support → score → total, reject_covered against the opposite
// class, canonical order.
// enumerate = false: m.cand[c].rows already hold the candidates (multi-GPU
// owner shard); only support -> score -> purify -> order run.
// Optional evidence of a test encoding fused into the fit: each class's
// matcher runs on its own stream right after that class's pure dictionary is
// ready, overlapping the other class's fit.
struct FusedEvidence {
    RowIndexJob* job = nullptr;  // the test rows' background index
    int64_t* out[2] = {nullptr, nullptr};
    bool done = false;           // set when both classes' evidence ran here
};

// row_perm (optional): each class's canonical row permutation, already known
// (a shard computed it for its distinct rows).
// pre (optional): each class's training postings, already built on the
// context's aux stream (a shard builds them while its records travel).
// max_row_tokens (optional): an upper bound on the set bits of a training row
// (an encoding's feature count: one token per column), which bounds every
// pattern's token list and spares the index build a read-back.
void fit_impl(igb::Ctx& ctx, View X[2], uint32_t L, ig_model& m, bool enumerate = true, FusedEvidence* ev = nullptr,
              const uint32_t* const* row_perm = nullptr, igb::Postings* pre = nullptr, uint32_t max_row_tokens = 0) {
    m.L = L;
    const size_t k = igb::words_for(L);
    for (int c = 0; c < 2; ++c)
        if (X[c].n == 0) fail(IG_E_DATA, "enumerate_candidates: empty class");
    Timer tm(ctx.stream);
    tm.mark();  // 0
    const bool vertical = igb::postings_supported(L, std::max(X[0].n, X[1].n));
    // Small fits are launch/sync bound: overlap the classes.  Large ones fill the
    // GPU with each class alone, and concurrent multi-GB allocations on two
    // streams only fragment the memory pool, so they run one after the other.
    // (an owner shard's finish: decided by its candidate counts)
    const bool concurrent = enumerate ? X[0].n + X[1].n <= kConcurrentRows
                                      : m.cand[0].rows.n + m.cand[1].rows.n <= kConcurrentCandidates;
    DevBuf perm[2];
    igb::Postings PX[2];
    // phase A1 (per class): canonical row order (shared by enumeration and the
    // postings), candidates, postings
    for_both_classes(ctx, [&](igb::Ctx& cx, int c) {
        igb::Trace tr(cx, "fitA", c);
        const uint32_t* pc;
        if (row_perm && row_perm[c]) {
            pc = row_perm[c];
        } else {
            perm[c].alloc(X[c].n * 4, cx.stream);
            igb::sort_rows_canonical(cx, X[c].p, X[c].n, k, perm[c].as<uint32_t>());
            pc = perm[c].as<uint32_t>();
        }
        tr.mark("sort_rows");
        if (enumerate) {
            igb::enumerate_dev(cx, X[c].p, X[c].n, k, L, m.cand[c].rows, &m.stats[c], pc);
            m.cand[c].pairs = m.stats[c].pairs;
            m.cand[c].ordered = false;
        }
        tr.mark("enumerate");
        // every training row (support counts identical rows);
        // distinct rows weighted by their multiplicity measured slower
        //
        if (vertical && pre && pre[c].L)
            PX[c] = std::move(pre[c]);
        else if (vertical)
            igb::build_postings(cx, X[c].p, X[c].n, k, L, PX[c], true, false, pc);
        tr.mark("postings");
    }, concurrent);
    // one token rank space for every scan of this fit: frequencies over all
    // training rows.  Each candidate set gets one index (token lists + groups)
    // shared by its support and coverage scans; the pure subset inherits it.
    igb::RankSpace R;
    igb::PatternIndex CI[2];
    if (vertical) igb::combined_rank_space(ctx, PX[0], PX[1], R);
    // the test index keeps building on its own stream through phase B; the
    // matchers (phase C) wait for it
    const bool fuse = ev && ev->job && vertical;
    tm.mark();  // 1
    // phase B (per class): candidate index, support, score, checked total, purify
    DevBuf tot_buf[2];
    unsigned tot_g[2] = {0, 0};
    for_both_classes(ctx, [&](igb::Ctx& cx, int c) {
        igb::Trace tr(cx, "fitA", c);
        ig_candidates& C = m.cand[c];
        const size_t np = C.rows.n;
        C.support.alloc(std::max<size_t>(np, 1) * 8, cx.stream);
        C.score.alloc(std::max<size_t>(np, 1) * 8, cx.stream);
        if (vertical) {
            igb::build_pattern_index(cx, C.rows.data(), np, k, R, CI[c], max_row_tokens);
            igb::posting_support(cx, C.rows.data(), np, k, PX[c], C.support.as<int64_t>(), &CI[c]);
        } else {
            igb::count_support_dev(cx, C.rows.data(), np, X[c].p, X[c].n, k, C.support.as<int64_t>());
        }
        tr.mark("support");
        // (the total and the overflow checks are collected at the end of the fit)
        tot_g[c] = igb::score_total_launch(cx, C.rows.data(), np, k, C.support.as<int64_t>(), C.score.as<int64_t>(),
                                           tot_buf[c]);
        C.has_support = C.has_score = true;
        tr.mark("score+total");
        // then (same class, no wait for the other class's support): reject_covered
        // against the other class's postings, compaction, canonical order of the
        // pure dictionary (the model output; the candidate sets B^c are ordered
        // on first copy-out)
        DevBuf mask(std::max<size_t>(np, 1), cx.stream);
        if (vertical && X[1 - c].n > 0)
            igb::posting_cover(cx, C.rows.data(), np, k, PX[1 - c], mask.as<uint8_t>(), &CI[c]);
        else
            igb::coverage_any_dev(cx, C.rows.data(), np, X[1 - c].p, X[1 - c].n, k, mask.as<uint8_t>());
        tr.mark("cover");
        ig_candidates& P = m.pure[c];
        P.rows.k = k;
        P.rows.L = L;
        P.rows.buf.alloc(std::max<size_t>(np * k, 1) * 8, cx.stream);
        P.support.alloc(std::max<size_t>(np, 1) * 8, cx.stream);
        P.score.alloc(std::max<size_t>(np, 1) * 8, cx.stream);
        P.rows.n = igb::compact_unflagged(cx, C.rows.data(), C.support.as<int64_t>(), C.score.as<int64_t>(),
                                          mask.as<uint8_t>(), np, k, P.rows.data(), P.support.as<int64_t>(),
                                          P.score.as<int64_t>(), nullptr);
        P.has_support = P.has_score = true;
        tr.mark("compact");
        igb::canonical_order(cx, P.rows, &P.support, &P.score, nullptr);
        tr.mark("order");
        if (vertical) {
            // the pure dictionary's scan index = the candidates' index with the
            // pure patterns' positions selected (no re-grouping), scores in
            // candidate ids
            igb::select_unflagged_positions(cx, CI[c], mask.as<uint8_t>(), P.rows.n);
            m.pidx[c] = std::move(CI[c]);
            m.pscore[c].alloc(std::max<size_t>(np, 1) * 8, cx.stream);
            if (np)
                IGB_CUDA(cudaMemcpyAsync(m.pscore[c].p, C.score.p, np * 8, cudaMemcpyDeviceToDevice, cx.stream));
            for (DevBuf* b : {&m.pidx[c].beg, &m.pidx[c].len, m.pidx[c].toks.get(), &m.pidx[c].order, &m.pidx[c].gid,
                              &m.pidx[c].gkey, &m.pidx[c].pid, &m.pidx[c].pkey, &m.pidx[c].sel, &m.pscore[c]})
                b->persist();
            tr.mark("pure_index");
        }
        // (no host sync: for_both_classes joins the class streams on the
        // device, so phase C's launches queue behind both phase Bs at once)
    }, concurrent);
    m.has_pidx = vertical;
    // phase C (per class): evidence of the test encoding, once both classes'
    // pure dictionaries are indexed — the matchers fill the GPU, and a class's
    // small index kernels queued behind the other class's matcher would stall
    bool fused = false;
    if (fuse) {
        ev->job->wait(&ctx);  // (built during phases A and B)
        fused = ev->job->has_postings && ev->job->P.L == (uint32_t)(64 * k);
    }
    if (fused) {
        for_both_classes(ctx, [&](igb::Ctx& cx, int c) {
            igb::Trace tr(cx, "fitC", c);
            const ig_candidates& P = m.pure[c];
            // Σ scores <= Σ candidate scores, checked <= INT64_MAX above: unchecked sums
            IGB_CUDA(cudaStreamWaitEvent(cx.stream, ev->job->done, 0));
            igb::posting_match(cx, P.rows.data(), P.rows.n, k, m.pscore[c].as<int64_t>(), ev->job->P, ev->out[c],
                               nullptr, true, &m.pidx[c]);
            tr.mark("evidence");
        }, concurrent);
    }
    if (ev) ev->done = fused;
    tm.mark();  // 2
    IGB_CUDA(cudaStreamSynchronize(ctx.stream));
    IGB_CUDA(cudaStreamSynchronize(ctx.aux));
    for (int c = 0; c < 2; ++c) {
        int64_t total = 0;
        if (igb::score_total_collect(ctx, tot_buf[c], tot_g[c], &total) != IG_OK)
            fail(IG_E_OVERFLOW, "pattern score or total score overflows int64");
        m.partial_total[c] = (uint64_t)total;
    }
    m.ms[0] = 0;
    m.ms[1] = tm.ms(0, 1);  // canonical rows + enumerate + postings (both classes, concurrent)
    m.ms[2] = 0;
    m.ms[3] = tm.ms(1, 2);  // index + support + score + purify + order
    m.ms[4] = 0;
    m.ms[5] = tm.ms(0, 2);
    for (int c = 0; c < 2; ++c) {
        for (ig_candidates* C : {&m.cand[c], &m.pure[c]}) {
            C->rows.buf.persist();
            C->support.persist();
            C->score.persist();
        }
    }
}

void copy_out(igb::Ctx& ctx, ig_candidates& c, int64_t* words, int64_t* sup, int64_t* sc) {
    // the first copy-out orders the set in place; concurrent readers of one set
    // (from different contexts) wait for that
    static std::mutex order_mu;
    std::lock_guard<std::mutex> lock(order_mu);
    if (!c.ordered) {
        igb::canonical_order(ctx, c.rows, c.has_support ? &c.support : nullptr, c.has_score ? &c.score : nullptr);
        c.rows.buf.persist();
        c.support.persist();
        c.score.persist();
        c.ordered = true;
    }
    const size_t n = c.rows.n, k = c.rows.k;
    if (words && n * k)
        IGB_CUDA(cudaMemcpyAsync(words, c.rows.data(), n * k * 8, cudaMemcpyDeviceToHost, ctx.stream));
    if (sup) {
        if (!c.has_support) fail(IG_E_INVALID_ARG, "supports not counted");
        if (n) IGB_CUDA(cudaMemcpyAsync(sup, c.support.p, n * 8, cudaMemcpyDeviceToHost, ctx.stream));
    }
    if (sc) {
        if (!c.has_score) fail(IG_E_INVALID_ARG, "scores not computed");
        if (n) IGB_CUDA(cudaMemcpyAsync(sc, c.score.p, n * 8, cudaMemcpyDeviceToHost, ctx.stream));
    }
    IGB_CUDA(cudaStreamSynchronize(ctx.stream));
}

void evidence_impl(igb::Ctx& ctx, const ig_model& m, const int64_t* d_tests, size_t nt, uint32_t L, int64_t* d_A,
                   int64_t* d_N, const igb::Postings* pre = nullptr) {
    if (L != m.L) fail(IG_E_INVALID_ARG, "fused_score: logical length mismatch");
    const size_t k = igb::words_for(L);
    // Fit scores are support * size^2 >= 0, so the vertical matcher applies;
    // test-row postings are built once and shared by both dictionaries.
    if (igb::postings_supported(L, nt)) {
        igb::Trace tr(ctx, "evidence", -1);
        igb::Postings own;
        if (!pre) igb::build_postings(ctx, d_tests, nt, k, L, own, true, true);
        const igb::Postings& PT = pre ? *pre : own;
        tr.mark("test_postings");
        DevBuf flag(sizeof(int), ctx.stream);
        IGB_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx.stream));
        for_both_classes(ctx, [&](igb::Ctx& cx, int c) {
            const ig_candidates& P = m.pure[c];
            // the fit checked Σ candidate scores <= INT64_MAX (total_score); pure ⊆ candidates
            igb::Trace trc(cx, "evidence", c);
            igb::posting_match(cx, P.rows.data(), P.rows.n, k,
                               m.has_pidx ? m.pscore[c].as<int64_t>() : P.score.as<int64_t>(), PT,
                               c == 0 ? d_A : d_N, flag.as<int>(), m.sum_fits, m.has_pidx ? &m.pidx[c] : nullptr);
            trc.mark("match");
        }, m.pure[0].rows.n + m.pure[1].rows.n <= kConcurrentPatterns);
        int h = 0;
        igb::read_back(ctx, &h, flag.p, sizeof(int));
        if (h) fail(IG_E_OVERFLOW, "evidence score sum overflows int64");
        return;
    }
    for (int c = 0; c < 2; ++c) {
        const ig_candidates& P = m.pure[c];
        if (igb::fused_score_dev(ctx, P.rows.data(), P.rows.n, P.score.as<int64_t>(), d_tests, nt, k,
                                 c == 0 ? d_A : d_N) != IG_OK)
            fail(IG_E_OVERFLOW, "evidence score sum overflows int64");
    }
}

}  // namespace

namespace igb {
void set_last_error(const std::string& msg) { g_err = msg; }
}  // namespace igb

extern "C" {

const char* ig_version(void) { return "ig_b200 0.2.0 (sm_100a)"; }

const char* ig_last_error(const ig_ctx* /*ctx*/) { return g_err.c_str(); }

void ig_kernel_config_default(ig_kernel_config* cfg) {
    cfg->pair_batch = 8192;  // kernels.hpp:15-18 defaults
    cfg->coverage_block = 4096;
    cfg->memory_budget_bytes = size_t{2} << 30;
    cfg->threads = 0;
}

int ig_ctx_create(int device, ig_ctx** out) {
    *out = nullptr;
    auto c = std::make_unique<ig_ctx>();
    c->device = device;
    int st = guard(c.get(), [&] {
        c->class_worker = std::make_unique<igb::Worker>(device);
        c->worker = c->class_worker.get();
        c->index_bg = std::make_unique<igb::Worker>(device);
        c->index_worker = c->index_bg.get();
        c->vocab_bg = std::make_unique<igb::Worker>(device);
        c->vocab_worker = c->vocab_bg.get();
        IGB_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
        IGB_CUDA(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
        IGB_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        IGB_CUDA(cudaStreamCreateWithFlags(&c->index, cudaStreamNonBlocking));
        c->stream = c->own;
        cudaDeviceProp prop;
        IGB_CUDA(cudaGetDeviceProperties(&prop, device));
        c->sm_count = prop.multiProcessorCount;
        c->smem_optin = prop.sharedMemPerBlockOptin;
        if (prop.major < 10) fail(IG_E_CUDA, std::string("device ") + prop.name + " is not sm_100-class");
        cudaMemPool_t pool;
        IGB_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        IGB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        // Map the working set once: growing the pool later (new physical pages)
        // costs ~100 ms per first-time allocation pattern inside a fit.
        size_t free_b = 0, total_b = 0;
        IGB_CUDA(cudaMemGetInfo(&free_b, &total_b));
        // (C4 alone measured 370 ms per step with 24 GB — the pool kept growing —
        // and 136 ms with 60 GB)
        size_t reserve = std::min<size_t>(free_b / 2, size_t{64} << 30);
        if (const char* e = getenv("IG_POOL_RESERVE_GB")) reserve = (size_t)(atof(e) * (1ull << 30));
        if (reserve) {
            void* p = nullptr;
            if (cudaMallocAsync(&p, reserve, c->own) == cudaSuccess) cudaFreeAsync(p, c->own);
            cudaGetLastError();
            IGB_CUDA(cudaStreamSynchronize(c->own));
        }
    });
    if (st != IG_OK) return st;
    *out = c.release();
    return IG_OK;
}

void ig_ctx_destroy(ig_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    for (cudaStream_t st : {ctx->own, ctx->aux, ctx->copy, ctx->index}) {
        if (!st) continue;
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    delete ctx;
}

int ig_ctx_set_stream(ig_ctx* ctx, void* stream) {
    return guard(ctx, [&] { ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own; });
}

uint64_t ig_ctx_launch_count(const ig_ctx* ctx) {
    if (!ctx) return 0;
    std::lock_guard<std::recursive_mutex> lock(const_cast<ig_ctx*>(ctx)->mu);
    return ctx->launches;
}

int ig_ctx_set_diagnostics(ig_ctx* ctx, int on) {
    return guard(ctx, [&] {
        ctx->diag = on != 0;
        for (auto& d : ctx->diag_k) d = igb::DiagStat{};
    });
}

int ig_ctx_diag_kernel(ig_ctx* ctx, int kernel, double* kernel_ms, uint64_t* word_ands, uint64_t* launches) {
    return guard(ctx, [&] {
        if (kernel < 0 || kernel >= igb::kDiagKinds) fail(IG_E_INVALID_ARG, "diag: unknown kernel id");
        const igb::DiagStat& d = ctx->diag_k[kernel];
        if (kernel_ms) *kernel_ms = d.ms;
        if (word_ands) *word_ands = d.work;
        if (launches) *launches = d.launches;
    });
}

int ig_measure_int_peaks(ig_ctx* ctx, double* lop3_per_s, double* popc_per_s) {
    return guard(ctx, [&] { igb::measure_int_peaks(*ctx, lop3_per_s, popc_per_s); });
}

// ------------------------------------------------------------------ KernelBackend
int ig_pair_intersect_batch(ig_ctx* ctx, const int64_t* rows, size_t n, uint32_t L, size_t left, size_t jb,
                            size_t je, int64_t* out) {
    return guard(ctx, [&] {
        // kernels.cpp:19-32
        if (left >= n) fail(IG_E_INVALID_ARG, "pair_intersect_batch: left index out of range");
        if (jb <= left)
            fail(IG_E_INVALID_ARG,
                 "pair_intersect_batch: window overlaps [0, left]; only ordered pairs left < j are valid");
        if (je < jb || je > n) fail(IG_E_INVALID_ARG, "pair_intersect_batch: window out of range");
        const size_t k = igb::words_for(L);
        const size_t cnt = je - jb;
        if (cnt == 0 || k == 0) return;
        DevRows d;
        upload_rows(*ctx, rows + jb * k, cnt, L, d);
        DevRows l;
        upload_rows(*ctx, rows + left * k, 1, L, l);
        DevBuf o(cnt * k * 8, ctx->stream);
        igb::pair_window_dev(*ctx, l.data(), d.data(), cnt, k, o.as<int64_t>());
        IGB_CUDA(cudaMemcpyAsync(out, o.p, cnt * k * 8, cudaMemcpyDeviceToHost, ctx->stream));
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int ig_coverage_any(ig_ctx* ctx, const int64_t* pat, size_t np, uint32_t Lp, const int64_t* opp, size_t no,
                    uint32_t Lo, size_t block, uint8_t* mask) {
    return guard(ctx, [&] {
        if (Lp != Lo) fail(IG_E_INVALID_ARG, "coverage_any: logical length mismatch");  // kernels.cpp:34-38
        if (block < 1) fail(IG_E_INVALID_ARG, "coverage_block must be >= 1");          // kernels.cpp:93
        if (np == 0) return;
        DevRows P, X;
        upload_rows(*ctx, pat, np, Lp, P);
        upload_rows(*ctx, opp, no, Lo, X);
        DevBuf m(np, ctx->stream);
        igb::coverage_any_dev(*ctx, P.data(), np, X.data(), no, P.k, m.as<uint8_t>());
        IGB_CUDA(cudaMemcpyAsync(mask, m.p, np, cudaMemcpyDeviceToHost, ctx->stream));
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int ig_fused_score(ig_ctx* ctx, const int64_t* pat, size_t np, uint32_t Lp, const int64_t* scores, size_t ns,
                   const int64_t* tests, size_t nt, uint32_t Lt, int64_t* out) {
    return guard(ctx, [&] {
        if (Lp != Lt) fail(IG_E_INVALID_ARG, "fused_score: logical length mismatch");
        if (ns != np) fail(IG_E_INVALID_ARG, "fused_score: scores length != pattern count");  // kernels.cpp:110
        if (nt == 0) return;
        DevRows P, T;
        upload_rows(*ctx, pat, np, Lp, P);
        upload_rows(*ctx, tests, nt, Lt, T);
        DevBuf s(std::max<size_t>(np, 1) * 8, ctx->stream), o(nt * 8, ctx->stream);
        if (np) IGB_CUDA(cudaMemcpyAsync(s.p, scores, np * 8, cudaMemcpyHostToDevice, ctx->stream));
        if (igb::fused_score_dev(*ctx, P.data(), np, s.as<int64_t>(), T.data(), nt, P.k, o.as<int64_t>()) != IG_OK)
            fail(IG_E_OVERFLOW, "evidence score sum overflows int64");
        IGB_CUDA(cudaMemcpyAsync(out, o.p, nt * 8, cudaMemcpyDeviceToHost, ctx->stream));
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ------------------------------------------------------------------ mine
int ig_enumerate_candidates(ig_ctx* ctx, const int64_t* rows, size_t n, uint32_t L, const ig_kernel_config* cfg,
                            ig_progress_fn progress, void* user, ig_candidates** out) {
    *out = nullptr;
    return guard(ctx, [&] {
        check_cfg(cfg);
        if (n == 0) fail(IG_E_DATA, "enumerate_candidates: empty class");
        DevRows X;
        upload_rows(*ctx, rows, n, L, X);
        auto c = std::make_unique<ig_candidates>();
        igb::EnumStats st;
        // progress (mine.hpp:31-33): pairs done over the pairs (u <= v) of the
        // distinct rows the device enumerates, candidates found so far
        igb::ProgressHook hook;
        struct Mapped {
            unsigned long long* h = nullptr;
            ~Mapped() {
                if (h) cudaFreeHost(h);
            }
        } mapped;
        igb::DevBuf pctr;
        if (progress) {
            IGB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&mapped.h), 2 * sizeof(unsigned long long),
                                   cudaHostAllocMapped));
            mapped.h[0] = mapped.h[1] = 0;
            IGB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&hook.dev), mapped.h, 0));
            pctr.alloc(8, ctx->stream);
            IGB_CUDA(cudaMemsetAsync(pctr.p, 0, 8, ctx->stream));
            hook.fn = progress;
            hook.user = user;
            hook.host = mapped.h;
            hook.ctr = pctr.as<unsigned long long>();
            ctx->progress = &hook;
        }
        struct Unhook {
            igb::Ctx& c;
            ~Unhook() { c.progress = nullptr; }
        } unhook{*ctx};
        igb::enumerate_dev(*ctx, X.data(), n, X.k, L, c->rows, &st);
        ctx->progress = nullptr;
        igb::canonical_order(*ctx, c->rows, nullptr, nullptr);
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
        c->rows.buf.persist();
        c->pairs = st.pairs;
        if (progress) {
            const uint64_t m = st.distinct_rows, total = m * (m + 1) / 2;
            progress(total, total, c->rows.n, user);
        }
        *out = c.release();
    });
}

int ig_count_support(ig_ctx* ctx, ig_candidates* c, const int64_t* rows, size_t n, uint32_t L,
                     const ig_kernel_config* cfg) {
    return guard(ctx, [&] {
        check_cfg(cfg);
        if (L != c->rows.L) fail(IG_E_INVALID_ARG, "count_support: logical length mismatch");
        DevRows X;
        upload_rows(*ctx, rows, n, L, X);
        c->support.alloc(std::max<size_t>(c->rows.n, 1) * 8, ctx->stream);
        igb::count_support_dev(*ctx, c->rows.data(), c->rows.n, X.data(), n, X.k, c->support.as<int64_t>());
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
        c->support.persist();
        c->has_support = true;
    });
}

int ig_count_support_rows(ig_ctx* ctx, const int64_t* pat, size_t np, uint32_t Lp, const int64_t* rows, size_t n,
                          uint32_t Lr, int64_t* support) {
    return guard(ctx, [&] {
        if (Lp != Lr) fail(IG_E_INVALID_ARG, "count_support: logical length mismatch");
        if (np == 0) return;
        DevRows P, X;
        upload_rows(*ctx, pat, np, Lp, P);
        upload_rows(*ctx, rows, n, Lr, X);
        DevBuf s(np * 8, ctx->stream);
        igb::count_support_dev(*ctx, P.data(), np, X.data(), n, P.k, s.as<int64_t>());
        IGB_CUDA(cudaMemcpyAsync(support, s.p, np * 8, cudaMemcpyDeviceToHost, ctx->stream));
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int ig_score_patterns(ig_ctx* ctx, ig_candidates* c) {
    return guard(ctx, [&] {
        if (!c->has_support) fail(IG_E_INVALID_ARG, "score_patterns: supports not counted");
        c->score.alloc(std::max<size_t>(c->rows.n, 1) * 8, ctx->stream);
        if (igb::score_dev(*ctx, c->rows.data(), c->rows.n, c->rows.k, c->support.as<int64_t>(),
                           c->score.as<int64_t>()) != IG_OK)
            fail(IG_E_OVERFLOW, "pattern score overflows int64");
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
        c->score.persist();
        c->has_score = true;
    });
}

int ig_total_score(const int64_t* s, size_t n, int64_t* out) {
    return guard(nullptr, [&] {
        int64_t acc = 0;
        for (size_t i = 0; i < n; ++i)
            if (__builtin_add_overflow(acc, s[i], &acc)) fail(IG_E_OVERFLOW, "total score overflows int64");
        *out = acc;
    });
}

int ig_fit_normal_stats(const int64_t* n_vals, size_t n, double* mu, double* sigma) {
    return guard(nullptr, [&] {
        if ((!n_vals && n) || !mu || !sigma) fail(IG_E_INVALID_ARG, "fit_normal_stats: null pointer");
        igb::fit_normal_stats(n_vals, n, mu, sigma);
    });
}

int ig_classify(const int64_t* A, const int64_t* N, size_t n, double mu, double sigma, double r, uint8_t* label,
                uint8_t* regulation) {
    return guard(nullptr, [&] {
        if (n && (!A || !N)) fail(IG_E_INVALID_ARG, "classify: null pointer");
        igb::classify(A, N, n, mu, sigma, r, label, regulation);
    });
}

size_t ig_candidates_count(const ig_candidates* c) { return c ? c->rows.n : 0; }
uint32_t ig_candidates_logical_len(const ig_candidates* c) { return c ? c->rows.L : 0; }

int ig_candidates_copy(ig_ctx* ctx, const ig_candidates* c, int64_t* words, int64_t* sup, int64_t* sc) {
    return guard(ctx, [&] { copy_out(*ctx, const_cast<ig_candidates&>(*c), words, sup, sc); });
}

void ig_candidates_free(ig_candidates* c) { delete c; }

// ------------------------------------------------------------------ fit / evidence
int ig_fit(ig_ctx* ctx, const int64_t* attack, size_t na, const int64_t* normal, size_t nn, uint32_t L,
           const ig_kernel_config* cfg, ig_model** out) {
    *out = nullptr;
    return guard(ctx, [&] {
        check_cfg(cfg);
        DevRows A, N;
        upload_rows(*ctx, attack, na, L, A);
        upload_rows(*ctx, normal, nn, L, N);
        View X[2] = {{A.data(), na, A.k}, {N.data(), nn, N.k}};
        auto m = std::make_unique<ig_model>();
        fit_impl(*ctx, X, L, *m);
        *out = m.release();
    });
}

int ig_fit_device(ig_ctx* ctx, const int64_t* d_attack, size_t na, const int64_t* d_normal, size_t nn, uint32_t L,
                  const ig_kernel_config* cfg, ig_model** out) {
    *out = nullptr;
    return guard(ctx, [&] {
        check_cfg(cfg);
        const size_t k = igb::words_for(L);
        View X[2] = {{d_attack, na, k}, {d_normal, nn, k}};
        auto m = std::make_unique<ig_model>();
        fit_impl(*ctx, X, L, *m);
        *out = m.release();
    });
}

size_t ig_model_count(const ig_model* m, int cls, int which) {
    if (!m || cls < 0 || cls > 1) return 0;
    return which == 0 ? m->cand[cls].rows.n : m->pure[cls].rows.n;
}

uint32_t ig_model_logical_len(const ig_model* m) { return m ? m->L : 0; }

int ig_model_copy(ig_ctx* ctx, const ig_model* m, int cls, int which, int64_t* words, int64_t* sup, int64_t* sc) {
    return guard(ctx, [&] {
        if (cls < 0 || cls > 1) fail(IG_E_INVALID_ARG, "class must be 0 (attack) or 1 (normal)");
        ig_model* mm = const_cast<ig_model*>(m);  // ordering on demand does not change the content
        copy_out(*ctx, which == 0 ? mm->cand[cls] : mm->pure[cls], words, sup, sc);
    });
}

int ig_model_phase_ms(const ig_model* m, double* ms6) {
    if (!m) return IG_E_INVALID_ARG;
    std::memcpy(ms6, m->ms, sizeof(m->ms));
    return IG_OK;
}

void ig_model_free(ig_model* m) { delete m; }

// ------------------------------------------------------------------ page-locked result storage
namespace {
struct HostPool {
    std::mutex mu;
    std::multimap<size_t, void*> free_blocks;  // capacity -> block
    std::unordered_map<void*, size_t> cap;     // every block this pool made
    size_t cached = 0;
    static constexpr size_t kKeep = size_t{16} << 30;  // cached bytes kept for reuse
    ~HostPool() {
        for (auto& kv : free_blocks) cudaFreeHost(kv.second);
    }
};
HostPool& host_pool() {
    static HostPool* p = new HostPool();  // never destroyed: frees may run at interpreter teardown
    return *p;
}
size_t host_class(size_t bytes) {
    if (bytes <= (size_t{1} << 20)) {
        size_t c = 4096;
        while (c < bytes) c <<= 1;
        return c;
    }
    const size_t g = size_t{2} << 20;
    return (bytes + g - 1) / g * g;
}
}  // namespace

int ig_host_alloc(size_t bytes, void** out) {
    *out = nullptr;
    return guard(nullptr, [&] {
        if (bytes == 0) fail(IG_E_INVALID_ARG, "ig_host_alloc: zero bytes");
        const size_t want = host_class(bytes);
        HostPool& P = host_pool();
        {
            std::lock_guard<std::mutex> lk(P.mu);
            auto it = P.free_blocks.lower_bound(want);
            if (it != P.free_blocks.end() && it->first <= 2 * want) {
                *out = it->second;
                P.cached -= it->first;
                P.free_blocks.erase(it);
                return;
            }
        }
        void* p = nullptr;
        if (cudaHostAlloc(&p, want, cudaHostAllocPortable) != cudaSuccess || !p) {
            cudaGetLastError();
            fail(IG_E_OOM, "ig_host_alloc: cannot page-lock " + std::to_string(want) + " bytes");
        }
        std::lock_guard<std::mutex> lk(P.mu);
        P.cap[p] = want;
        *out = p;
    });
}

void ig_host_free(void* p) {
    if (!p) return;
    HostPool& P = host_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.cap.find(p);
    if (it == P.cap.end()) return;  // not ours
    if (P.cached + it->second > HostPool::kKeep) {
        cudaFreeHost(p);
        P.cap.erase(it);
        return;
    }
    P.cached += it->second;
    // LIFO among equal capacities: the block just freed is the next one handed
    // out (its pages are still mapped hot), instead of rotating through all
    // cached blocks of that class
    P.free_blocks.emplace_hint(P.free_blocks.lower_bound(it->second), it->second, p);
}

int ig_evidence(ig_ctx* ctx, const ig_model* m, const int64_t* tests, size_t nt, uint32_t L, int64_t* A, int64_t* N) {
    return guard(ctx, [&] {
        if (nt == 0) return;
        DevRows T;
        upload_rows(*ctx, tests, nt, L, T);
        DevBuf a(nt * 8, ctx->stream), b(nt * 8, ctx->stream);
        evidence_impl(*ctx, *m, T.data(), nt, L, a.as<int64_t>(), b.as<int64_t>());
        igb::copy_to_host(*ctx, A, a.p, nt * 8);
        igb::copy_to_host(*ctx, N, b.p, nt * 8);
    });
}

int ig_evidence_device(ig_ctx* ctx, const ig_model* m, const int64_t* d_tests, size_t nt, uint32_t L, int64_t* d_A,
                       int64_t* d_N) {
    return guard(ctx, [&] {
        if (nt == 0) return;
        evidence_impl(*ctx, *m, d_tests, nt, L, d_A, d_N);
    });
}

// ------------------------------------------------------------------ pipeline
int ig_read_csv(const char* bytes, size_t len, ig_table** out) {
    *out = nullptr;
    return guard(nullptr, [&] {
        auto t = std::make_unique<ig_table>();
        igb::read_csv(bytes, len, *t);
        *out = t.release();
    });
}
size_t ig_table_rows(const ig_table* t) { return t ? t->n_rows : 0; }
size_t ig_table_cols(const ig_table* t) { return t ? t->header.size() : 0; }
int ig_table_slice(const ig_table* t, size_t begin, size_t end, ig_table** out) {
    *out = nullptr;
    return guard(nullptr, [&] {
        if (begin > end || end > t->n_rows) fail(IG_E_INVALID_ARG, "table slice out of range");
        auto s = std::make_unique<ig_table>();
        s->header = t->header;
        const size_t nc = t->header.size();
        s->n_rows = end - begin;
        s->off.reserve(s->n_rows * nc);
        s->len.reserve(s->n_rows * nc);
        for (size_t r = begin; r < end; ++r)
            for (size_t j = 0; j < nc; ++j) {
                auto c = t->cell(r, j);
                s->off.push_back(s->arena.size());
                s->len.push_back((uint32_t)c.size());
                s->arena.append(c);
            }
        *out = s.release();
    });
}
void ig_table_free(ig_table* t) { delete t; }

int ig_infer_schema(const ig_table* t, const char* label, const char* attack, const char* normal, int decimals,
                    ig_schema** out) {
    *out = nullptr;
    return guard(nullptr, [&] {
        auto s = std::make_unique<ig_schema>();
        igb::infer_schema(*t, label ? label : "", igb::split_csv_list(attack), igb::split_csv_list(normal), decimals,
                          *s);
        *out = s.release();
    });
}
int ig_schema_column(const ig_schema* s, size_t j, int* kind, double* mean, double* sd) {
    if (!s || j >= s->names.size()) return IG_E_RANGE;
    *kind = s->kind[j];
    *mean = s->mean[j];
    *sd = s->sd[j];
    return IG_OK;
}
size_t ig_schema_label_index(const ig_schema* s) { return s ? s->label_index : 0; }
size_t ig_schema_cols(const ig_schema* s) { return s ? s->names.size() : 0; }
void ig_schema_free(ig_schema* s) { delete s; }

int ig_columns_build(const ig_table* t, const ig_schema* s, int with_labels, ig_columns** out) {
    *out = nullptr;
    return guard(nullptr, [&] {
        auto c = std::make_unique<ig_columns>();
        igb::build_columns(*t, *s, with_labels != 0, *c);
        igb::build_narrow(*c);
        // Page-lock the typed arrays once so every encode's H2D runs at full PCIe/C2C
        // speed; best effort (no GPU here -> plain pageable copies).
        auto pin = [&](void* p, size_t bytes) {
            if (bytes && cudaHostRegister(p, bytes, cudaHostRegisterDefault) == cudaSuccess)
                c->pinned.push_back(p);
            else
                cudaGetLastError();
        };
        pin(c->values.data(), c->values.size() * 8);
        pin(c->narrow.data(), c->narrow.size());
        pin(c->cat.data(), c->cat.size() * 4);
        pin(c->is_attack.data(), c->is_attack.size());
        *out = c.release();
    });
}
int ig_ingest_csv(ig_ctx* ctx, const char* bytes, size_t len, const char* label_column, const char* attack_values,
                  const char* normal_values, int decimals, long long train_rows, int ratio_k, ig_schema** schema,
                  ig_columns** train, ig_columns** test) {
    *schema = nullptr;
    *train = *test = nullptr;
    return guard(ctx, [&] {
        auto S = std::make_unique<ig_schema>();
        auto TR = std::make_unique<ig_columns>(), TE = std::make_unique<ig_columns>();
        const auto attack = igb::split_csv_list(attack_values), normal = igb::split_csv_list(normal_values);
        const std::string label = label_column ? label_column : "label";
        if (!igb::ingest_csv(*ctx, bytes, len, label, attack, normal, decimals, train_rows, ratio_k, *S, *TR, *TE)) {
            // the host reader (quoted fields, ...), then resident copies
            ig_table t;
            igb::read_csv(bytes, len, t);
            const size_t n = t.n_rows;
            const size_t ntr = train_rows >= 0 ? std::min<size_t>((size_t)train_rows, n) : (size_t)ratio_k * n / 10;
            auto slice = [&](size_t lo, size_t hi) {
                ig_table o;
                o.header = t.header;
                o.n_rows = hi - lo;
                for (size_t r = lo; r < hi; ++r)
                    for (size_t j = 0; j < t.header.size(); ++j) {
                        auto c = t.cell(r, j);
                        o.off.push_back(o.arena.size());
                        o.len.push_back((uint32_t)c.size());
                        o.arena.append(c);
                    }
                return o;
            };
            ig_table a = slice(0, ntr), b = slice(ntr, n);
            igb::infer_schema(a, label, attack, normal, decimals, *S);
            igb::build_columns(a, *S, true, *TR);
            igb::build_columns(b, *S, false, *TE);
            igb::upload_columns(*ctx, *TR);
            igb::upload_columns(*ctx, *TE);
        }
        *schema = S.release();
        *train = TR.release();
        *test = TE.release();
    });
}

int ig_columns_upload(ig_ctx* ctx, ig_columns* c) {
    return guard(ctx, [&] { igb::upload_columns(*ctx, *c); });
}
int ig_columns_prefetch(ig_ctx* ctx, ig_columns* c) {
    if (!ctx || !c) return IG_E_INVALID_ARG;
    return guard(ctx, [&] { igb::prefetch_columns(*ctx, *c); });
}
size_t ig_columns_rows(const ig_columns* c) { return c ? c->n_rows : 0; }
size_t ig_columns_bytes(const ig_columns* c) {
    if (!c) return 0;
    const size_t num = c->narrow.empty() ? c->values.size() * 8 : c->narrow.size();
    return num + c->cat.size() * 4 + c->is_attack.size();
}
void ig_columns_free(ig_columns* c) {
    if (!c) return;
    igb::drop_prefetch(*c);
    for (void* p : c->pinned) cudaHostUnregister(p);
    delete c;
}

int ig_encode_training(ig_ctx* ctx, const ig_columns* cols, ig_encoding** out) {
    *out = nullptr;
    return guard(ctx, [&] {
        auto e = std::make_unique<ig_encoding>();
        igb::encode_training_dev(*ctx, *cols, *e);
        e->attack.buf.persist();
        e->normal.buf.persist();
        *out = e.release();
    });
}

int ig_encode_rows(ig_ctx* ctx, const ig_columns* cols, const ig_encoding* train, ig_encoding** out) {
    *out = nullptr;
    return guard(ctx, [&] {
        auto e = std::make_unique<ig_encoding>();
        auto job = std::make_shared<RowIndexJob>();
        IGB_CUDA(cudaEventCreateWithFlags(&job->rows_ready, cudaEventDisableTiming));
        IGB_CUDA(cudaEventCreateWithFlags(&job->done, cudaEventDisableTiming));
        // the index stream runs after everything already queued on the context stream
        IGB_CUDA(cudaEventRecord(job->rows_ready, ctx->stream));
        IGB_CUDA(cudaStreamWaitEvent(ctx->index, job->rows_ready, 0));
        igb::Ctx cx = *ctx;
        cx.stream = ctx->index;
        cx.launches = 0;
        igb::encode_rows_dev(cx, *cols, *train, *e, /*queue_only=*/true);
        ctx->launches += cx.launches;
        e->all.buf.persist();
        IGB_CUDA(cudaEventRecord(job->rows_ready, ctx->index));
        const size_t n = e->all.n, k = e->all.k;
        const uint32_t L = e->L;
        if (n && igb::postings_supported(L, n)) {
            job->has_postings = true;
            cx.launches = 0;
            const int64_t* rows = e->all.data();
            RowIndexJob* j = job.get();
            job->task.start(ctx->index_worker, [j, cx, rows, n, k, L]() mutable {
                try {
                    IGB_CUDA(cudaSetDevice(cx.device));
                    igb::build_postings(cx, rows, n, k, L, j->P, true, true);
                    for (DevBuf* b : {&j->P.dense, &j->P.df, &j->P.nz_off, &j->P.nz_idx, &j->P.perm, &j->P.group,
                                      &j->P.rep})
                        b->persist();  // read by evidence on other streams
                    IGB_CUDA(cudaEventRecord(j->done, cx.stream));
                } catch (...) {
                    j->err = std::current_exception();
                }
                j->launches = cx.launches;
            });
        } else {
            IGB_CUDA(cudaEventRecord(job->done, ctx->index));
        }
        e->job = std::move(job);
        *out = e.release();
    });
}

namespace {
// rows of a background test encoding are usable once packed
void rows_ready(ig_ctx* ctx, const ig_encoding* e) {
    if (e && e->job) IGB_CUDA(cudaStreamWaitEvent(ctx->stream, e->job->rows_ready, 0));
}
}  // namespace

uint32_t ig_encoding_logical_len(const ig_encoding* e) { return e ? e->L : 0; }
static const DevRows* enc_rows(const ig_encoding* e, int which) {
    return which == 0 ? &e->attack : which == 1 ? &e->normal : &e->all;
}
size_t ig_encoding_rows(const ig_encoding* e, int which) { return e ? enc_rows(e, which)->n : 0; }
const int64_t* ig_encoding_device_rows(const ig_encoding* e, int which) {
    if (e && e->job) cudaEventSynchronize(e->job->rows_ready);  // raw pointer: the caller's stream is unknown
    return e ? enc_rows(e, which)->data() : nullptr;
}
int ig_encoding_copy_rows(ig_ctx* ctx, const ig_encoding* e, int which, int64_t* out) {
    return guard(ctx, [&] {
        rows_ready(ctx, e);
        const DevRows* r = enc_rows(e, which);
        if (r->n * r->k)
            IGB_CUDA(cudaMemcpyAsync(out, r->data(), r->n * r->k * 8, cudaMemcpyDeviceToHost, ctx->stream));
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}
const char* ig_encoding_vocabulary(const ig_encoding* e) {
    if (!e) return "";
    try {
        return e->host_vocab().vocab_blob.c_str();
    } catch (const igb::Error& err) {
        igb::set_last_error(err.msg);
        return "";
    }
}
size_t ig_encoding_removed_count(const ig_encoding* e) { return e ? e->removed.size() : 0; }
int ig_encoding_removed_rows(const ig_encoding* e, uint64_t* rows) {
    if (!e) return IG_E_INVALID_ARG;
    std::copy(e->removed.begin(), e->removed.end(), rows);
    return IG_OK;
}
void ig_encoding_free(ig_encoding* e) { delete e; }

int ig_fit_encoded(ig_ctx* ctx, const ig_encoding* train, const ig_kernel_config* cfg, ig_model** out) {
    *out = nullptr;
    return guard(ctx, [&] {
        check_cfg(cfg);
        View X[2] = {{train->attack.data(), train->attack.n, train->attack.k},
                     {train->normal.data(), train->normal.n, train->normal.k}};
        auto m = std::make_unique<ig_model>();
        fit_impl(*ctx, X, train->L, *m, true, nullptr, nullptr, nullptr, (uint32_t)train->n_cols);
        *out = m.release();
    });
}

namespace {
void evidence_of_encoding(ig_ctx* ctx, const ig_model* m, const ig_encoding* tests, int64_t* d_A, int64_t* d_N) {
    const size_t nt = tests->all.n;
    const igb::Postings* pre = nullptr;
    if (tests->job) {
        tests->job->wait(ctx);
        IGB_CUDA(cudaStreamWaitEvent(ctx->stream, tests->job->done, 0));
        if (tests->job->has_postings) pre = &tests->job->P;
    }
    evidence_impl(*ctx, *m, tests->all.data(), nt, tests->L, d_A, d_N, pre);
}
}  // namespace

int ig_evidence_encoded(ig_ctx* ctx, const ig_model* m, const ig_encoding* tests, int64_t* A, int64_t* N) {
    return guard(ctx, [&] {
        const size_t nt = tests->all.n;
        if (nt == 0) return;
        DevBuf a(nt * 8, ctx->stream), b(nt * 8, ctx->stream);
        evidence_of_encoding(ctx, m, tests, a.as<int64_t>(), b.as<int64_t>());
        igb::copy_to_host(*ctx, A, a.p, nt * 8);
        igb::copy_to_host(*ctx, N, b.p, nt * 8);
    });
}

int ig_fit_evidence_encoded(ig_ctx* ctx, const ig_encoding* train, const ig_encoding* tests, const ig_kernel_config* cfg,
                            ig_model** out, int64_t* d_A, int64_t* d_N) {
    *out = nullptr;
    return guard(ctx, [&] {
        check_cfg(cfg);
        if (tests->L != train->L) fail(IG_E_INVALID_ARG, "fused_score: logical length mismatch");
        View X[2] = {{train->attack.data(), train->attack.n, train->attack.k},
                     {train->normal.data(), train->normal.n, train->normal.k}};
        auto m = std::make_unique<ig_model>();
        FusedEvidence ev;
        ev.job = tests->job.get();
        ev.out[0] = d_A;
        ev.out[1] = d_N;
        if (tests->all.n == 0) ev.job = nullptr;
        fit_impl(*ctx, X, train->L, *m, true, &ev, nullptr, nullptr, (uint32_t)train->n_cols);
        if (!ev.done && tests->all.n) evidence_of_encoding(ctx, m.get(), tests, d_A, d_N);
        *out = m.release();
    });
}

int ig_fit_evidence_encoded_host(ig_ctx* ctx, const ig_encoding* train, const ig_encoding* tests,
                                 const ig_kernel_config* cfg, ig_model** out, int64_t* A, int64_t* N) {
    *out = nullptr;
    const size_t nt = tests ? tests->all.n : 0;
    igb::DevBuf a, b;
    int st = guard(ctx, [&] {
        a.alloc(std::max<size_t>(nt, 1) * 8, ctx->stream);
        b.alloc(std::max<size_t>(nt, 1) * 8, ctx->stream);
    });
    if (st) return st;
    st = ig_fit_evidence_encoded(ctx, train, tests, cfg, out, a.as<int64_t>(), b.as<int64_t>());
    if (st) return st;
    return guard(ctx, [&] {
        // through the page-locked bounce buffer: a pageable D2H is staged by
        // the driver at a fraction of the link rate
        igb::copy_to_host(*ctx, A, a.p, nt * 8);
        igb::copy_to_host(*ctx, N, b.p, nt * 8);
    });
}

int ig_evidence_encoded_device(ig_ctx* ctx, const ig_model* m, const ig_encoding* tests, int64_t* d_A, int64_t* d_N) {
    return guard(ctx, [&] {
        if (tests->all.n == 0) return;
        evidence_of_encoding(ctx, m, tests, d_A, d_N);
    });
}


// ------------------------------------------------------------------ multi-GPU shards
// rows replicated, pair tiles split round-robin, candidates
// routed to the owner of their content fingerprint, owner-local support /
// coverage / scores, matcher partials summed by the caller.
struct ig_shard {
    int rank = 0, world = 1;
    uint32_t L = 0;
    size_t k = 0;
    const ig_encoding* train = nullptr;
    igb::DevBuf U[2];
    igb::DevBuf perm[2];  // canonical order of each class's rows (reused by the finish)
    size_t m[2] = {0, 0};
    igb::DevBuf send[2];
    std::vector<uint64_t> counts[2];
    bool received[2] = {false, false};
    ig_model model;
    // each class's training postings (replicated work: every rank scans its own
    // candidates against all training rows), built on the context's aux stream
    // by its worker while the class's records travel; finish() takes them
    igb::Postings PX[2];
    std::unique_ptr<igb::Ctx> px_ctx[2];
    std::future<void> px_done[2];
    std::exception_ptr px_err[2];
    void wait_postings(igb::Ctx& ctx) {
        for (int c = 0; c < 2; ++c) {
            if (!px_done[c].valid()) continue;
            px_done[c].wait();
            px_done[c] = {};
            ctx.launches += px_ctx[c]->launches;
            ctx.diag_merge(*px_ctx[c]);
            px_ctx[c].reset();
        }
        for (auto& e : px_err)
            if (e) std::rethrow_exception(std::exchange(e, nullptr));
    }
    ~ig_shard() {
        for (auto& f : px_done)
            if (f.valid()) f.wait();
    }
};

int ig_shard_create(ig_ctx* ctx, const ig_encoding* train, int rank, int world, const ig_kernel_config* cfg,
                    ig_shard** out) {
    *out = nullptr;
    return guard(ctx, [&] {
        check_cfg(cfg);
        if (world < 1 || rank < 0 || rank >= world) fail(IG_E_INVALID_ARG, "shard: rank must be in [0, world)");
        auto s = std::make_unique<ig_shard>();
        s->rank = rank;
        s->world = world;
        s->train = train;
        s->L = train->L;
        s->k = igb::words_for(train->L);
        const igb::DevRows* X[2] = {&train->attack, &train->normal};
        for (int c = 0; c < 2; ++c) {
            if (X[c]->n == 0) fail(IG_E_DATA, "enumerate_candidates: empty class");
            s->m[c] = igb::distinct_rows(*ctx, X[c]->data(), X[c]->n, s->k, s->U[c], nullptr, &s->perm[c]);
            s->U[c].persist();
            s->perm[c].persist();
        }
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = s.release();
    });
}

int ig_shard_enumerate(ig_ctx* ctx, ig_shard* s, int cls, uint64_t* counts, const void** d_send) {
    return guard(ctx, [&] {
        if (cls < 0 || cls > 1) fail(IG_E_INVALID_ARG, "class must be 0 (attack) or 1 (normal)");
        igb::PairSource src;
        src.tile_begin = (uint64_t)s->rank;
        src.tile_step = (uint64_t)s->world;
        igb::DevBuf reps;
        igb::Trace tr(*ctx, "shard_enumerate", cls);
        // one rank: its deduplicated records are the whole class's, all owned here
        const bool solo = s->world == 1;
        const uint64_t c = igb::dedup_pairs(*ctx, s->U[cls].as<int64_t>(), s->m[cls], s->k, src, reps,
                                            solo ? &s->model.stats[cls] : nullptr);
        tr.mark("dedup");
        if (solo) {
            s->send[cls] = std::move(reps);
            s->counts[cls].assign(1, c);
        } else {
            igb::bucket_by_owner(*ctx, s->U[cls].as<int64_t>(), s->k, reps.as<uint2>(), c, s->world, s->send[cls],
                                 s->counts[cls]);
        }
        tr.mark("bucket");
        s->send[cls].persist();
        for (int r = 0; r < s->world; ++r) counts[r] = s->counts[cls][r];
        *d_send = s->send[cls].p;
        // this class's training postings, off the caller's thread and stream
        const igb::DevRows& X = cls == 0 ? s->train->attack : s->train->normal;
        const size_t nmax = std::max(s->train->attack.n, s->train->normal.n);
        if (ctx->worker && !s->px_done[cls].valid() && !s->PX[cls].L && igb::postings_supported(s->L, nmax)) {
            s->px_ctx[cls] = std::make_unique<igb::Ctx>(*ctx);
            igb::Ctx* cx = s->px_ctx[cls].get();
            cx->stream = ctx->aux;
            cx->launches = 0;
            cx->progress = nullptr;
            for (auto& d : cx->diag_k) d = igb::DiagStat{};
            ig_shard* sh = s;
            s->px_done[cls] = ctx->worker->submit([sh, cx, cls, &X] {
                try {
                    IGB_CUDA(cudaSetDevice(cx->device));
                    igb::build_postings(*cx, X.data(), X.n, sh->k, sh->L, sh->PX[cls], true, false,
                                        sh->perm[cls].as<uint32_t>());
                } catch (...) {
                    sh->px_err[cls] = std::current_exception();
                }
            });
        }
    });
}

int ig_shard_receive(ig_ctx* ctx, ig_shard* s, int cls, const void* d_recv, uint64_t n_records) {
    return guard(ctx, [&] {
        if (cls < 0 || cls > 1) fail(IG_E_INVALID_ARG, "class must be 0 (attack) or 1 (normal)");
        igb::PairSource src;
        src.list = static_cast<const uint2*>(d_recv);
        src.n_list = n_records;
        igb::DevBuf reps;
        ig_candidates& C = s->model.cand[cls];
        if (s->world == 1) {
            // a single sender's records are already distinct (its own dedup)
            igb::materialize_pairs(*ctx, s->U[cls].as<int64_t>(), s->k, src.list, n_records, s->L, C.rows);
        } else {
            const uint64_t c = igb::dedup_pairs(*ctx, s->U[cls].as<int64_t>(), s->m[cls], s->k, src, reps,
                                                &s->model.stats[cls]);
            igb::materialize_pairs(*ctx, s->U[cls].as<int64_t>(), s->k, reps.as<uint2>(), c, s->L, C.rows);
        }
        C.ordered = false;
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
        s->received[cls] = true;
    });
}

int ig_shard_finish(ig_ctx* ctx, ig_shard* s, uint64_t* partial_totals) {
    return guard(ctx, [&] {
        if (!s->received[0] || !s->received[1]) fail(IG_E_INVALID_ARG, "shard: receive both classes first");
        View X[2] = {{s->train->attack.data(), s->train->attack.n, s->train->attack.k},
                     {s->train->normal.data(), s->train->normal.n, s->train->normal.k}};
        const uint32_t* rp[2] = {s->perm[0].p ? s->perm[0].as<uint32_t>() : nullptr,
                                 s->perm[1].p ? s->perm[1].as<uint32_t>() : nullptr};
        s->wait_postings(*ctx);
        cudaEvent_t built;
        IGB_CUDA(cudaEventCreateWithFlags(&built, cudaEventDisableTiming));
        IGB_CUDA(cudaEventRecord(built, ctx->aux));
        IGB_CUDA(cudaStreamWaitEvent(ctx->stream, built, 0));
        cudaEventDestroy(built);
        fit_impl(*ctx, X, s->L, s->model, /*enumerate=*/false, nullptr, rp, s->PX, (uint32_t)s->train->n_cols);
        partial_totals[0] = s->model.partial_total[0];
        partial_totals[1] = s->model.partial_total[1];
    });
}

const ig_model* ig_shard_model(const ig_shard* s) { return s ? &s->model : nullptr; }

void ig_shard_free(ig_shard* s) { delete s; }


// ------------------------------------------------------------------ archive / explain
int ig_schema_to_text(const ig_schema* s, char* buf, size_t cap, size_t* len) {
    return guard(nullptr, [&] {
        const std::string t = igb::schema_to_text(*s);
        *len = t.size();
        if (buf && cap) {
            const size_t n = std::min(cap - 1, t.size());
            std::memcpy(buf, t.data(), n);
            buf[n] = '\0';
        }
    });
}

int ig_schema_from_text(const char* text, ig_schema** out) {
    *out = nullptr;
    return guard(nullptr, [&] {
        auto s = std::make_unique<ig_schema>();
        igb::schema_from_text(text, *s);
        *out = s.release();
    });
}

int ig_encoding_from_vocabulary(const ig_schema* s, const char* vocab_blob, ig_encoding** out) {
    *out = nullptr;
    return guard(nullptr, [&] {
        std::vector<std::string> toks;
        std::string cur;
        for (const char* p = vocab_blob; *p; ++p) {
            if (*p == '\n') {
                toks.push_back(cur);
                cur.clear();
            } else {
                cur += *p;
            }
        }
        if (!cur.empty()) toks.push_back(cur);
        auto e = std::make_unique<ig_encoding>();
        igb::encoding_from_vocab(*s, toks, *e);
        *out = e.release();
    });
}

int ig_model_from_dictionaries(ig_ctx* ctx, uint32_t L, const int64_t* wa, const int64_t* sa, const int64_t* ca,
                               size_t na, const int64_t* wn, const int64_t* sn, const int64_t* cn, size_t nn,
                               ig_model** out) {
    *out = nullptr;
    return guard(ctx, [&] {
        auto m = std::make_unique<ig_model>();
        m->L = L;
        const int64_t* W[2] = {wa, wn};
        const int64_t* S[2] = {sa, sn};
        const int64_t* C[2] = {ca, cn};
        const size_t Nn[2] = {na, nn};
        const size_t k = igb::words_for(L);
        for (int c = 0; c < 2; ++c) {
            ig_candidates& P = m->pure[c];
            upload_rows(*ctx, W[c], Nn[c], L, P.rows);
            P.support.alloc(std::max<size_t>(Nn[c], 1) * 8, ctx->stream);
            P.score.alloc(std::max<size_t>(Nn[c], 1) * 8, ctx->stream);
            if (Nn[c]) {
                IGB_CUDA(cudaMemcpyAsync(P.support.p, S[c], Nn[c] * 8, cudaMemcpyHostToDevice, ctx->stream));
                IGB_CUDA(cudaMemcpyAsync(P.score.p, C[c], Nn[c] * 8, cudaMemcpyHostToDevice, ctx->stream));
            }
            P.has_support = P.has_score = true;
            P.rows.buf.persist();
            P.support.persist();
            P.score.persist();
            bool neg = false;
            __int128 tot = 0;
            for (size_t i = 0; i < Nn[c]; ++i) {
                neg |= C[c][i] < 0;
                tot += C[c][i];
            }
            if (neg || tot > (__int128)INT64_MAX) m->sum_fits = false;  // evidence then uses checked sums
            m->cand[c].rows.k = k;
            m->cand[c].rows.L = L;
        }
        IGB_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = m.release();
    });
}

int ig_explain(ig_ctx* ctx, const ig_model* m, int cls, const int64_t* row, uint32_t L, uint32_t* idx, size_t cap,
               size_t* n_found) {
    return guard(ctx, [&] {
        if (cls < 0 || cls > 1) fail(IG_E_INVALID_ARG, "class must be 0 (attack) or 1 (normal)");
        if (L != m->L) fail(IG_E_INVALID_ARG, "explain: logical length mismatch");
        const ig_candidates& P = m->pure[cls];
        *n_found = igb::explain_dev(*ctx, P.rows.data(), P.rows.n, P.rows.k, row, idx, cap);
    });
}

}  // extern "C"
