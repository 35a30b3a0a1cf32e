// integration/ig_b200_backend.cpp — see ig_b200_backend.hpp.
#include "ig_b200_backend.hpp"

#include <stdexcept>
#include <string>
#include <unordered_map>

#include "ig/errors.hpp"
#include "ig_b200.h"

namespace ig {
namespace {

// ig_status -> the reference exception types (errors.hpp:9-32, kernels.cpp).
[[noreturn]] void raise(int st, const ig_ctx* ctx) {
    std::string msg = ig_last_error(ctx);
    switch (st) {
        case IG_E_INVALID_ARG: throw std::invalid_argument(msg);
        case IG_E_RANGE: throw std::out_of_range(msg);
        case IG_E_CONFIG: throw ConfigError(msg);
        case IG_E_IO: throw IoError(msg);
        case IG_E_DATA: throw DataError(msg);
        case IG_E_OVERFLOW: throw ArithmeticError(msg);
        default: throw std::runtime_error("ig_b200: " + msg);
    }
}
void check(int st, const ig_ctx* ctx) {
    if (st != IG_OK) raise(st, ctx);
}

struct Ctx {
    ig_ctx* p = nullptr;
    explicit Ctx(int device) { check(ig_ctx_create(device, &p), nullptr); }
    Ctx(const Ctx&) = delete;
    ~Ctx() { ig_ctx_destroy(p); }
};

// One context per calling thread and device: the backend's const methods are
// called concurrently (kernels.hpp:23-26; the OpenMP enumerate of
// oracle/ref_shim.cpp calls pair_intersect_batch from every worker), and each
// thread's calls then run on its own streams without waiting for the others.
ig_ctx* thread_ctx(int device) {
    thread_local std::unordered_map<int, std::unique_ptr<Ctx>> ctxs;
    auto& c = ctxs[device];
    if (!c) c = std::make_unique<Ctx>(device);
    return c->p;
}

ig_kernel_config to_c(const KernelConfig& k) {
    return ig_kernel_config{k.pair_batch, k.coverage_block, k.memory_budget_bytes, k.threads};
}

class B200Backend final : public KernelBackend {
public:
    explicit B200Backend(int device) : device_(device) {}
    std::string_view name() const override { return "b200"; }

    void pair_intersect_batch(const PackedMatrix& rows, std::size_t left, std::size_t j_begin, std::size_t j_end,
                              std::int64_t* out) const override {
        ig_ctx* c = thread_ctx(device_);
        check(ig_pair_intersect_batch(c, rows.data(), rows.rows(), rows.logical_len(), left, j_begin, j_end, out), c);
    }

    std::vector<std::uint8_t> coverage_any(const PackedMatrix& patterns, const PackedMatrix& opponents,
                                           std::size_t coverage_block) const override {
        std::vector<std::uint8_t> mask(patterns.rows(), 0);
        ig_ctx* c = thread_ctx(device_);
        check(ig_coverage_any(c, patterns.data(), patterns.rows(), patterns.logical_len(), opponents.data(),
                              opponents.rows(), opponents.logical_len(), coverage_block, mask.data()),
              c);
        return mask;
    }

    std::vector<std::int64_t> fused_score(const PackedMatrix& patterns, std::span<const std::int64_t> scores,
                                          const PackedMatrix& tests) const override {
        std::vector<std::int64_t> out(tests.rows(), 0);
        ig_ctx* c = thread_ctx(device_);
        check(ig_fused_score(c, patterns.data(), patterns.rows(), patterns.logical_len(), scores.data(),
                             scores.size(), tests.data(), tests.rows(), tests.logical_len(), out.data()),
              c);
        return out;
    }

private:
    int device_;
};

}  // namespace

std::unique_ptr<KernelBackend> make_b200_backend(int device) { return std::make_unique<B200Backend>(device); }

CandidateSet b200_enumerate_candidates(const PackedMatrix& rows, const KernelConfig& config,
                                       const ProgressFn& progress) {
    config.validate();
    ig_ctx* c = thread_ctx(0);
    ig_kernel_config k = to_c(config);
    ig_candidates* h = nullptr;
    // ProgressFn (mine.hpp:31-33) is called from this thread while the device enumerates
    auto trampoline = [](std::uint64_t done, std::uint64_t total, std::uint64_t found, void* user) {
        (*static_cast<const ProgressFn*>(user))(done, total, found);
    };
    check(ig_enumerate_candidates(c, rows.data(), rows.rows(), rows.logical_len(), &k,
                                  progress ? +trampoline : nullptr, const_cast<ProgressFn*>(&progress), &h),
          c);
    const std::size_t n = ig_candidates_count(h);
    std::vector<std::int64_t> words(n * rows.word_count());
    const int st = ig_candidates_copy(c, h, words.data(), nullptr, nullptr);
    ig_candidates_free(h);
    check(st, c);
    CandidateSet out;
    out.class_tag = rows.class_tag();
    out.source_rows = rows.rows();
    out.patterns = PackedMatrix(rows.logical_len(), rows.class_tag());
    out.patterns.reserve_rows(n);
    for (std::size_t i = 0; i < n; ++i) out.patterns.append_words(words.data() + i * rows.word_count());
    return out;
}

void b200_count_support(CandidateSet& candidates, const PackedMatrix& rows, const KernelConfig& config) {
    config.validate();
    ig_ctx* c = thread_ctx(0);
    candidates.supports.assign(candidates.patterns.rows(), 0);
    check(ig_count_support_rows(c, candidates.patterns.data(), candidates.patterns.rows(),
                                candidates.patterns.logical_len(), rows.data(), rows.rows(), rows.logical_len(),
                                candidates.supports.data()),
          c);
}

}  // namespace ig
