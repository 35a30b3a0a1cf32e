// integration/ig_b200_backend.hpp — the reference-side binding a maintainer adds
// to proj/ to use the B200 library: an ig::KernelBackend ("b200") and the
// mine.hpp free functions, implemented on the C-ABI in include/ig_b200.h.
//
// Compiled against the reference headers (proj/include/ig/*.hpp).  See
// INTEGRATION.md for the two-line registration in make_backend
// (proj/src/kernels.cpp:188-194).
#pragma once

#include <memory>

#include "ig/kernels.hpp"
#include "ig/mine.hpp"

namespace ig {

// KernelBackend over libig_b200.so (kernels.hpp:27-53).  Results are
// bit-identical to ReferenceBackend / ParallelCpuBackend (kernels.hpp:23-26).
std::unique_ptr<KernelBackend> make_b200_backend(int device = 0);

// mine.hpp:35-51 on the device: the whole candidate enumeration runs in one
// ABI call (the per-left-row window of pair_intersect_batch is not used).
CandidateSet b200_enumerate_candidates(const PackedMatrix& rows, const KernelConfig& config,
                                       const ProgressFn& progress = {});
void b200_count_support(CandidateSet& candidates, const PackedMatrix& rows, const KernelConfig& config);

}  // namespace ig
