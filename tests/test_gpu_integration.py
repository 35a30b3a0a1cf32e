"""The drop-in proof: the reference's own code path (oracle/_ref: proj/src/*.cpp
+ the restated mine/purify/infer) running on the "b200" KernelBackend that
integration/ig_b200_backend.cpp registers over the C-ABI — results identical to
the same code on the reference's ParallelCpuBackend (kernels.hpp:23-26)."""
import numpy as np
import pytest

from oracle import ref
from paper_2507_14222_b200 import synth

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(b200=True), reason="oracle/_ref/libigref_b200.so not built")]


def test_reference_pipeline_on_b200_backend():
    csv = synth.nsl_csv(900, seed=31)
    a = ref.run(csv, decimals=1, ratio_k=8, backend="parallel-cpu", pair_batch=64)
    b = ref.run(csv, decimals=1, ratio_k=8, backend="b200", pair_batch=64)
    assert a.L == b.L
    for c in range(2):
        for x, y in zip(a.cand[c], b.cand[c]):
            assert np.array_equal(x, y)
        for x, y in zip(a.pure[c], b.pure[c]):
            assert np.array_equal(x, y)
    assert np.array_equal(a.A, b.A) and np.array_equal(a.N, b.N)
    assert np.array_equal(a.labels, b.labels)


def test_backend_primitives_through_reference_types():
    rng = np.random.default_rng(4)
    L = 200
    k = (L + 63) // 64
    rows = rng.integers(-2**63, 2**63 - 1, (300, k), dtype=np.int64)
    rows[:, -1] &= (1 << (L - 64 * (k - 1))) - 1
    w1 = ref.pair_intersect_batch(rows, L, 5, 6, 300, backend="reference")
    w2 = ref.pair_intersect_batch(rows, L, 5, 6, 300, backend="b200")
    assert np.array_equal(w1, w2)
    pats = rows[:100] & rows[100:200]
    assert np.array_equal(ref.coverage_any(pats, L, rows, L, backend="reference"),
                          ref.coverage_any(pats, L, rows, L, backend="b200"))
    s = rng.integers(0, 1000, 100)
    assert np.array_equal(ref.fused_score(pats, L, s, rows, L, backend="reference"),
                          ref.fused_score(pats, L, s, rows, L, backend="b200"))
    with pytest.raises(ref.RefError) as e:
        ref.pair_intersect_batch(rows, L, 5, 5, 300, backend="b200")
    assert e.value.status == 1  # std::invalid_argument, as the reference


def _b200_lib():
    import ctypes as C
    L = ref.lib(b200=True)
    p64 = C.POINTER(C.c_int64)
    L.igref_b200_concurrency.argtypes = [p64, C.c_size_t, C.c_uint32, p64, C.c_size_t, p64, C.c_int, C.c_int,
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    L.igref_b200_enumerate_progress.argtypes = [p64, C.c_size_t, C.c_uint32, C.POINTER(C.c_uint64),
                                                C.POINTER(C.c_int), C.POINTER(C.c_uint64), C.POINTER(C.c_void_p)]
    return L


def test_backend_concurrent_calls_match_parallel_cpu():
    """kernels.hpp:23-26: eight host threads share ONE "b200" backend and call
    pair_intersect_batch / coverage_any / fused_score concurrently on shared
    inputs (as the OpenMP enumerate of the reference does); every result equals
    ParallelCpuBackend's."""
    import ctypes as C
    rng = np.random.default_rng(23)
    L = 150
    k = (L + 63) // 64
    rows = (rng.random((400, L)) < 0.7)
    X = np.zeros((400, k), np.uint64)
    for j in range(L):
        X[:, j // 64] |= rows[:, j].astype(np.uint64) << np.uint64(j % 64)
    X = X.view(np.int64)
    pats = X[rng.integers(0, 400, 300)] & X[rng.integers(0, 400, 300)]
    scores = rng.integers(0, 1 << 20, 300).astype(np.int64)
    bad, calls = C.c_uint64(), C.c_uint64()
    p64 = C.POINTER(C.c_int64)
    lib = _b200_lib()
    st = lib.igref_b200_concurrency(X.ctypes.data_as(p64), 400, L, pats.ctypes.data_as(p64), 300,
                                    scores.ctypes.data_as(p64), 8, 12, C.byref(bad), C.byref(calls))
    assert st == 0, lib.igref_last_error().decode()
    assert calls.value == 8 * 12 * 3 and bad.value == 0


def test_enumerate_progress_reported_while_running(golden_dir):
    """mine.hpp:31-33: ProgressFn is called from the calling thread while the
    device enumerates (pairs done and candidates found never decrease), and the
    last call reports the total and the final candidate count.  The normal
    class of C4 (61k rows, ~30 ms on the device) so that polls land mid-run."""
    import ctypes as C
    import json
    import os
    csv = synth.nsl_csv(148517, seed=2507)
    r = ref.run(csv, decimals=1, ratio_k=8, stages=0)
    X = np.ascontiguousarray(r.normal)
    n_calls, mono, last, h = C.c_uint64(), C.c_int(), (C.c_uint64 * 3)(), C.c_void_p()
    lib = _b200_lib()
    p64 = C.POINTER(C.c_int64)
    st = lib.igref_b200_enumerate_progress(X.ctypes.data_as(p64), X.shape[0], r.L, C.byref(n_calls), C.byref(mono),
                                           last, C.byref(h))
    assert st == 0, lib.igref_last_error().decode()
    try:
        n = lib.igref_cand_count(h)
        assert mono.value == 1 and n_calls.value >= 2
        assert last[0] == last[1] and last[2] == n
        g = os.path.join(golden_dir, "nsl_c4.json")
        if os.path.exists(g):
            assert n == json.load(open(g))["cand_counts"][1]  # the reference's |B^-| at C4
    finally:
        lib.igref_cand_free(h)
