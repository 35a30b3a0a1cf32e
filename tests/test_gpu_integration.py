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
