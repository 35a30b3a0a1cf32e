"""GPU parity of the KernelBackend primitives (kernels.hpp:27-53) against the
plain-C oracle, through the C-ABI.  Bit-exact; edge cases from SPEC.md:225-258."""
import numpy as np
import pytest

from oracle import oracle, pipeline
from tests.helpers import random_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2507_14222_b200 import api as a
    return a


def M(api, w, L):
    return api.PackedMatrix(w, L)


@pytest.mark.parametrize("L", [1, 5, 63, 64, 65, 130, 700, 2000, 4200])
def test_coverage_and_fused_random(api, L):
    rng = np.random.default_rng(L)
    be = api.make_backend("b200")
    for dens in (0.3, 0.8, 0.97):
        P = random_rows(rng, 700, L, dens * 0.6)
        X = random_rows(rng, 900, L, dens)
        s = rng.integers(0, 1000, P.shape[0])
        mask = be.coverage_any(M(api, P, L), M(api, X, L), 4096)
        assert np.array_equal(mask, oracle.coverage_any(P, X)), (L, dens)
        out = be.fused_score(M(api, P, L), s, M(api, X, L))
        assert np.array_equal(out, oracle.fused_score(P, s, X)), (L, dens)


def test_coverage_block_invariance(api):
    rng = np.random.default_rng(1)
    L = 300
    P = random_rows(rng, 3000, L, 0.4)
    X = random_rows(rng, 500, L, 0.85)
    be = api.make_backend("b200")
    ref_mask = oracle.coverage_any(P, X)
    for block in (1, 7, 4096, 10**9):
        assert np.array_equal(be.coverage_any(M(api, P, L), M(api, X, L), block), ref_mask)


def test_kernel_spec_examples(api):
    # SPEC.md:231, 241-243, 251-253 (a..e = bits 0..4)
    a, b, c, d, e = range(5)
    L = 5
    pk = lambda s: pipeline.pack(s, L)  # noqa: E731
    be = api.make_backend("b200")
    rows = M(api, np.stack([pk([a, b, c]), pk([a, b, d]), pk([a, c, d])]), L)
    win = be.pair_intersect_batch(rows, 0, 1, 3)
    assert win.tolist() == [pk([a, b]).tolist(), pk([a, c]).tolist()]
    assert be.pair_intersect_batch(rows, 2, 3, 3).shape == (0, 1)  # i = n-1: empty window
    pats = M(api, np.stack([pk([a, b]), pk([a, c])]), L)
    assert be.coverage_any(pats, M(api, np.stack([pk([a, b, e])]), L)).tolist() == [1, 0]
    assert be.coverage_any(pats, M(api, np.zeros((0, 1), np.int64), L)).tolist() == [0, 0]
    assert be.coverage_any(M(api, np.stack([pk([])]), L), M(api, np.stack([pk([c])]), L)).tolist() == [1]
    P = M(api, np.stack([pk([a, c]), pk([a, d]), pk([a, c, d])]), L)
    assert be.fused_score(P, [8, 8, 9], M(api, np.stack([pk([a, c, d, e])]), L)).tolist() == [25]
    assert be.fused_score(P, [8, 8, 9], M(api, np.stack([pk([b])]), L)).tolist() == [0]
    assert be.fused_score(M(api, np.stack([pk([])]), L), [7], M(api, np.stack([pk([b]), pk([])]), L)).tolist() == [7, 7]


def test_pair_window_contract(api):
    rng = np.random.default_rng(2)
    L = 200
    X = random_rows(rng, 50, L, 0.5)
    be = api.make_backend("b200")
    out = be.pair_intersect_batch(M(api, X, L), 3, 4, 50)
    assert np.array_equal(out, X[3] & X[4:50])
    for bad in ((50, 51, 51), (3, 3, 10), (3, 2, 10), (3, 10, 9), (3, 10, 51)):
        with pytest.raises(ValueError):
            be.pair_intersect_batch(M(api, X, L), *bad)


def test_shape_errors(api):
    be = api.make_backend("b200")
    with pytest.raises(ValueError):
        be.coverage_any(M(api, np.zeros((1, 1), np.int64), 5), M(api, np.zeros((1, 2), np.int64), 70))
    with pytest.raises(ValueError):
        be.fused_score(M(api, np.zeros((2, 1), np.int64), 5), [1], M(api, np.zeros((1, 1), np.int64), 5))
    with pytest.raises(ValueError):
        be.coverage_any(M(api, np.zeros((1, 1), np.int64), 5), M(api, np.zeros((1, 1), np.int64), 5), 0)


def test_fused_overflow_semantics(api):
    L = 3
    pk = lambda s: pipeline.pack(s, L)  # noqa: E731
    be = api.make_backend("b200")
    P = M(api, np.stack([pk([0]), pk([1]), pk([2])]), L)
    T = M(api, np.stack([pk([0, 1, 2]), pk([0])]), L)
    big = 2**62
    with pytest.raises(api.IGArithmeticError):
        be.fused_score(P, [big, big, big], T)
    with pytest.raises(api.IGArithmeticError):           # prefix overflow, total fits
        be.fused_score(P, [big, big, -big], T)
    assert be.fused_score(P, [big, -big, big], T).tolist() == [big, big]
    assert be.fused_score(P, [2**63 - 1, 0, 0], T).tolist() == [2**63 - 1, 2**63 - 1]


def test_fused_many_patterns_sliced(api):
    # small test side, huge pattern side: exercises the sliced partial-sum path
    rng = np.random.default_rng(3)
    L = 128
    P = random_rows(rng, 60000, L, 0.15)
    T = random_rows(rng, 40, L, 0.7)
    s = rng.integers(0, 2**40, P.shape[0])
    be = api.make_backend("b200")
    assert np.array_equal(be.fused_score(M(api, P, L), s, M(api, T, L)), oracle.fused_score(P, s, T))
    s2 = s.copy()
    s2[::7] *= -1                                        # mixed signs → ordered path
    assert np.array_equal(be.fused_score(M(api, P, L), s2, M(api, T, L)), oracle.fused_score(P, s2, T))
