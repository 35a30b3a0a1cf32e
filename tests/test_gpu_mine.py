"""GPU parity of mine/purify (mine.hpp:35-51) against the
reference-generated golden fixtures and the plain-C oracle.  Bit-exact."""
import os

import numpy as np
import pytest

from oracle import oracle
from tests.helpers import random_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2507_14222_b200 import api as a
    return a


def test_golden_random_cases(api, golden_dir):
    z = np.load(os.path.join(golden_dir, "random_mine.npz"))
    be = api.make_backend("b200")
    for i in range(int(z["count"])):
        p = f"c{i}_"
        L = int(z[p + "L"])
        Xa = api.PackedMatrix(z[p + "attack"], L, "attack")
        Xn = api.PackedMatrix(z[p + "normal"], L, "normal")
        cs = api.enumerate_candidates(Xa, be, api.KernelConfig(pair_batch=int(i % 5) + 1))
        assert np.array_equal(cs.patterns.words, z[p + "ca_words"]), i
        api.count_support(cs, Xa)
        api.score_patterns(cs)
        assert np.array_equal(cs.supports, z[p + "ca_sup"]), i
        assert np.array_equal(cs.scores, z[p + "ca_sc"]), i
        m = api.fit(Xa.words, Xn.words, L)
        for c, key in ((0, "ca"), (1, "cn")):
            d = m.dictionary(c, 0)
            assert np.array_equal(d.words, z[p + key + "_words"]), (i, c)
            assert np.array_equal(d.supports, z[p + key + "_sup"]), (i, c)
            assert np.array_equal(d.scores, z[p + key + "_sc"]), (i, c)
            keep = z[p + ("keep_a" if c == 0 else "keep_n")] == 1
            pd = m.dictionary(c, 1)
            assert np.array_equal(pd.words, z[p + key + "_words"][keep]), (i, c)
            assert np.array_equal(pd.scores, z[p + key + "_sc"][keep]), (i, c)
        A, N = m.evidence(z[p + "tests"])
        assert np.array_equal(A, z[p + "A"]) and np.array_equal(N, z[p + "N"]), i


def test_degenerate_classes(api):
    L = 70
    rng = np.random.default_rng(9)
    row = random_rows(rng, 1, L, 0.5)
    same = np.repeat(row, 37, axis=0)
    cs = api.enumerate_candidates(api.PackedMatrix(same, L))
    assert np.array_equal(cs.patterns.words, row)             # SPEC.md:308 all identical → 1
    a = np.zeros((2, 2), np.int64)
    a[0, 0] = 1
    a[1, 1] = 1                                               # disjoint rows → the two signatures
    cs = api.enumerate_candidates(api.PackedMatrix(a, L))
    assert cs.patterns.rows == 2
    with pytest.raises(api.DataError):
        api.enumerate_candidates(api.PackedMatrix(np.zeros((0, 2), np.int64), L))
    with pytest.raises(api.ConfigError):
        api.enumerate_candidates(api.PackedMatrix(a, L), config=api.KernelConfig(pair_batch=0))
    z = np.zeros((3, 2), np.int64)                            # all-empty rows → no candidates
    assert api.enumerate_candidates(api.PackedMatrix(z, L)).patterns.rows == 0


@pytest.mark.parametrize("n,L,dens", [(600, 96, 0.6), (2500, 300, 0.93), (1500, 1000, 0.985), (300, 12000, 0.9985), (200, 40000, 0.9996)])
def test_fit_vs_oracle_random(api, n, L, dens):
    rng = np.random.default_rng(n + L)
    Xa = random_rows(rng, n, L, dens)
    Xn = random_rows(rng, n + 17, L, dens)
    ref = oracle.fit(Xa, Xn)
    m = api.fit(Xa, Xn, L)
    for c in range(2):
        for which, want in ((0, ref.candidates[c]), (1, ref.pure[c])):
            d = m.dictionary(c, which)
            assert np.array_equal(d.words, want.words), (c, which)
            assert np.array_equal(d.supports, want.supports), (c, which)
            assert np.array_equal(d.scores, want.scores), (c, which)
    T = random_rows(rng, 777, L, dens)
    A, N = m.evidence(T)
    assert np.array_equal(A, oracle.fused_score(ref.pure[0].words, ref.pure[0].scores, T))
    assert np.array_equal(N, oracle.fused_score(ref.pure[1].words, ref.pure[1].scores, T))


def test_progress_callback(api):
    rng = np.random.default_rng(5)
    X = random_rows(rng, 100, 64, 0.7)
    seen = []
    cs = api.enumerate_candidates(api.PackedMatrix(X, 64), progress=lambda d, t, f: seen.append((d, t, f)))
    # pairs (u <= v) of the distinct rows the device enumerates (include/ig_b200.h); 100 distinct rows here
    m = len({tuple(r) for r in X.tolist()})
    total = m * (m + 1) // 2
    assert seen and seen[-1] == (total, total, cs.patterns.rows)
    assert all(a[0] <= b[0] and a[2] <= b[2] and a[1] == total for a, b in zip(seen, seen[1:]))


@pytest.mark.parametrize("bits", [10, 16])
def test_forced_fingerprint_collisions_stay_exact(api, monkeypatch, bits):
    """Fingerprints narrowed to `bits` bits (test knob) make most distinct
    candidates collide: the tile-local and device-wide tables must still keep
    exactly the distinct contents, through as many collision levels as needed."""
    monkeypatch.setenv("IG_TEST_FP_BITS", str(bits))
    rng = np.random.default_rng(bits)
    L = 200
    Xa = random_rows(rng, 150, L, 0.8)
    Xn = random_rows(rng, 130, L, 0.8)
    ref = oracle.fit(Xa, Xn)
    m = api.fit(Xa, Xn, L)
    for c in range(2):
        for which, want in ((0, ref.candidates[c]), (1, ref.pure[c])):
            d = m.dictionary(c, which)
            assert which == 1 or len(want.words) > (8 << bits if bits == 10 else 4000)
            assert np.array_equal(d.words, want.words), (c, which)
            assert np.array_equal(d.supports, want.supports), (c, which)


def test_fit_fuzz_small_shapes(api):
    """Many small random fits (duplicate and empty rows, 1..3 token patterns,
    single-row classes, widths around word boundaries) against the oracle."""
    rng = np.random.default_rng(2024)
    for case in range(30):
        L = int(rng.choice([1, 3, 40, 63, 64, 65, 127, 200, 513]))
        na, nn = (int(x) for x in rng.integers(1, 120, 2))
        dens = float(rng.uniform(0.05, 0.95))
        Xa = random_rows(rng, na, L, dens)
        Xn = random_rows(rng, nn, L, dens)
        if na > 3:
            Xa[1] = Xa[0]                      # duplicate rows
            Xa[2] = 0                          # an empty row
        if nn > 2:
            Xn[0] = Xa[0]                      # a row shared by both classes
        ref = oracle.fit(Xa, Xn)
        m = api.fit(Xa, Xn, L)
        for c in range(2):
            for which, want in ((0, ref.candidates[c]), (1, ref.pure[c])):
                d = m.dictionary(c, which)
                assert np.array_equal(d.words, want.words), (case, c, which)
                assert np.array_equal(d.supports, want.supports), (case, c, which)
                assert np.array_equal(d.scores, want.scores), (case, c, which)
        T = random_rows(rng, int(rng.integers(1, 300)), L, dens)
        A, N = m.evidence(T)
        assert np.array_equal(A, oracle.fused_score(ref.pure[0].words, ref.pure[0].scores, T)), case
        assert np.array_equal(N, oracle.fused_score(ref.pure[1].words, ref.pure[1].scores, T)), case


def _canonical_pair_set(X):
    """Distinct non-empty {X[i] & X[j] : i < j} ∪ {X[i]} in words::less order
    (unsigned lexicographic over words 0..K-1, bitpack.hpp:61-68)."""
    n, k = X.shape
    iu, ju = np.triu_indices(n, 1)
    c = np.concatenate([X & X, X[iu] & X[ju]]).view(np.uint64)
    c = c[(c != 0).any(axis=1)]
    c = np.unique(c, axis=0)  # lexicographic over unsigned columns
    return c.view(np.int64)


@pytest.mark.parametrize("word0_values,expect", [(64, "runs"), (1, "one run")])
def test_canonical_order_long_and_short_key_runs(api, word0_values, expect):
    """> 24,576 candidates, K = 66: the canonical sort (csrc/sort.cu) takes its
    MSD branch (stable sort on the first packed rank key, then ranks by
    counting inside runs of equal first key) when word 0 leaves short runs, and
    its LSD fallback when the first 64 rank bits are constant (one run of every
    candidate).  Both must return exactly the reference's order."""
    rng = np.random.default_rng(7 + word0_values)
    n, k = 250, 66
    X = np.empty((n, k), np.uint64)
    X[:, 1:64] = np.uint64(0x8000000000000001)
    X[:, 0] = rng.integers(1, 2**63, size=word0_values, dtype=np.uint64)[rng.integers(0, word0_values, size=n)]
    X[:, 64:] = rng.integers(0, 2**63, size=(n, 2), dtype=np.uint64) | rng.integers(0, 2**63, size=(n, 2), dtype=np.uint64) << np.uint64(1)
    X = X.view(np.int64)
    want = _canonical_pair_set(X)
    assert want.shape[0] > 24576
    cs = api.enumerate_candidates(api.PackedMatrix(X, 64 * k))
    assert np.array_equal(cs.patterns.words, want)


def _onehot_rows(rng, n, card):
    """One-hot records over categorical fields of the given cardinalities
    (skewed values, like encoded NSL-KDD/CICIDS columns): bool [n, sum(card)]."""
    B = np.zeros((n, sum(card)), bool)
    off = 0
    for c in card:
        v = np.minimum(rng.geometric(0.35, n) - 1, c - 1)
        B[np.arange(n), off + v] = True
        off += c
    return B


@pytest.mark.parametrize("seed", [5, 6])
def test_fit_fuzz_injected_contradictions(api, seed):
    """SPEC.md:643 fuzzed pipeline at ~10^6 candidates: encoded-shape records
    (15 one-hot fields, L = 88), with contradictions injected — 10 % of the
    normal rows are copies of attack rows (every candidate they hold becomes
    impure in both classes) and 4 % are attack rows with extra tokens (supersets
    that cover attack patterns).  Candidates, supports, scores, both pure
    dictionaries and A/N must equal the oracle's exactly."""
    from tests.helpers import pack_bits
    rng = np.random.default_rng(seed)
    card = [3, 5, 8, 2, 12, 4, 6, 2, 9, 3, 7, 2, 5, 16, 4]
    L = sum(card)
    A = _onehot_rows(rng, 2500, card)
    N = _onehot_rows(rng, 2000, card)
    N[:250] = A[rng.choice(len(A), 250, replace=False)]
    N[250:330] = A[rng.choice(len(A), 80, replace=False)] | _onehot_rows(rng, 80, card)
    N = N[rng.permutation(len(N))]
    Xa, Xn = pack_bits(A), pack_bits(N)
    ref = oracle.fit(Xa, Xn)
    assert len(ref.candidates[0].words) > 500_000
    assert len(ref.pure[0].words) < len(ref.candidates[0].words) // 4   # the injections bite
    m = api.fit(Xa, Xn, L)
    for c in range(2):
        for which, want in ((0, ref.candidates[c]), (1, ref.pure[c])):
            d = m.dictionary(c, which)
            assert np.array_equal(d.words, want.words), (c, which)
            assert np.array_equal(d.supports, want.supports), (c, which)
            assert np.array_equal(d.scores, want.scores), (c, which)
    T = pack_bits(_onehot_rows(rng, 3000, card))
    T[:200] = Xn[:200]                                       # test rows equal to training rows
    A_, N_ = m.evidence(T)
    assert np.array_equal(A_, oracle.fused_score(ref.pure[0].words, ref.pure[0].scores, T))
    assert np.array_equal(N_, oracle.fused_score(ref.pure[1].words, ref.pure[1].scores, T))
