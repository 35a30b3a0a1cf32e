"""C4 (148,517 NSL-shape records, 80/20: 118,813 training rows, ~17 M
candidates and ~16 M pure patterns per class) at full size.  The oracle would
take CPU-hours here, so parity is checked through properties
that do not depend on size, each against a plain numpy restatement of the
reference's definition on a seeded sample:

  * canonical order: every dictionary strictly increasing in `words::less`
    (unsigned word-lexicographic, bitpack.hpp:59-68) — also proves the dedup;
  * completeness: for sampled pairs (i, j) of a class, X[i] & X[j] is in B^c,
    and it is in P^c exactly when no opposite-class row contains it
    (SPEC.md:301-309, 371-379);
  * support / score: f = #{class rows ⊇ b} over all rows, S = f·|b|²
     for sampled candidates and pure patterns;
  * purity: no sampled pure pattern is contained in an opposite-class row;
  * evidence: A/N of sampled test rows = Σ score over contained pure patterns
    (SPEC.md:424-428);
  * determinism: a second fit of the same encoding is byte-identical.
"""
import numpy as np
import pytest

from paper_2507_14222_b200 import synth

pytestmark = pytest.mark.gpu

C4_ROWS, C4_RATIO = 148517, 8
_MUL = np.uint64(0x9E3779B97F4A7C15)


@pytest.fixture(scope="module")
def c4():
    from paper_2507_14222_b200 import api
    csv = synth.nsl_csv(C4_ROWS, seed=2507)
    r = api.train_and_score(csv, decimals=1, ratio_k=C4_RATIO)
    X = [r.train.matrix(0).view(np.uint64), r.train.matrix(1).view(np.uint64)]
    D = {(c, w): r.model.dictionary(c, w) for c in range(2) for w in range(2)}
    return api, r, X, D


def _row_hash(U):
    h = np.zeros(U.shape[0], np.uint64)
    with np.errstate(over="ignore"):
        for w in range(U.shape[1]):
            h = (h ^ U[:, w]) * _MUL
            h ^= h >> np.uint64(29)
    return h


def _popcount(U):
    return np.unpackbits(np.ascontiguousarray(U).view(np.uint8), axis=-1).sum(axis=-1, dtype=np.int64)


def _contained_in_any(p, X):
    return bool(((X & p) == p).all(axis=1).any())


def _support(p, X):
    return int(((X & p) == p).all(axis=1).sum())


def test_dictionaries_are_strictly_canonical(c4):
    _, _, _, D = c4
    for key, d in D.items():
        U = d.words.view(np.uint64)
        assert U.shape[0] > 1_000_000, key  # full size, not a toy
        for s in range(0, U.shape[0] - 1, 1 << 21):
            a, b = U[s:s + (1 << 21)], U[s + 1:s + 1 + (1 << 21)]
            a = a[:b.shape[0]]
            ne = a != b
            assert ne.any(axis=1).all(), key  # no duplicates
            first = ne.argmax(axis=1)
            r = np.arange(first.shape[0])
            assert (b[r, first] > a[r, first]).all(), key  # increasing


def test_sampled_pairs_are_enumerated_and_purified(c4):
    _, _, X, D = c4
    rng = np.random.default_rng(4)
    for c in range(2):
        hc, hp = _row_hash(D[(c, 0)].words.view(np.uint64)), _row_hash(D[(c, 1)].words.view(np.uint64))
        Uc, Up = D[(c, 0)].words.view(np.uint64), D[(c, 1)].words.view(np.uint64)
        n = X[c].shape[0]
        checked_pure = checked_impure = 0
        for _ in range(150):
            i, j = sorted(rng.choice(n, 2, replace=False))
            p = X[c][i] & X[c][j]
            if not p.any():
                continue
            h = _row_hash(p[None, :])[0]
            hits = np.nonzero(hc == h)[0]
            assert any(np.array_equal(Uc[t], p) for t in hits), (c, i, j)
            pure = not _contained_in_any(p, X[1 - c])
            hits = np.nonzero(hp == h)[0]
            assert any(np.array_equal(Up[t], p) for t in hits) == pure, (c, i, j)
            checked_pure += pure
            checked_impure += not pure
        assert checked_pure > 0 and checked_pure + checked_impure > 100, (checked_pure, checked_impure)
        # every training row is its own candidate (the diagonal)
        for i in rng.choice(n, 20, replace=False):
            h = _row_hash(X[c][i][None, :])[0]
            assert any(np.array_equal(Uc[t], X[c][i]) for t in np.nonzero(hc == h)[0])


def test_sampled_supports_scores_and_purity(c4):
    _, _, X, D = c4
    rng = np.random.default_rng(5)
    for c in range(2):
        for w in range(2):
            d = D[(c, w)]
            U = d.words.view(np.uint64)
            for t in rng.choice(U.shape[0], 60, replace=False):
                p = U[t]
                f = _support(p, X[c])
                assert d.supports[t] == f, (c, w, t)
                assert d.scores[t] == f * int(_popcount(p)) ** 2, (c, w, t)
                if w == 1:
                    assert not _contained_in_any(p, X[1 - c]), (c, t)


def test_sampled_evidence(c4):
    _, r, _, D = c4
    T = r.test.matrix(2).view(np.uint64)
    rng = np.random.default_rng(6)
    for t in rng.choice(T.shape[0], 3, replace=False):
        row = T[t]
        for c, ev in ((0, r.A), (1, r.N)):
            P = D[(c, 1)]
            U = P.words.view(np.uint64)
            hit = ((U & row) == U).all(axis=1)
            assert ev[t] == int(P.scores[hit].sum()), (c, t)


def test_refit_is_byte_identical(c4):
    api, r, _, D = c4
    m2 = api.fit_encoded(r.train)
    for (c, w), d in D.items():
        d2 = m2.dictionary(c, w)
        assert np.array_equal(d2.words, d.words), (c, w)
        assert np.array_equal(d2.supports, d.supports) and np.array_equal(d2.scores, d.scores), (c, w)
    A2, N2 = m2.evidence_encoded(r.test)
    assert np.array_equal(A2, r.A) and np.array_equal(N2, r.N)
