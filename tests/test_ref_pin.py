"""SPEC.md:636 acceptance 1 — oracle equivalence on randomized datasets.

The plain-C oracle is compared with (a) the reference itself (oracle/_ref, when
built in this container) on 500 random datasets and (b) a naive frozenset
brute force on smaller ones.  Zero tolerance.  CPU only.
"""
import numpy as np
import pytest

from oracle import oracle, ref
from tests.helpers import brute_force_fit, random_rows, sets_to_sorted_words, to_sets


def _case(rng):
    L = int(rng.integers(1, 97))
    dens = float(rng.uniform(0.1, 0.95))
    na, nn = (int(x) for x in rng.integers(1, 41, 2))
    return L, random_rows(rng, na, L, dens), random_rows(rng, nn, L, dens)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (reference absent)")
def test_oracle_vs_reference_500_random():
    rng = np.random.default_rng(636)
    for case in range(500):
        L, Xa, Xn = _case(rng)
        fit = oracle.fit(Xa, Xn, threads=1)
        for c, X, opp in ((0, Xa, Xn), (1, Xn, Xa)):
            r = ref.mine(X, L, pair_batch=int(rng.choice([1, 7, 8192])), backend="reference", threads=1)
            assert np.array_equal(fit.candidates[c].words, r.words), case
            assert np.array_equal(fit.candidates[c].supports, r.supports), case
            assert np.array_equal(fit.candidates[c].scores, r.scores), case
            keep = ref.coverage_any(r.words, L, opp, L, block=int(rng.integers(1, 50))) == 0
            assert np.array_equal(fit.pure[c].words, r.words[keep]), case


def test_oracle_vs_bruteforce_sets():
    rng = np.random.default_rng(637)
    for case in range(150):
        L = int(rng.integers(1, 70))
        dens = float(rng.uniform(0.2, 0.9))
        Xa = random_rows(rng, int(rng.integers(1, 16)), L, dens)
        Xn = random_rows(rng, int(rng.integers(1, 16)), L, dens)
        bf = brute_force_fit(to_sets(Xa), to_sets(Xn))
        fit = oracle.fit(Xa, Xn, threads=1)
        for c in range(2):
            B, sup, sc, pure = bf[c]
            w = sets_to_sorted_words(sorted(B, key=sorted), L)
            assert np.array_equal(fit.candidates[c].words, w), case
            sets = to_sets(fit.candidates[c].words)
            assert [sup[s] for s in sets] == fit.candidates[c].supports.tolist()
            assert [sc[s] for s in sets] == fit.candidates[c].scores.tolist()
            assert set(to_sets(fit.pure[c].words)) == pure
        T = random_rows(rng, 8, L, dens)
        for c in range(2):
            exp = [sum(bf[c][2][b] for b in bf[c][3] if b <= t) for t in to_sets(T)]
            assert oracle.fused_score(fit.pure[c].words, fit.pure[c].scores, T).tolist() == exp
