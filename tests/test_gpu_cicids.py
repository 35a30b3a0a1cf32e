"""CICIDS-shape (78 numeric columns, p = 2, wide token universe: K ≈ 80-90 words)
through the whole device path — exercises the wide-row code paths (32-row pair
tiles, 64-bit-K rank-space fallbacks) against the reference and the oracle."""
import numpy as np
import pytest

from oracle import oracle, ref
from paper_2507_14222_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rows", [6000, 14000])
def test_cicids_shape_fit_and_evidence(rows):
    from paper_2507_14222_b200 import api
    csv = synth.cicids_csv(rows, seed=3)
    r = api.train_and_score(csv, label_column="Label", normal_values=["BENIGN"], decimals=2, ratio_k=8)
    L = r.train.logical_len
    assert (L + 63) // 64 >= 64  # wide rows
    Xa, Xn, T = r.train.matrix(0), r.train.matrix(1), r.test.matrix(2)
    if ref.available():
        rr = ref.run(csv, label_col="Label", normal_values="BENIGN", decimals=2, ratio_k=8, stages=0)
        assert rr.vocab == r.train.vocabulary
        assert np.array_equal(rr.attack, Xa) and np.array_equal(rr.normal, Xn)
    fit = oracle.fit(Xa, Xn)
    for c in range(2):
        for which, want in ((0, fit.candidates[c]), (1, fit.pure[c])):
            d = r.model.dictionary(c, which)
            assert np.array_equal(d.words, want.words), (c, which)
            assert np.array_equal(d.supports, want.supports), (c, which)
            assert np.array_equal(d.scores, want.scores), (c, which)
    idx = np.random.default_rng(1).choice(T.shape[0], 300, replace=False)
    assert np.array_equal(r.A[idx], oracle.fused_score(fit.pure[0].words, fit.pure[0].scores, T[idx]))
    assert np.array_equal(r.N[idx], oracle.fused_score(fit.pure[1].words, fit.pure[1].scores, T[idx]))
