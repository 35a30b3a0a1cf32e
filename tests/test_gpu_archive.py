"""ModelArchive round trip and explain."""
import numpy as np
import pytest

from paper_2507_14222_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def trained():
    from paper_2507_14222_b200 import api
    csv = synth.nsl_csv(3000, seed=12)
    table = api.read_csv(csv)
    ntr = 8 * table.rows // 10
    tr, te = table.slice(0, ntr), table.slice(ntr, table.rows)
    schema = api.infer_schema(tr, "label", decimals=1)
    enc = api.encode_training(api.Columns(tr, schema, True))
    model = api.fit_encoded(enc)
    tenc = api.encode_rows(api.Columns(te, schema, False), enc)
    A, N = model.evidence_encoded(tenc)
    return api, te, schema, enc, model, tenc, A, N


def test_archive_round_trip_is_byte_stable_and_predicts_identically(trained):
    api, te, schema, enc, model, tenc, A, N = trained
    blob = api.save_model(model, schema, enc.vocabulary)
    loaded = api.load_model(blob)
    assert api.save_model(loaded.model, loaded.schema, loaded.vocabulary) == blob
    t2 = api.encode_rows(api.Columns(te, loaded.schema, False), loaded.encoding)
    assert np.array_equal(t2.matrix(2), tenc.matrix(2))
    A2, N2 = loaded.model.evidence_encoded(t2)
    assert np.array_equal(A2, A) and np.array_equal(N2, N)
    for c in range(2):
        a, b = model.dictionary(c, 1), loaded.model.dictionary(c, 1)
        assert np.array_equal(a.words, b.words) and np.array_equal(a.scores, b.scores)


def test_explain_scores_sum_to_evidence(trained):
    api, te, schema, enc, model, tenc, A, N = trained
    T = tenc.matrix(2)
    dicts = [model.dictionary(0, 1), model.dictionary(1, 1)]
    vocab = enc.vocabulary
    rng = np.random.default_rng(3)
    for t in rng.choice(T.shape[0], 40, replace=False):
        ex = api.explain_row(model, T[t], vocab, dicts)
        assert ex["A"] == A[t] and ex["N"] == N[t]  # SPEC.md:465 score consistency
        for item in ex["attack"]:
            assert all(tok in vocab for tok in item["tokens"])
    empty = np.zeros_like(T[0])
    ex = api.explain_row(model, empty, vocab, dicts)
    assert ex["attack"] == [] and ex["normal"] == [] and ex["A"] == 0 and ex["N"] == 0
