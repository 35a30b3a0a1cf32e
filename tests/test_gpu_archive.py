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
        assert np.array_equal(a.supports, b.supports)


def test_archive_fields_provenance_and_frozen_stats(trained):
    """format_version, classifier params (r, stats mode with
    frozen mu_N / sigma_N), provenance (input digest, tool version); the C-ABI
    writer (ig_model_save) keeps all of them through load -> save."""
    import hashlib
    api, te, schema, enc, model, tenc, A, N = trained
    mu, sg = api.fit_normal_stats(N)
    prov = "input_sha256=" + hashlib.sha256(b"synthetic nsl 3000 seed 12").hexdigest() + "\ncreated=2026-10-19T00:00Z"
    blob = api.save_model(model, schema, enc.vocabulary, r=0.75, stats=(mu, sg), provenance=prov)
    text = blob.decode("utf-8", errors="surrogateescape")
    lines = text.split("\n")
    assert lines[0] == "ig-b200-archive 2" and lines[1] == "format_version 2"
    assert lines[2].startswith("tool ig_b200 ")
    assert lines[4].startswith("r ") and float.fromhex(lines[4][2:]) == 0.75
    assert lines[5].startswith("stats_mode frozen ")
    loaded = api.load_model(blob)
    assert loaded.provenance == prov and loaded.r == 0.75 and loaded.stats == (mu, sg)
    assert api.save_model(loaded.model, loaded.schema, loaded.vocabulary, r=loaded.r, stats=loaded.stats,
                          provenance=loaded.provenance) == blob
    for bad in (blob[:-5], blob.replace(b"format_version 2", b"format_version 9"), b"not an archive\n"):
        with pytest.raises(api.DataError):
            api.load_model(bad)


def test_explain_matches_brute_force_subset_scan(trained):
    """ig_explain's index sets equal a numpy brute force
    {p : (P[p] & row) == P[p]} over the whole pure dictionary."""
    api, te, schema, enc, model, tenc, A, N = trained
    T = tenc.matrix(2)
    rng = np.random.default_rng(454)
    for cls in range(2):
        P = model.dictionary(cls, 1).words.view(np.uint64)
        for t in rng.choice(T.shape[0], 25, replace=False):
            row = T[t].view(np.uint64)
            want = np.nonzero(np.all((P & row) == P, axis=1))[0]
            got = api.explain(model, T[t], cls)
            assert np.array_equal(got, want), (cls, t)


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
