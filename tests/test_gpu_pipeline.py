"""GPU parity of the whole path on NSL-shape data: tokenise/pack (kernel 1),
fit (2)-(5) and evidence (6) against the reference's golden digests (C1) and
the plain-C oracle computed live (C2 in full; C3 fit in full, matcher on a
bounded test sample)."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle, pipeline
from paper_2507_14222_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2507_14222_b200 import api as a
    return a


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def test_tokenizer_golden_runs(api, golden_dir):
    g = json.load(open(os.path.join(golden_dir, "tokenizer.json")))
    for name, run in g["runs"].items():
        t = api.read_csv(run["csv"].encode())
        tr = t.slice(0, run["train_rows"])
        s = api.infer_schema(tr, "label", decimals=run["decimals"])
        enc = api.encode_training(api.Columns(tr, s, True))
        assert enc.vocabulary == run["vocab"], name
        assert enc.logical_len == run["L"]
        assert enc.matrix(0).tolist() == run["attack"], name
        assert enc.matrix(1).tolist() == run["normal"], name
        assert enc.removed_rows.tolist() == run["removed"], name


def test_tokenizer_errors(api):
    t = api.read_csv(b"a,label\n1,normal\n1,normal\n")
    s = api.infer_schema(t, "label")
    with pytest.raises(api.DataError):  # only one class
        api.encode_training(api.Columns(t, s, True))
    t = api.read_csv(b"a,label\n1,normal\n1,neptune\n")
    s = api.infer_schema(t, "label")
    with pytest.raises(api.DataError):  # filter empties both classes
        api.encode_training(api.Columns(t, s, True))
    tr = api.read_csv(b"a,label\n1,normal\n2,neptune\n")
    s = api.infer_schema(tr, "label")
    with pytest.raises(api.DataError):  # unparsable test cell in a numeric column
        api.Columns(api.read_csv(b"a,label\nx,normal\n"), s, False)


def test_nsl_c1_golden_end_to_end(api, golden_dir):
    g = json.load(open(os.path.join(golden_dir, "nsl_c1.json")))
    csv = synth.nsl_csv(g["rows"], seed=g["seed"])
    r = api.train_and_score(csv, decimals=g["decimals"], ratio_k=g["ratio_k"])
    assert r.train.logical_len == g["L"]
    assert hashlib.sha256("\n".join(r.train.vocabulary).encode()).hexdigest() == g["vocab_sha256"]
    assert _digest(r.train.matrix(0), r.train.matrix(1), r.test.matrix(2)) == g["rows_digest"]
    for c in range(2):
        d = r.model.dictionary(c, 0)
        assert _digest(d.words, d.supports, d.scores) == g["cand_digest"][c]
        p = r.model.dictionary(c, 1)
        assert _digest(p.words, p.supports, p.scores) == g["pure_digest"][c]
    assert _digest(r.A) == g["A_digest"] and _digest(r.N) == g["N_digest"]
    mu, sg = api.fit_normal_stats(r.N)
    label, reg = api.classify(r.A, r.N, mu, sg, 0.568)
    assert _digest(label) == g["labels_digest"] and _digest(reg) == g["regulation_digest"]


def _oracle_encode(csv, ratio_k=None, train_rows=None, decimals=1):
    hdr, rows = pipeline.read_csv(csv)
    ntr = train_rows if train_rows is not None else ratio_k * len(rows) // 10
    sch = pipeline.infer_schema(hdr, rows[:ntr], "label", decimals=decimals)
    enc = pipeline.encode_training(rows[:ntr], sch)
    return hdr, rows, ntr, sch, enc


@pytest.mark.parametrize("rows,ratio_k,test_sample", [(15000, 8, None)])
def test_nsl_fit_vs_oracle(api, rows, ratio_k, test_sample):
    """C2 (15k, 80/20) in full against the plain-C oracle computed live (C3 and
    C4 in full against the reference's digests: test_gpu_fullsize_golden.py)."""
    csv = synth.nsl_csv(rows, seed=2507)
    r = api.train_and_score(csv, decimals=1, ratio_k=ratio_k)
    Xa, Xn = r.train.matrix(0), r.train.matrix(1)
    T = r.test.matrix(2)
    # encode parity on the first rows with the Python restatement (bounded cost)
    if rows <= 15000:
        hdr, prow, ntr, sch, enc = _oracle_encode(csv, ratio_k=ratio_k)
        assert enc.vocab == r.train.vocabulary
        assert np.array_equal(enc.attack, Xa) and np.array_equal(enc.normal, Xn)
        assert np.array_equal(pipeline.encode_rows(prow[ntr:ntr + 2000], sch, enc.vocab), T[:2000])
    ref = oracle.fit(Xa, Xn)
    for c in range(2):
        for which, want in ((0, ref.candidates[c]), (1, ref.pure[c])):
            d = r.model.dictionary(c, which)
            assert np.array_equal(d.words, want.words), (c, which)
            assert np.array_equal(d.supports, want.supports), (c, which)
            assert np.array_equal(d.scores, want.scores), (c, which)
    idx = np.arange(T.shape[0]) if test_sample is None else \
        np.random.default_rng(7).choice(T.shape[0], test_sample, replace=False)
    A = oracle.fused_score(ref.pure[0].words, ref.pure[0].scores, T[idx])
    N = oracle.fused_score(ref.pure[1].words, ref.pure[1].scores, T[idx])
    assert np.array_equal(r.A[idx], A) and np.array_equal(r.N[idx], N)


def test_prefetched_columns_encode_identically(api, golden_dir):
    """ig_columns_prefetch: the copy-stream transfer feeds the next encode with
    the same bytes as the synchronous path (and is consumed once)."""
    g = json.load(open(os.path.join(golden_dir, "nsl_c1.json")))
    csv = synth.nsl_csv(g["rows"], seed=g["seed"])
    table = api.read_csv(csv)
    ntr = g["ratio_k"] * table.rows // 10
    tr, te = table.slice(0, ntr), table.slice(ntr, table.rows)
    schema = api.infer_schema(tr, "label", decimals=g["decimals"])
    ctr, cte = api.Columns(tr, schema, True), api.Columns(te, schema, False)
    ctx = api.default_context()
    want = api.encode_training(ctr, ctx)
    ctr.prefetch(ctx)
    got = api.encode_training(ctr, ctx)
    assert got.vocabulary == want.vocabulary
    for c in range(2):
        assert np.array_equal(got.matrix(c), want.matrix(c))
    t_want = api.encode_rows(cte, want, ctx).matrix(2)
    cte.prefetch(ctx)
    t_got = api.encode_rows(cte, want, ctx).matrix(2)
    assert np.array_equal(t_got, t_want)
    assert np.array_equal(api.encode_rows(cte, want, ctx).matrix(2), t_want)  # prefetch consumed
    assert _digest(t_want) == _digest(api.train_and_score(csv, decimals=g["decimals"],
                                                          ratio_k=g["ratio_k"]).test.matrix(2))
    cte.prefetch(ctx)  # dropped unconsumed when the columns are freed
    del cte


def test_background_test_index_overlapping_the_fit(api, golden_dir):
    """encode_rows before the fit (resident columns: packed and indexed on the
    index stream while the fit runs) gives the same A/N, host or device outputs."""
    import torch
    g = json.load(open(os.path.join(golden_dir, "nsl_c1.json")))
    csv = synth.nsl_csv(g["rows"], seed=g["seed"])
    table = api.read_csv(csv)
    ntr = g["ratio_k"] * table.rows // 10
    tr, te = table.slice(0, ntr), table.slice(ntr, table.rows)
    schema = api.infer_schema(tr, "label", decimals=g["decimals"])
    ctx = api.default_context()
    dtr = api.Columns(tr, schema, True).upload(ctx)
    dte = api.Columns(te, schema, False).upload(ctx)
    enc = api.encode_training(dtr, ctx)
    tenc = api.encode_rows(dte, enc, ctx)
    model = api.fit_encoded(enc)
    dA = torch.zeros(tenc.rows(2), dtype=torch.int64, device="cuda")
    dN = torch.zeros_like(dA)
    model.evidence_encoded_device(tenc, dA.data_ptr(), dN.data_ptr())
    torch.cuda.synchronize()
    A, N = model.evidence_encoded(tenc)
    assert _digest(A) == g["A_digest"] and _digest(N) == g["N_digest"]
    assert np.array_equal(dA.cpu().numpy(), A) and np.array_equal(dN.cpu().numpy(), N)
    assert _digest(tenc.matrix(2)) == _digest(api.encode_rows(api.Columns(te, schema, False), enc, ctx).matrix(2))


def test_fused_fit_evidence_matches_separate_calls(api, golden_dir):
    import torch
    g = json.load(open(os.path.join(golden_dir, "nsl_c1.json")))
    csv = synth.nsl_csv(g["rows"], seed=g["seed"])
    ctx = api.default_context()
    _, tr, te = api.ingest_csv(csv, decimals=g["decimals"], ratio_k=g["ratio_k"], ctx=ctx)
    enc = api.encode_training(tr, ctx)
    tenc = api.encode_rows(te, enc, ctx)
    model, A, N = api.fit_evidence_encoded(enc, tenc)
    assert _digest(A) == g["A_digest"] and _digest(N) == g["N_digest"]
    for c in range(2):
        p = model.dictionary(c, 1)
        assert _digest(p.words, p.supports, p.scores) == g["pure_digest"][c]
    dA = torch.zeros(tenc.rows(2), dtype=torch.int64, device="cuda")
    dN = torch.zeros_like(dA)
    tenc2 = api.encode_rows(te, enc, ctx)
    api.fit_evidence_encoded(enc, tenc2, d_A_ptr=dA.data_ptr(), d_N_ptr=dN.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(dA.cpu().numpy(), A) and np.array_equal(dN.cpu().numpy(), N)


def test_narrow_column_copy_edge_values(api):
    """ig_columns_prefetch's narrow exact form (host_pipeline.hpp) on values that
    stress it — negatives, -0.0, empty cells, integers past int16 / int32,
    many decimals, a column that needs the raw doubles — encodes exactly like
    the raw path (the host checks every code bitwise; this checks the decode)."""
    rng = np.random.default_rng(11)
    n = 3000
    cols = {
        "small": rng.integers(-100, 100, n).astype(str),
        "wide": rng.integers(-(2 ** 40), 2 ** 40, n).astype(str),
        "mid": rng.integers(-70000, 70000, n).astype(str),
        "rate": np.char.mod("%.2f", rng.random(n)),
        "fine": np.char.mod("%.6f", rng.normal(0, 1, n)),
        "raw": np.char.mod("%.17g", rng.normal(0, 1e-3, n)),
        "negzero": np.where(rng.random(n) < 0.5, "-0.0", "0.5"),
    }
    for k in cols:
        cols[k] = np.where(rng.random(n) < 0.05, "", cols[k])  # empty cells
    label = np.where(rng.random(n) < 0.4, "attack", "normal")
    head = ",".join(list(cols) + ["label"])
    body = "\n".join(",".join([cols[k][i] for k in cols] + [label[i]]) for i in range(n))
    table = api.read_csv((head + "\n" + body + "\n").encode())
    tr, te = table.slice(0, 1000), table.slice(1000, n)
    schema = api.infer_schema(tr, "label", decimals=2)
    ctx = api.default_context()
    want = api.encode_training(api.Columns(tr, schema, True), ctx)
    ctr, cte = api.Columns(tr, schema, True), api.Columns(te, schema, False)
    assert cte.nbytes < (n - 1000) * 8 * len(cols)  # the narrow form is smaller than the doubles
    ctr.prefetch(ctx)
    got = api.encode_training(ctr, ctx)
    assert got.vocabulary == want.vocabulary
    for c in range(2):
        assert np.array_equal(got.matrix(c), want.matrix(c))
    t_want = api.encode_rows(api.Columns(te, schema, False), want, ctx).matrix(2)
    cte.prefetch(ctx)
    assert np.array_equal(api.encode_rows(cte, want, ctx).matrix(2), t_want)
