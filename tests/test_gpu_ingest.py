"""Device CSV ingest against the host path it replaces:
read_csv -> slice -> infer_schema -> build_columns (+ upload).  The schema must
be identical to the bit (hex-float text), and the encodings of the train and
test columns byte-identical, including the edge cases of the reader and of
std::from_chars."""
import numpy as np
import pytest

from paper_2507_14222_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2507_14222_b200 import api as a
    return a


def _host(api, csv, label, decimals, ratio_k=None, train_rows=None, attack=(), normal=()):
    t = api.read_csv(csv)
    ntr = train_rows if train_rows is not None else ratio_k * t.rows // 10
    tr, te = t.slice(0, ntr), t.slice(ntr, t.rows)
    s = api.infer_schema(tr, label, attack, normal, decimals)
    return s, api.Columns(tr, s, True), api.Columns(te, s, False)


def _same(api, csv, label="label", decimals=1, ratio_k=8, train_rows=None, attack=(), normal=()):
    ctx = api.default_context()
    s1, tr1, te1 = _host(api, csv, label, decimals, ratio_k, train_rows, attack, normal)
    s2, tr2, te2 = api.ingest_csv(csv, label, attack, normal, decimals, train_rows, ratio_k, ctx)
    assert api.schema_to_text(s2) == api.schema_to_text(s1)
    assert tr2.rows == tr1.rows and te2.rows == te1.rows
    e1, e2 = api.encode_training(tr1, ctx), api.encode_training(tr2, ctx)
    assert e2.vocabulary == e1.vocabulary
    for c in range(2):
        assert np.array_equal(e2.matrix(c), e1.matrix(c)), c
    assert e2.removed_rows.tolist() == e1.removed_rows.tolist()
    if te1.rows:
        assert np.array_equal(api.encode_rows(te2, e1, ctx).matrix(2), api.encode_rows(te1, e1, ctx).matrix(2))
    return s2


@pytest.mark.parametrize("rows,ratio_k", [(2000, 8), (15000, 1), (20000, 8)])
def test_nsl_shape_matches_host(api, rows, ratio_k):
    _same(api, synth.nsl_csv(rows, seed=rows), decimals=1, ratio_k=ratio_k)


def test_cicids_shape_matches_host(api):
    _same(api, synth.cicids_csv(6000, seed=5), label="Label", decimals=2, normal=("BENIGN",))


def test_reader_and_number_edge_cases(api):
    rows = [
        "1,a,0.05,normal", "-0,b,-0.0,neptune", "1e3,,1.5E-3,normal", "00012,a,.5,smurf",
        "123456789012345678901,b,1.,normal",       # > 19 digits: host from_chars
        "0.1234567890123456789,a,7e-30,neptune",   # > 15 significant digits / |exp| > 22: host
        "2.5e+2,c,3,normal", "-.25,a,4e22,smurf", ",b,,normal", "7,a,8,neptune",
    ]
    body = "\n".join(rows)
    for csv in (("x,cat,y,label\n" + body + "\n").encode(),           # LF, trailing newline
                ("x,cat,y,label\r\n" + body.replace("\n", "\r\n")).encode(),  # CRLF, no trailing newline
                ("﻿x,cat,y,label\r" + body.replace("\n", "\r") + "\r").encode()):  # BOM, lone CR
        s = _same(api, csv, decimals=2, train_rows=7)
        assert s.column(0)[0] == "numeric" and s.column(1)[0] == "categorical" and s.column(2)[0] == "numeric"


def test_text_makes_a_column_categorical(api):
    # inf / nan / leading '+' / blanks are not finite numbers for from_chars
    for bad in ("inf", "nan", "+1", " 1", "1e", "1.2.3", "0x10", "-"):
        csv = ("x,label\n1,normal\n%s,neptune\n2,normal\n3,neptune\n" % bad).encode()
        s = _same(api, csv, train_rows=4)
        assert s.column(0)[0] == "categorical", bad


def test_quoted_input_takes_the_host_reader(api):
    csv = b'x,"c,d",label\n1,"p,q",normal\n2,r,neptune\n3,"s""t",normal\n'
    _same(api, csv, train_rows=2)


def test_errors_match_host(api):
    with pytest.raises(api.DataError):
        api.ingest_csv(b"a,label\n1,normal\n2\n", train_rows=1)          # ragged record
    with pytest.raises(api.DataError):
        api.ingest_csv(b"a,label\n1,normal\n2,neptune\nxx,normal\n", train_rows=2)  # text in a numeric test cell
    with pytest.raises(api.ConfigError):
        api.ingest_csv(b"a,b\n1,2\n", label_column="label")
    with pytest.raises(api.DataError):
        api.ingest_csv(b"a,label\n1,x\n2,y\n", normal_values=["x"], attack_values=["z"], train_rows=2)
    with pytest.raises(api.DataError):
        api.ingest_csv(b"a,label\n", train_rows=0)


def test_ingested_columns_fit_like_host_columns(api):
    csv = synth.nsl_csv(3000, seed=11)
    ctx = api.default_context()
    _, tr1, te1 = _host(api, csv, "label", 1, ratio_k=8)
    _, tr2, te2 = api.ingest_csv(csv, decimals=1, ratio_k=8, ctx=ctx)
    m1 = api.fit_encoded(api.encode_training(tr1, ctx))
    e2 = api.encode_training(tr2, ctx)
    m2 = api.fit_encoded(e2)
    for c in range(2):
        assert np.array_equal(m1.dictionary(c, 1).words, m2.dictionary(c, 1).words)
    A1, N1 = m1.evidence_encoded(api.encode_rows(te1, api.encode_training(tr1, ctx), ctx))
    A2, N2 = m2.evidence_encoded(api.encode_rows(te2, e2, ctx))
    assert np.array_equal(A1, A2) and np.array_equal(N1, N2)


def test_all_rows_train_and_explicit_counts(api):
    csv = synth.nsl_csv(1500, seed=21)
    ctx = api.default_context()
    s, tr, te = api.ingest_csv(csv, decimals=1, ratio_k=10, ctx=ctx)
    assert tr.rows == 1500 and te.rows == 0
    s2, tr2, te2 = api.ingest_csv(csv, decimals=1, train_rows=999, ctx=ctx)
    assert tr2.rows == 999 and te2.rows == 501
    _same(api, csv, decimals=1, train_rows=999)
    # the ingested training columns prefetch / upload as no-ops (already resident)
    tr2.prefetch(ctx)
    tr2.upload(ctx)
    assert np.array_equal(api.encode_training(tr2, ctx).matrix(0),
                          api.encode_training(_host(api, csv, "label", 1, train_rows=999)[1], ctx).matrix(0))
