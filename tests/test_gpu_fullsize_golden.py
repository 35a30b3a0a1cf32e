"""Full-size parity pinned to the reference: C3 (148,517 records, 10/90) and
C4 (148,517, 80/20), every output of the CUDA path against digests of
oracle/_ref's outputs (tests/golden/make_fullsize.py) — tokenisation (schema,
vocabulary, attack / normal / test rows), both candidate dictionaries B^c and
both pure dictionaries P^c (words, supports, scores, canonical order), all
A / N rows, the normal statistics and the labels.  Bit-exact, no sampling.

The reference outputs these digests stand for: proj/src/pipeline.cpp:107-339
(schema, encode), SPEC.md:301-379 (mine, purify; restated in
oracle/ref_shim.cpp on the reference's ParallelCpuBackend),
proj/src/kernels.cpp:105-118 + SPEC.md:424-452 (evidence, infer)."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2507_14222_b200 import synth

pytestmark = pytest.mark.gpu


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def _blocks(block, *arrays):
    n = arrays[0].shape[0]
    return [_digest(*(a[i:i + block] for a in arrays)) for i in range(0, n, block)]


def _first_bad(want, got):
    for i, (w, g) in enumerate(zip(want, got)):
        if w != g:
            return i
    return None if len(want) == len(got) else min(len(want), len(got))


def _golden(golden_dir, name):
    path = os.path.join(golden_dir, f"{'cicids' if name == 'c5s' else 'nsl'}_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/golden/make_fullsize.py {name})")
    return json.load(open(path))


def _schema_digest(schema, ncols):
    """(kind, mean, std) per column as igref_run_schema reports them; the label
    column keeps ColumnSchema's defaults (categorical, 0, 0; pipeline.hpp:17-22)."""
    kind = np.array([0 if schema.column(j)[0] == "numeric" else 1 for j in range(ncols)], np.uint8)
    mean = np.array([schema.column(j)[1] for j in range(ncols)])
    sd = np.array([schema.column(j)[2] for j in range(ncols)])
    kind[schema.label_index] = 1
    mean[schema.label_index] = sd[schema.label_index] = 0.0
    return _digest(kind, mean, sd)


def _check_encoding(g, enc, tenc):
    assert enc.logical_len == g["L"]
    assert hashlib.sha256("\n".join(enc.vocabulary).encode()).hexdigest() == g["vocab_sha256"]
    assert enc.removed_rows.shape[0] == g["removed"]
    assert _digest(enc.matrix(0)) == g["attack_digest"], "attack rows differ from the reference encode"
    assert _digest(enc.matrix(1)) == g["normal_digest"], "normal rows differ from the reference encode"
    assert _digest(tenc.matrix(2)) == g["tests_digest"], "test rows differ from the reference encode_rows"


def _check_model(g, model):
    for c in range(2):
        for which, key in ((0, "cand"), (1, "pure")):
            d = model.dictionary(c, which)
            assert d.words.shape[0] == g[f"{key}_counts"][c], (key, c)
            got = _digest(d.words, d.supports, d.scores)
            if got != g[f"{key}_digest"][c]:
                bad = _first_bad(g[f"{key}_blocks"][c], _blocks(g["dict_block"], d.words, d.supports, d.scores))
                pytest.fail(f"{key} dictionary of class {c} differs from the reference (first block {bad} "
                            f"of {g['dict_block']} patterns)")
            if which == 1:
                assert int(d.scores.astype(object).sum()) == g["score_totals"][c]


def _check_evidence(g, A, N, api):
    for name, v in (("A", A), ("N", N)):
        if _digest(v) != g[f"{name}_digest"]:
            bad = _first_bad(g[f"{name}_blocks"], _blocks(g["an_block"], v))
            pytest.fail(f"{name} differs from the reference (first block {bad} of {g['an_block']} rows)")
    mu, sg = api.fit_normal_stats(N)
    assert mu == g["mu"] and sg == g["sigma"]
    label, reg = api.classify(A, N, mu, sg, 0.568)
    assert _digest(label) == g["labels_digest"] and _digest(reg) == g["regulation_digest"]


@pytest.fixture(scope="module")
def api():
    from paper_2507_14222_b200 import api as a
    return a


@pytest.mark.parametrize("name,prefetch", [("c3", False), ("c4", False), ("c5s", False), ("c3", True),
                                           ("c5s", True)])
def test_fullsize_host_pipeline_vs_reference(api, golden_dir, name, prefetch):
    """Host CSV reader + schema -> device encode -> fused fit + evidence, every
    output against the reference's digests.  prefetch: the columns go over in
    their narrow exact form (ig_columns_prefetch; code / scale per column,
    decoded on the device) — the bench's e2e path.  c5s: configs[4]'s CICIDS
    shape (p = 2, wide rows) on a 25,000-record sample."""
    g = _golden(golden_dir, name)
    gen = synth.cicids_csv if g.get("shape") == "cicids" else synth.nsl_csv
    csv = gen(g["rows"], seed=g["seed"])
    assert hashlib.sha256(csv).hexdigest() == g["csv_sha256"]
    ctx = api.default_context()
    table = api.read_csv(csv)
    ntr = g["ratio_k"] * table.rows // 10
    assert ntr == g["n_train"]
    tr, te = table.slice(0, ntr), table.slice(ntr, table.rows)
    normal = [g["normal_values"]] if g.get("normal_values") else []
    schema = api.infer_schema(tr, g.get("label", "label"), normal_values=normal, decimals=g["decimals"])
    assert _schema_digest(schema, table.columns) == g["schema_digest"]
    ctr, cte = api.Columns(tr, schema, True), api.Columns(te, schema, False)
    if prefetch:
        ctr.prefetch(ctx)
        cte.prefetch(ctx)
    enc = api.encode_training(ctr, ctx)
    tenc = api.encode_rows(cte, enc, ctx)
    _check_encoding(g, enc, tenc)
    model, A, N = api.fit_evidence_encoded(enc, tenc)
    _check_evidence(g, A, N, api)
    _check_model(g, model)


def test_fullsize_device_ingest_vs_reference(api, golden_dir):
    """Device CSV ingest (ig_ingest_csv: records, numbers, schema statistics on
    the GPU) at C3 -> the same tokens, rows and evidence as the reference."""
    g = _golden(golden_dir, "c3")
    csv = synth.nsl_csv(g["rows"], seed=g["seed"])
    ctx = api.default_context()
    schema, tr, te = api.ingest_csv(csv, decimals=g["decimals"], ratio_k=g["ratio_k"], ctx=ctx)
    assert _schema_digest(schema, 42) == g["schema_digest"]
    enc = api.encode_training(tr, ctx)
    tenc = api.encode_rows(te, enc, ctx)
    _check_encoding(g, enc, tenc)
    model, A, N = api.fit_evidence_encoded(enc, tenc)
    _check_evidence(g, A, N, api)
