"""CPU checks of the product library: it loads, exports every symbol
include/ig_b200.h declares, and its host-side pipeline pieces (CSV reader,
schema inference, checked total, config validation, infer/eval arithmetic)
match the reference semantics.  No GPU compute is called here."""
import json
import math
import os
import re

import numpy as np
import pytest

from oracle import pipeline as opipe

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "ig_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ig_[a-z0-9_]+)\s*\(", src)) - {"ig_progress_fn"})


def test_library_exports_every_declared_symbol():
    from paper_2507_14222_b200 import _native
    syms = _header_symbols()
    assert len(syms) >= 50
    for s in syms:
        assert hasattr(_native.lib, s), s
    bound = {name for name, _, _ in _native.SIGNATURES}
    assert set(syms) == bound


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2507_14222_b200", "libig_b200.so")
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_csv_reader_matches_reference_restatement(golden_dir):
    from paper_2507_14222_b200 import api
    g = json.load(open(os.path.join(golden_dir, "tokenizer.json")))
    for name, run in g["runs"].items():
        csv = run["csv"].encode()
        t = api.read_csv(csv)
        hdr, rows = opipe.read_csv(csv)
        assert t.rows == len(rows) and t.columns == len(hdr)
        tr = t.slice(0, run["train_rows"])
        s = api.infer_schema(tr, "label", decimals=run["decimals"])
        for j in range(t.columns - 1):
            kind, mean, sd = s.column(j)
            assert (0 if kind == "numeric" else 1) == run["kind"][j]
            assert mean == run["mean"][j] and sd == run["std"][j]


@pytest.mark.parametrize("bad, exc", [
    (b"a,b\n1,2\n3\n", "DataError"),
    (b"a,b\n\"1,2\n", "DataError"),
    (b"", "DataError"),
])
def test_csv_errors(bad, exc):
    from paper_2507_14222_b200 import api
    with pytest.raises(getattr(api, exc)):
        api.read_csv(bad)


def test_schema_errors():
    from paper_2507_14222_b200 import api
    t = api.read_csv(b"a,label\n1,normal\n2,neptune\n")
    with pytest.raises(api.ConfigError):
        api.infer_schema(t, "nolabel")
    with pytest.raises(api.ConfigError):
        api.infer_schema(t, "label", decimals=13)
    with pytest.raises(api.DataError):
        api.infer_schema(t, "label", attack_values=["neptune"], normal_values=["x"])
    with pytest.raises(api.DataError):
        api.infer_schema(api.read_csv(b"a,label\n"), "label")


def test_total_score_checked():
    from paper_2507_14222_b200 import api
    assert api.total_score(np.array([1, 2, 3])) == 6
    with pytest.raises(api.IGArithmeticError):
        api.total_score(np.array([2**62, 2**62]))


def test_config_and_backend_factory():
    from paper_2507_14222_b200 import api
    with pytest.raises(api.ConfigError):
        api.KernelConfig(pair_batch=0).validate()
    with pytest.raises(api.ConfigError):
        api.KernelConfig(coverage_block=0).validate()
    with pytest.raises(api.ConfigError, match="available: b200"):
        api.make_backend("cuda-magic")
    assert api.backend_names() == ["b200"]


def test_decision_table_property():
    """procedural R1-R3 == closed form on 10^6 random tuples."""
    from paper_2507_14222_b200 import api
    rng = np.random.default_rng(639)
    n = 1_000_000
    A = rng.integers(0, 50, n)
    Nv = rng.integers(0, 50, n)
    mu = float(rng.uniform(0, 60))
    sg = float(rng.uniform(0, 20))
    r = float(rng.uniform(0, 2))
    label, reg = api.classify(A, Nv, mu, sg, r)
    closed = (A >= Nv) | (Nv.astype(float) < opipe.fma(-r, sg, mu))
    assert np.array_equal(label.astype(bool), closed)
    idx = rng.integers(0, n, 2000)
    for i in idx:
        assert (int(label[i]), int(reg[i])) == opipe.classify(int(A[i]), int(Nv[i]), mu, sg, r)


def test_metrics_against_direct_formulas():
    """confusion metrics to 1e-12; rank AUC vs the O(P*N) pairwise oracle."""
    from paper_2507_14222_b200 import api
    rng = np.random.default_rng(640)
    for _ in range(2000):
        n = int(rng.integers(1, 60))
        truth = rng.integers(0, 2, n)
        pred = rng.integers(0, 2, n)
        m = rng.integers(-5, 5, n)
        got = api.compute_metrics(pred, truth, m)
        tp = int(((pred == 1) & (truth == 1)).sum())
        fp = int(((pred == 1) & (truth == 0)).sum())
        fn = int(((pred == 0) & (truth == 1)).sum())
        tn = n - tp - fp - fn
        assert math.isclose(got["accuracy"], (tp + tn) / n, abs_tol=1e-12)
        assert math.isclose(got["recall"], tp / (tp + fn) if tp + fn else 0.0, abs_tol=1e-12)
        assert math.isclose(got["precision"], tp / (tp + fp) if tp + fp else 0.0, abs_tol=1e-12)
        pos = m[truth == 1]
        neg = m[truth == 0]
        if len(pos) and len(neg):
            pairs = sum((1.0 if p > q else 0.5 if p == q else 0.0) for p in pos for q in neg)
            assert got["rank_auc"] == pairs / (len(pos) * len(neg))
    # invariance under strictly increasing transforms
    m = rng.integers(-50, 50, 200)
    t = rng.integers(0, 2, 200)
    assert api.compute_metrics(t, t, m)["rank_auc"] == api.compute_metrics(t, t, 3 * m + 7)["rank_auc"]


def test_normal_stats_examples():
    from paper_2507_14222_b200 import api
    assert api.fit_normal_stats([10, 10, 10, 0]) == (10.0, 0.0)
    mu, sg = api.fit_normal_stats([40, 50, 60])
    assert mu == 50.0 and abs(sg - 8.16496580927726) < 1e-12
    assert api.fit_normal_stats([0, 0, 0]) == (0.0, 0.0)


def test_schema_text_round_trip():
    """Archive schema section: exact hex-float statistics and escaped names."""
    from paper_2507_14222_b200 import api
    t = api.read_csv(b'a b,"x\ny",lab\\el\n0.1,p,normal\n0.2,"q,r",neptune\n0.3,,normal\n')
    s = api.infer_schema(t, "lab\\el", decimals=3, normal_values=["normal"])
    txt = api.schema_to_text(s)
    s2 = api.schema_from_text(txt)
    assert api.schema_to_text(s2) == txt
    for j in range(3):
        assert s.column(j) == s2.column(j)
    assert s2.label_index == 2


def _fma_sensitive_csv(seed=159, rows=3000, cols=24):
    """Numeric columns whose population std differs between `ss += d*d` rounded
    twice and the reference's FMA-contracted loop (pipeline.cpp:159)."""
    rng = np.random.default_rng(seed)
    lines = [",".join(f"c{j}" for j in range(cols)) + ",label"]
    scale = 10.0 ** rng.integers(-3, 7, cols)
    for i in range(rows):
        v = rng.normal(0, 1, cols) * scale + scale * 3.1
        lines.append(",".join(repr(float(x)) for x in v) + ("," + ("normal" if i % 3 else "neptune")))
    return ("\n".join(lines) + "\n").encode()


def test_schema_std_rounds_like_the_reference():
    """infer_schema's std: the product's host pipeline and the Python restatement
    equal oracle/_ref (the reference's own pipeline.cpp, FMA-contracted like its
    -march=native build) bit for bit, on columns where the unfused sum differs."""
    from oracle import ref
    from paper_2507_14222_b200 import api
    if not ref.available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    csv = _fma_sensitive_csv()
    r = ref.run(csv, decimals=1, train_rows=3000, stages=0)
    s = api.infer_schema(api.read_csv(csv), "label", decimals=1)
    hdr, rows = opipe.read_csv(csv)
    ps = opipe.infer_schema(hdr, rows, "label", decimals=1)
    unfused_differs = 0
    for j in range(len(hdr) - 1):
        _, mean, sd = s.column(j)
        assert mean == r.mean[j] and sd == r.std[j], j
        assert ps.mean[j] == r.mean[j] and ps.std[j] == r.std[j], j
        vals = [float(row[j]) for row in rows]
        ss = 0.0
        for v in vals:
            ss += (v - mean) * (v - mean)
        unfused_differs += math.sqrt(ss / len(vals)) != sd
    assert unfused_differs > 0  # the fixture discriminates the two roundings


def test_normal_stats_fma_rounding():
    """fit_normal_stats: the product's C++ equals the Python
    restatement bit for bit (both FMA-rounded as the reference's native build)."""
    from paper_2507_14222_b200 import api
    rng = np.random.default_rng(434)
    for _ in range(50):
        nv = rng.integers(-5, 1 << 40, int(rng.integers(0, 2000)))
        assert api.fit_normal_stats(nv) == opipe.fit_normal_stats(nv.tolist())
