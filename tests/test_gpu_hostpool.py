"""Page-locked result storage (ig_host_alloc / ig_host_free, include/ig_b200.h):
dictionaries and A/N land in pool blocks that outlive the model, are reused
once freed, and never alias live arrays."""
import ctypes as C
import gc

import numpy as np
import pytest

from paper_2507_14222_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2507_14222_b200 import api as a
    return a


def _fit(api, rows=3000, seed=31):
    csv = synth.nsl_csv(rows, seed=seed)
    table = api.read_csv(csv)
    ntr = 8 * table.rows // 10
    tr, te = table.slice(0, ntr), table.slice(ntr, table.rows)
    schema = api.infer_schema(tr, "label", decimals=1)
    enc = api.encode_training(api.Columns(tr, schema, True))
    tenc = api.encode_rows(api.Columns(te, schema, False), enc)
    model, A, N = api.fit_evidence_encoded(enc, tenc)
    return model, A, N


def test_results_outlive_the_model_and_are_not_aliased(api):
    model, A, N = _fit(api)
    d = model.dictionary(0, 1)
    words, sup, sc = d.words.copy(), d.supports.copy(), d.scores.copy()
    A0, N0 = A.copy(), N.copy()
    del model
    gc.collect()
    # a second fit of other data must not write into the first fit's live arrays
    model2, A2, N2 = _fit(api, rows=2500, seed=32)
    d2 = model2.dictionary(0, 1)
    assert np.array_equal(d.words, words) and np.array_equal(d.supports, sup) and np.array_equal(d.scores, sc)
    assert np.array_equal(A, A0) and np.array_equal(N, N0)
    assert d2.words.ctypes.data != d.words.ctypes.data
    # views keep their block alive
    head = d2.words[:4]
    want = head.copy()
    del d2, model2
    gc.collect()
    _fit(api, rows=2500, seed=33)
    assert np.array_equal(head, want)


def test_blocks_are_reused_once_freed(api):
    seen = set()
    for i in range(20):
        a = api.pinned_array((1 << 18,), np.int64)  # 2 MB class
        a[:] = i
        seen.add(a.ctypes.data)
        del a
        gc.collect()
    assert len(seen) <= 3  # recycled, not 20 fresh page-locked blocks
    b = api.pinned_array((1 << 18,), np.int64)
    c = api.pinned_array((1 << 18,), np.int64)
    assert c.ctypes.data != b.ctypes.data  # live blocks are never handed out twice


def test_zero_and_invalid_sizes(api):
    assert api.pinned_array((0, 14), np.int64).shape == (0, 14)
    out = C.c_void_p()
    assert api.lib.ig_host_alloc(0, C.byref(out)) == 1  # IG_E_INVALID_ARG
    assert not out.value
    api.lib.ig_host_free(None)  # no-op
