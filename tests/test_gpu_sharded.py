"""Multi-GPU data path (shard ABI) emulated on one device: `world` ranks run one
after another and the all-to-all is a concatenation (no rank waits on another).
The union of owned dictionaries and the summed partial evidence must equal the
single-device fit bit for bit, for every world size."""
import numpy as np
import pytest

from paper_2507_14222_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2507_14222_b200 import api, sharded
    return api, sharded


def _union(dicts, k):
    w = np.concatenate([d.words.reshape(-1, k) for d in dicts])
    s = np.concatenate([d.supports for d in dicts])
    sc = np.concatenate([d.scores for d in dicts])
    order = np.lexsort(w.view(np.uint64).T[::-1])
    return w[order], s[order], sc[order]


@pytest.mark.parametrize("shape,rows,ratio", [("nsl", 2500, 8), ("nsl", 20000, 1), ("cicids", 12000, 8)])
def test_emulated_world_matches_single_device(mods, shape, rows, ratio):
    """cicids: configs[4]'s shape (p = 2, K ~ 70 wide rows, 80/20) on a sample
    that fits one device — the 1-GPU vs N-GPU identity C5 relies on."""
    import torch
    api, sharded = mods
    cic = shape == "cicids"
    csv = synth.cicids_csv(rows, seed=77) if cic else synth.nsl_csv(rows, seed=77)
    ctx = api.default_context()
    table = api.read_csv(csv)
    ntr = ratio * table.rows // 10
    tr, te = table.slice(0, ntr), table.slice(ntr, table.rows)
    schema = api.infer_schema(tr, "Label" if cic else "label", normal_values=["BENIGN"] if cic else [],
                              decimals=2 if cic else 1)
    enc = api.encode_training(api.Columns(tr, schema, True), ctx)
    tenc = api.encode_rows(api.Columns(te, schema, False), enc, ctx)
    single = api.fit_encoded(enc)
    A1, N1 = single.evidence_encoded(tenc)
    k = (enc.logical_len + 63) // 64
    for world in (1, 2, 3, 5):
        shards = sharded.fit_emulated(ctx, enc, world)
        for c in range(2):
            for which in (0, 1):
                got = _union([sh.model.dictionary(c, which) for sh in shards], k)
                want = single.dictionary(c, which)
                assert np.array_equal(got[0], want.words), (world, c, which)
                assert np.array_equal(got[1], want.supports), (world, c, which)
                assert np.array_equal(got[2], want.scores), (world, c, which)
        A = torch.zeros(tenc.rows(2), dtype=torch.int64, device="cuda")
        N = torch.zeros_like(A)
        for sh in shards:
            a, n = sh.partial_evidence(tenc)
            A += a
            N += n
        assert np.array_equal(A.cpu().numpy(), A1) and np.array_equal(N.cpu().numpy(), N1), world


def test_shard_model_outlives_its_shard_handle(mods):
    """A shard's model view keeps the shard alive (the bench keeps only the model)."""
    import gc
    api, sharded = mods
    csv = synth.nsl_csv(2500, seed=78)
    ctx = api.default_context()
    table = api.read_csv(csv)
    ntr = 8 * table.rows // 10
    tr, te = table.slice(0, ntr), table.slice(ntr, table.rows)
    schema = api.infer_schema(tr, "label", decimals=1)
    enc = api.encode_training(api.Columns(tr, schema, True), ctx)
    tenc = api.encode_rows(api.Columns(te, schema, False), enc, ctx)
    single = api.fit_encoded(enc)
    model = sharded.fit_emulated(ctx, enc, 1)[0].model  # the shard list is dropped here
    gc.collect()
    A, N = model.evidence_encoded(tenc)
    A1, N1 = single.evidence_encoded(tenc)
    assert np.array_equal(A, A1) and np.array_equal(N, N1)
