"""bench.py e2e step at C3 under different H2D orders (diagnostic): wall ms,
median of 9 after 4 warm-ups."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_14222_b200 import api, synth

csv = synth.nsl_csv(148517, seed=2507)
ctx = api.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
table = api.read_csv(csv); n = table.rows; ntr = n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
cols_tr = api.Columns(tr, schema, True)
cols_te = api.Columns(te, schema, False)


def v_both_first():
    cols_tr.prefetch(ctx); cols_te.prefetch(ctx)
    enc = api.encode_training(cols_tr, ctx)
    tenc = api.encode_rows(cols_te, enc, ctx)
    return api.fit_evidence_encoded(enc, tenc)


def v_test_after_encode():
    cols_tr.prefetch(ctx)
    enc = api.encode_training(cols_tr, ctx)
    cols_te.prefetch(ctx)
    tenc = api.encode_rows(cols_te, enc, ctx)
    return api.fit_evidence_encoded(enc, tenc)


def v_no_prefetch():
    enc = api.encode_training(cols_tr, ctx)
    tenc = api.encode_rows(cols_te, enc, ctx)
    return api.fit_evidence_encoded(enc, tenc)


for name, f in (("both_first", v_both_first), ("test_after_encode", v_test_after_encode), ("no_prefetch", v_no_prefetch),
                ("both_first", v_both_first)):
    for _ in range(4):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(9):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
    print(name, round(statistics.median(ts), 3), flush=True)
