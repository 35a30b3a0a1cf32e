"""e2e step timing at C3 with/without the test-column prefetch (diagnostic)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_14222_b200 import api, synth
csv = synth.nsl_csv(148517, seed=2507)
ctx = api.Context(0)
table = api.read_csv(csv); n = table.rows; ntr = n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
ctr, cte = api.Columns(tr, schema, True), api.Columns(te, schema, False)
dtr, dte = api.Columns(tr, schema, True).upload(ctx), api.Columns(te, schema, False).upload(ctx)
def step(c1, c2, pre):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    enc = api.encode_training(c1, ctx); t1 = time.perf_counter()
    if pre: c2.prefetch(ctx)
    m = api.fit_encoded(enc); t2 = time.perf_counter()
    tenc = api.encode_rows(c2, enc, ctx); t3 = time.perf_counter()
    A, N = m.evidence_encoded(tenc); t4 = time.perf_counter()
    return [1e3 * x for x in (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)]
for name, c1, c2, pre in (("resident", dtr, dte, False), ("host", ctr, cte, False), ("host+prefetch", ctr, cte, True)):
    for _ in range(3): step(c1, c2, pre)
    rs = [step(c1, c2, pre) for _ in range(7)]
    med = [statistics.median(r[i] for r in rs) for i in range(5)]
    print(name, "enc %.2f fit %.2f enc_test %.2f evid %.2f total %.2f" % tuple(med), flush=True)
