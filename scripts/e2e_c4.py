"""Diagnose e2e vs resident step timing at C4 (80/20)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_14222_b200 import api, synth
csv = synth.nsl_csv(148517, seed=2507)
ctx = api.Context(0)
table = api.read_csv(csv); n = table.rows; ntr = 8 * n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
ctr, cte = api.Columns(tr, schema, True), api.Columns(te, schema, False)
dtr, dte = api.Columns(tr, schema, True).upload(ctx), api.Columns(te, schema, False).upload(ctx)
def step(c1, c2, hold=None):
    t0 = time.perf_counter(); enc = api.encode_training(c1, ctx); t1 = time.perf_counter()
    m = api.fit_encoded(enc); t2 = time.perf_counter()
    tenc = api.encode_rows(c2, enc, ctx); A, N = m.evidence_encoded(tenc); t3 = time.perf_counter()
    print(f"enc {1e3*(t1-t0):.1f} fit {1e3*(t2-t1):.1f} ev {1e3*(t3-t2):.1f} total {1e3*(t3-t0):.1f}", flush=True)
    return enc, m, tenc
keep = None
for i in range(3):
    keep = None
    keep = step(dtr, dte)
print("e2e with resident model alive")
for i in range(3):
    r = step(ctr, cte)
print("e2e with nothing alive")
keep = None; r = None
for i in range(3):
    r = None
    r = step(ctr, cte)
print("free", torch.cuda.mem_get_info())
