"""One C3 step with IG_TRACE=1 per-operation timings (stderr) + host-side phase timings."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["IG_TRACE"] = "1"
from paper_2507_14222_b200 import api, synth
csv = synth.nsl_csv(148517, seed=2507)
ctx = api.default_context()
table = api.read_csv(csv); n = table.rows; ntr = n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
ctr = api.Columns(tr, schema, True).upload(ctx); cte = api.Columns(te, schema, False).upload(ctx)
for it in range(3):
    t0 = time.perf_counter(); enc = api.encode_training(ctr, ctx); t1 = time.perf_counter()
    model = api.fit_encoded(enc); t2 = time.perf_counter()
    tenc = api.encode_rows(cte, enc, ctx); t3 = time.perf_counter()
    A, N = model.evidence_encoded(tenc); t4 = time.perf_counter()
    print(f"step {it}: encode_train {1e3*(t1-t0):.2f} fit {1e3*(t2-t1):.2f} encode_test {1e3*(t3-t2):.2f} evidence {1e3*(t4-t3):.2f} total {1e3*(t4-t0):.2f} ms", file=sys.stderr, flush=True)
