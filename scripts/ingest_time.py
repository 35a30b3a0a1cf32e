"""Host prep vs device ingest at C3 (148,517 records, 10/90)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("IG_TRACE", "0")
from paper_2507_14222_b200 import api, synth
csv = synth.nsl_csv(148517, seed=2507)
ctx = api.default_context()
def host():
    t = api.read_csv(csv); n = t.rows; ntr = n // 10
    tr, te = t.slice(0, ntr), t.slice(ntr, n)
    s = api.infer_schema(tr, "label", decimals=1)
    return s, api.Columns(tr, s, True).upload(ctx), api.Columns(te, s, False).upload(ctx)
def dev():
    return api.ingest_csv(csv, decimals=1, ratio_k=1, ctx=ctx)
for name, f in (("host", host), ("device", dev)):
    f()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); r = f(); ts.append(time.perf_counter() - t0); del r
    print(name, "median %.2f ms" % (1e3 * statistics.median(ts)), flush=True)
