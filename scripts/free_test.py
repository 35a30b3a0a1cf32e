import os, sys, time
sys.path.insert(0, "/root/repo")
from paper_2507_14222_b200 import api, synth
csv = synth.nsl_csv(148517, seed=2507)
ctx = api.default_context()
table = api.read_csv(csv); n = table.rows; ntr = n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
ctr = api.Columns(tr, schema, True).upload(ctx)
for it in range(4):
    enc = api.encode_training(ctr, ctx)
    t0 = time.perf_counter(); model = api.fit_encoded(enc); t1 = time.perf_counter()
    del model; t2 = time.perf_counter()
    del enc; t3 = time.perf_counter()
    print(f"fit {1e3*(t1-t0):.1f} ms, free model {1e3*(t2-t1):.1f} ms, free enc {1e3*(t3-t2):.1f} ms", flush=True)
