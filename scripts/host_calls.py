"""Host-side wall time of each public call in bench.py's resident step (no
synchronisation between calls): where the host spends the step while the GPU
waits.  Prints per-call medians in microseconds."""
import os, sys, statistics, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_14222_b200 import api, synth

csv = synth.nsl_csv(148517, seed=2507)
ctx = api.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
table = api.read_csv(csv); n = table.rows; ntr = int(os.environ.get("RATIO", "1")) * n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
dtr = api.Columns(tr, schema, True).upload(ctx); dte = api.Columns(te, schema, False).upload(ctx)
dA = torch.empty(n - ntr, dtype=torch.int64, device="cuda"); dN = torch.empty_like(dA)
rec = {"encode_training": [], "encode_rows": [], "fit_evidence_encoded": [], "sync": [], "step": []}
for it in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    enc = api.encode_training(dtr, ctx)
    t1 = time.perf_counter()
    tenc = api.encode_rows(dte, enc, ctx)
    t2 = time.perf_counter()
    m = api.fit_evidence_encoded(enc, tenc, d_A_ptr=dA.data_ptr(), d_N_ptr=dN.data_ptr())
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    if it >= 2:
        for k, a, b in (("encode_training", t0, t1), ("encode_rows", t1, t2), ("fit_evidence_encoded", t2, t3),
                        ("sync", t3, t4), ("step", t0, t4)):
            rec[k].append((b - a) * 1e6)
print({k: round(statistics.median(v), 1) for k, v in rec.items()})
