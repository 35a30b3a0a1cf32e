"""Host wall time of each public call in bench.py's e2e step (host columns in,
host A/N out), medians in microseconds."""
import os, sys, statistics, time
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
rec = {}
for it in range(14):
    torch.cuda.synchronize()
    ts = [time.perf_counter()]
    cols_tr.prefetch(ctx); ts.append(time.perf_counter())
    cols_te.prefetch(ctx); ts.append(time.perf_counter())
    enc = api.encode_training(cols_tr, ctx); ts.append(time.perf_counter())
    tenc = api.encode_rows(cols_te, enc, ctx); ts.append(time.perf_counter())
    m = api.fit_evidence_encoded(enc, tenc); ts.append(time.perf_counter())
    torch.cuda.synchronize(); ts.append(time.perf_counter())
    if it >= 4:
        for k, i in (("prefetch_tr", 1), ("prefetch_te", 2), ("encode_training", 3), ("encode_rows", 4),
                     ("fit_evidence_host", 5), ("sync", 6)):
            rec.setdefault(k, []).append((ts[i] - ts[i - 1]) * 1e6)
        rec.setdefault("step", []).append((ts[-1] - ts[0]) * 1e6)
print({k: round(statistics.median(v), 1) for k, v in rec.items()})
