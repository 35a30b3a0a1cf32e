"""Chrome trace (TRACE=path) of one bench.py e2e step at C3: host columns
prefetched on the copy stream, encode, fit + evidence to host A/N."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2507_14222_b200 import api, synth

csv = synth.nsl_csv(148517, seed=2507)
ctx = api.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
table = api.read_csv(csv); n = table.rows; ntr = n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
cols_tr = api.Columns(tr, schema, True)
cols_te = api.Columns(te, schema, False)


def step():
    cols_tr.prefetch(ctx)
    cols_te.prefetch(ctx)
    enc = api.encode_training(cols_tr, ctx)
    tenc = api.encode_rows(cols_te, enc, ctx)
    return api.fit_evidence_encoded(enc, tenc)


for _ in range(4):
    step()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter(); step(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print("e2e wall ms", [round(1e3 * t, 2) for t in ts])
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    step()
    torch.cuda.synchronize()
prof.export_chrome_trace(os.environ.get("TRACE", "gpurun_out/trace_e2e.json"))
