"""Chrome trace (TRACE=path) and host call times of bench.py's e2e_csv step at
C3: CSV bytes -> ig_ingest_csv -> encode -> fit + evidence -> host A/N."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2507_14222_b200 import api, synth

csv = synth.nsl_csv(148517, seed=2507)
ctx = api.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
rec = {}


def step(timed=False):
    t = [time.perf_counter()]
    _, ctr, cte = api.ingest_csv(csv, decimals=1, ratio_k=1, ctx=ctx); t.append(time.perf_counter())
    enc = api.encode_training(ctr, ctx); t.append(time.perf_counter())
    tenc = api.encode_rows(cte, enc, ctx); t.append(time.perf_counter())
    r = api.fit_evidence_encoded(enc, tenc); t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    if timed:
        for k, i in (("ingest", 1), ("encode_training", 2), ("encode_rows", 3), ("fit_evidence_host", 4), ("sync", 5)):
            rec.setdefault(k, []).append((t[i] - t[i - 1]) * 1e6)
        rec.setdefault("step", []).append((t[-1] - t[0]) * 1e6)


for _ in range(3):
    step()
for _ in range(8):
    step(True)
print({k: round(statistics.median(v), 1) for k, v in rec.items()})
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
prof.export_chrome_trace(os.environ.get("TRACE", "gpurun_out/trace_csv.json"))
