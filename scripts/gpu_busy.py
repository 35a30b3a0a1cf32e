"""GPU-busy fraction of one C3 step (bench.py's resident step): kernel
intervals from a torch.profiler (CUPTI) trace of the library's launches,
merged across streams, against the step's span.  Idle gaps = host read-backs
and launch latency.  Prints one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2507_14222_b200 import api, synth

csv = synth.nsl_csv(148517, seed=2507)
ctx = api.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
table = api.read_csv(csv); n = table.rows; ntr = int(os.environ.get("RATIO", "1")) * n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
dtr = api.Columns(tr, schema, True).upload(ctx); dte = api.Columns(te, schema, False).upload(ctx)
dA = torch.empty(n - ntr, dtype=torch.int64, device="cuda"); dN = torch.empty_like(dA)


def step():
    enc = api.encode_training(dtr, ctx)
    tenc = api.encode_rows(dte, enc, ctx)
    return api.fit_evidence_encoded(enc, tenc, d_A_ptr=dA.data_ptr(), d_N_ptr=dN.data_ptr())


for _ in range(4):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
if os.environ.get("TRACE"):
    prof.export_chrome_trace(os.environ["TRACE"])
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "memcpy" not in e.name.lower()
      and "memset" not in e.name.lower()]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
span = iv[-1][1] - iv[0][0]
busy, cur_s, cur_e = 0.0, None, None
gaps = []
for s, e, name in iv:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, name))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
gaps.sort(reverse=True)
per = {}
for s, e, name in iv:
    k = name.split("(")[0][-60:]
    per[k] = per.get(k, 0.0) + (e - s)
top = sorted(per.items(), key=lambda x: -x[1])[:15]
print(json.dumps({"ratio": os.environ.get("RATIO", "1"), "kernels": len(iv), "span_us": round(span, 1), "busy_us": round(busy, 1),
                  "kernel_us_top": [(k, round(v, 1)) for k, v in top],
                  "busy_frac": round(busy / span, 3), "idle_us": round(span - busy, 1),
                  "largest_gaps_us_before": [(round(g, 1), nm[:60]) for g, nm in gaps[:12]]}))
