"""e2e step timing at C3: resident vs host columns (with test-column prefetch) (diagnostic)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_14222_b200 import api, synth
csv = synth.nsl_csv(148517, seed=2507)
ctx = api.Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
table = api.read_csv(csv); n = table.rows; ntr = n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
ctr, cte = api.Columns(tr, schema, True), api.Columns(te, schema, False)
dtr, dte = api.Columns(tr, schema, True).upload(ctx), api.Columns(te, schema, False).upload(ctx)
dA = torch.empty(cte.rows, dtype=torch.int64, device="cuda"); dN = torch.empty_like(dA)
def step(c1, c2, pre, host_out):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    enc = api.encode_training(c1, ctx); t1 = time.perf_counter()
    if pre: c2.prefetch(ctx)
    tenc = api.encode_rows(c2, enc, ctx); t2 = time.perf_counter()
    m = api.fit_encoded(enc); t3 = time.perf_counter()
    if host_out:
        A, N = m.evidence_encoded(tenc)
    else:
        m.evidence_encoded_device(tenc, dA.data_ptr(), dN.data_ptr()); torch.cuda.synchronize()
    t4 = time.perf_counter()
    return [1e3 * x for x in (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t4 - t0)]
for name, c1, c2, pre, ho in (("resident/dev-out", dtr, dte, False, False), ("resident/host-out", dtr, dte, False, True),
                              ("host+prefetch/host-out", ctr, cte, True, True), ("host/host-out", ctr, cte, False, True)):
    for _ in range(3): step(c1, c2, pre, ho)
    rs = [step(c1, c2, pre, ho) for _ in range(9)]
    med = [statistics.median(r[i] for r in rs) for i in range(5)]
    print(name, "enc %.2f enc_test %.2f fit %.2f evid %.2f total %.2f" % tuple(med), flush=True)
