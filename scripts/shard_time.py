"""Time the shard path phases at C3 with world = 1 (emulated exchange)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_14222_b200 import api, synth, sharded
csv = synth.nsl_csv(148517, seed=2507)
ctx = api.default_context()
table = api.read_csv(csv); n = table.rows; ntr = n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
enc = api.encode_training(api.Columns(tr, schema, True), ctx)
tenc = api.encode_rows(api.Columns(te, schema, False), enc, ctx)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sh = sharded.Shard(ctx, enc, 0, 1); torch.cuda.synchronize(); t1 = time.perf_counter()
    ts = []
    for cls in range(2):
        a = time.perf_counter(); counts, send = sh.enumerate(cls); torch.cuda.synchronize(); b = time.perf_counter()
        recv = send.clone(); sh.receive(cls, recv, int(recv.numel())); torch.cuda.synchronize(); c = time.perf_counter()
        ts += [b - a, c - b]
    d = time.perf_counter(); sh.finish(); torch.cuda.synchronize(); e = time.perf_counter()
    A, N = sh.partial_evidence(tenc); torch.cuda.synchronize(); f = time.perf_counter()
    print("create %.1f enum/recv %s finish %.1f evid %.1f total %.1f ms" % (1e3*(t1-t0), ["%.1f" % (1e3*x) for x in ts], 1e3*(e-d), 1e3*(f-e), 1e3*(f-t0)), flush=True)
    del sh
