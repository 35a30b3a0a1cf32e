"""CICIDS-shape at scale (78 numeric columns, p = 2, wide rows): ingest + fit +
evidence timing and sizes.  ROWS / RATIO from the environment."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_14222_b200 import api, synth
rows = int(os.environ.get("ROWS", "100000")); ratio = int(os.environ.get("RATIO", "8"))
t0 = time.perf_counter(); csv = synth.cicids_csv(rows, seed=2507); t1 = time.perf_counter()
ctx = api.default_context()
m = enc = tenc = None
for it in range(2):
    m = enc = tenc = None  # the previous model holds tens of GB at this size
    a = time.perf_counter()
    s, tr, te = api.ingest_csv(csv, "Label", normal_values=["BENIGN"], decimals=2, ratio_k=ratio, ctx=ctx)
    b = time.perf_counter()
    enc = api.encode_training(tr, ctx); tenc = api.encode_rows(te, enc, ctx)
    m = api.fit_encoded(enc)
    c = time.perf_counter()
    A, N = m.evidence_encoded(tenc)
    d = time.perf_counter()
    L = enc.logical_len
    print(f"rows {rows} L {L} K {(L + 63) // 64} train {enc.rows(0)}+{enc.rows(1)} cand {m.count(0, 0)}+{m.count(1, 0)} "
          f"pure {m.count(0, 1)}+{m.count(1, 1)} | gen {t1 - t0:.1f}s ingest {1e3 * (b - a):.1f} ms "
          f"encode+fit {1e3 * (c - b):.1f} ms evidence {1e3 * (d - c):.1f} ms", flush=True)
