"""Probe: how many pure patterns share their first packed rank key (the MSD
question for the canonical order sort, csrc/sort.cu).  C3 workload."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_14222_b200 import api, synth
csv = synth.nsl_csv(148517, seed=2507)
table = api.read_csv(csv); n = table.rows; ntr = n // 10
tr, te = table.slice(0, ntr), table.slice(ntr, n)
schema = api.infer_schema(tr, "label", decimals=1)
enc = api.encode_training(api.Columns(tr, schema, True))
model = api.fit_encoded(enc)
for cls in (0, 1):
    w = model.dictionary(cls, 1).words.view(np.uint64)
    n, k = w.shape
    ranks, bits = [], []
    for c in range(k):
        u, inv = np.unique(w[:, c], return_inverse=True)
        b = 1
        while (1 << b) < len(u): b += 1
        ranks.append(inv.astype(np.uint64)); bits.append(b)
    # key0: columns while the bits fit 64
    key = np.zeros(n, np.uint64); used = 0; c = 0
    while c < k and used + bits[c] <= 64:
        key = (key << np.uint64(bits[c])) | ranks[c]; used += bits[c]; c += 1
    _, cnt = np.unique(key, return_counts=True)
    tied = int(cnt[cnt > 1].sum())
    print(f"class {cls}: n={n} bits={bits} total={sum(bits)} key0 cols={c} bits={used} "
          f"distinct key0={len(cnt)} rows in tied segments={tied} ({100*tied/n:.1f}%) max seg={cnt.max()}")
