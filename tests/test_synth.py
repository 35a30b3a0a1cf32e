"""The synthetic workload generator is deterministic and has the SURVEY §8(d) shape."""
import hashlib

import numpy as np

from oracle import pipeline
from paper_2507_14222_b200 import synth


def test_nsl_deterministic_and_shaped():
    a = synth.nsl_csv(3000, seed=5)
    b = synth.nsl_csv(3000, seed=5)
    assert hashlib.sha256(a).digest() == hashlib.sha256(b).digest()
    assert synth.nsl_csv(3000, seed=6) != a
    hdr, rows = pipeline.read_csv(a)
    assert len(hdr) == 42 and hdr[-1] == "label" and len(rows) == 3000
    frac = np.mean([r[-1] != "normal" for r in rows])
    assert 0.43 < frac < 0.53  # 0.4812 target
    assert {r[19] for r in rows} == {"0"}                       # constant column
    assert {r[1] for r in rows} <= set(synth.PROTOCOLS)
    sch = pipeline.infer_schema(hdr, rows, "label", decimals=1)
    assert sch.kind[1:4] == ["categorical"] * 3
    assert all(k == "numeric" for j, k in enumerate(sch.kind[:-1]) if j not in (1, 2, 3))


def test_cicids_shape():
    csv = synth.cicids_csv(500, seed=3)
    hdr, rows = pipeline.read_csv(csv)
    assert len(hdr) == 79 and len(rows) == 500
