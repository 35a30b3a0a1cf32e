"""One C3 train-and-score through the public API (profiling target for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_14222_b200 import api, synth
csv = synth.nsl_csv(int(os.environ.get("ROWS", "148517")), seed=2507)
r = api.train_and_score(csv, decimals=1, ratio_k=int(os.environ.get("RATIO", "1")))
print("pure", r.model.count(0, 1), r.model.count(1, 1), "A0", int(r.A[0]))
