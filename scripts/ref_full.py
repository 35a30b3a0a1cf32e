"""One full C3 step of the reference's CPU path (oracle/_ref, every host
thread): encode + fit + ALL 133,666 test rows matched, wall-clock measured —
the check of bench.py --impl reference's slice-and-scale estimate."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2507_14222_b200 import synth


class A:
    rows, ratio, decimals, seed = 148517, 1, 1, 2507


bench._all_host_threads()
csv = synth.nsl_csv(A.rows, seed=A.seed)
n_test = A.rows - A.rows // 10
t0 = time.perf_counter()
r = bench.cpu_reference(csv, A, n_test, 0)
r["wall_s_total"] = time.perf_counter() - t0
r["note"] = "full step: every test row matched (no scaling); compare value with bench.py --impl reference"
print(json.dumps(r))
