"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    ns = v * {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1)
    name = r[ki].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += ns
tot = sum(v[1] for v in agg.values())
for name, (c, ns) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{ns / 1e6:9.3f} ms {100 * ns / tot:5.1f}%  n={c:5d}  {name}")
print(f"total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches")
