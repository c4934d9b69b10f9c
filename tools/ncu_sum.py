"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel (dev tool)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h, start = r, i + 1
        break
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
ig = h.index("Grid Size") if "Grid Size" in h else None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start:]:
    if len(r) <= iv:
        continue
    key = (r[ik].split("(")[0].replace("void ", ""), r[ig] if ig is not None else "")
    agg[key][0] += 1
    agg[key][1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"total {tot / 1e3:.1f} us")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v[1] / 1e3:10.1f} us {v[0]:5d} x {v[1] / v[0] / 1e3:8.1f} us  {k[0][:50]} {k[1]}")
