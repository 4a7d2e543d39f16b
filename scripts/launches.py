"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per kernel count and mean us."""
import collections, csv, sys
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    if len(r) > vi:
        d[r[ki].split("(")[0][-60:]].append(float(r[vi].replace(",", "")) / 1000)
for k, v in d.items():
    print(f"{k:60s} n={len(v):3d} mean={sum(v)/len(v):8.1f} us  {[round(x,1) for x in v[:6]]}")
