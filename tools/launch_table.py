"""Aggregate an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv` launch list per kernel name (optionally only launches with ID >= --from)."""
import collections, csv, sys
path = sys.argv[1]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[1:]:
    d.setdefault((int(r[ii]), r[ki].split("(")[0]), {})[r[mi]] = float(r[vi].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (i, k), m in d.items():
    if i < lo:
        continue
    a = agg[k]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0) / 1e3
    a[2] += (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
tot = sum(a[1] for a in agg.values())
print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:44]:44s} n={a[0]:4d} {a[1]:9.1f} us {a[2]:9.1f} MB")
