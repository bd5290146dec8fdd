"""Summarise an `ncu --metrics ... --csv` launch list: one row per launch, metrics as columns."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = {}
for r in rows[1:]:
    d.setdefault((int(r[ii]), r[ki].split("(")[0][:40]), {})[r[mi]] = r[vi]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, len(d))
for (i, k), v in sorted(d.items())[lo:hi]:
    print(i, k, " ".join(f"{m.split('.')[0].split('__')[-1]}={x}" for m, x in sorted(v.items())))
