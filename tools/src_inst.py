"""Per-source-line instruction and stall totals of one kernel, all files, sorted by
instructions: `ncu -i REP --page source --csv --print-source cuda,sass -k regex:NAME > f.csv`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
f, out = "?", []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif len(r) > 7 and r[0].isdigit():
        try:
            out.append((int(r[7]), int(r[4]), f, int(r[0]), r[1].strip()[:80]))
        except ValueError:
            pass
ti = sum(x[0] for x in out) or 1
ts_ = sum(x[1] for x in out) or 1
print(f"warp-inst {ti/1e6:.1f}M  stall samples {ts_}")
for i, s, fn, ln, src in sorted(out, reverse=True)[:n]:
    print(f"{100*i/ti:5.1f}% inst {100*s/ts_:5.1f}% stall {fn}:{ln:<5d} {src}")
