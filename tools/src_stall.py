"""Per-source-line samples of one stall reason from `ncu -i REP --page source --csv
--print-source cuda,sass` (column names as ncu prints them, e.g. stall_long_sb)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
f, hdr, out = "?", None, []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) > 7 and r[0].isdigit():
        try:
            out.append((int(r[hdr.index(reason)]), f, int(r[0]), r[1].strip()[:90]))
        except (ValueError, IndexError):
            pass
tot = sum(x[0] for x in out) or 1
print(f"{reason}: {tot} samples")
for v, fn, ln, src in sorted(out, reverse=True)[:n]:
    print(f"{100*v/tot:5.1f}% {fn}:{ln:<5d} {src}")
