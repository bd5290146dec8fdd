"""Top CUDA source lines of one kernel by warp-stall samples, from
`ncu -i REP --page source --csv --print-source cuda,sass -k regex:NAME`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ist, iex = 4, 7
lines = []
for r in rows:
    if len(r) > iex and r[0] and r[0] != "Line No" and r[0].isdigit():
        try:
            lines.append((int(r[ist]), int(r[iex]), int(r[0]), r[1]))
        except ValueError:
            pass
tst = sum(x[0] for x in lines) or 1
tex = sum(x[1] for x in lines) or 1
print(f"stall samples {tst}  warp-inst {tex/1e6:.1f}M")
for st, ex, ln, src in sorted(lines, reverse=True)[:n]:
    print(f"{100*st/tst:5.1f}% stall {100*ex/tex:5.1f}% inst  L{ln:<5d} {src.strip()[:90]}")
