"""Summarise an `ncu --page source --csv --print-source=sass` dump by SASS regions."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
width = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
iex = h.index('Instructions Executed'); ist = h.index('Warp Stall Sampling (All Samples)')
isrc = h.index('Source'); ith = h.index('Avg. Threads Executed')
data = []
for r in rows[2:]:
    if len(r) < len(h) - 1:
        continue
    try:
        int(r[iex])
    except ValueError:
        break
    data.append(r)
tot = sum(int(r[iex]) for r in data); stt = sum(int(r[ist] or 0) for r in data)
print(f"total warp-inst {tot/1e6:.1f}M  stall samples {stt}")
for b in range(0, len(data), width):
    seg = data[b:b + width]
    s = sum(int(r[iex]) for r in seg); st = sum(int(r[ist] or 0) for r in seg)
    if s / tot > 0.015 or st / max(stt, 1) > 0.03:
        marks = [r[isrc].strip()[:28] for r in seg if any(k in r[isrc] for k in ('CALL', 'MUFU', 'BAR', 'LDG', 'ATOM', 'RED', 'SHFL', 'DFMA'))]
        print(f"{b:5d} {100*s/tot:5.1f}% inst {100*st/max(stt,1):5.1f}% stall thr~{seg[len(seg)//2][ith]:>4} | {seg[0][isrc].strip()[:36]} | {marks[:3]}")
