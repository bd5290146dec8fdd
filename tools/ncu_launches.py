import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; agg=collections.OrderedDict()
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if not hdr or len(r)!=len(hdr): continue
    d=dict(zip(hdr,r))
    if d.get('Metric Name')!='gpu__time_duration.sum': continue
    k=d['Kernel Name'][:70]; v=float(d['Metric Value'].replace(',',''))
    a=agg.setdefault(k,[0,0]); a[0]+=1; a[1]+=v
div=float(sys.argv[2]) if len(sys.argv)>2 else 1
tot=0
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:40]:
    if k.startswith('void at::') : continue
    tot+=t/div; print(f"{t/div/1000:9.1f} us {n:3d} {k}")
print('ts total', tot/1000)
