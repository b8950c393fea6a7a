import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr is None or len(r)!=len(hdr): continue
    d=dict(zip(hdr,r))
    if d.get('Metric Name')!='gpu__time_duration.sum': continue
    v=float(d['Metric Value'].replace(',','')); u=d['Metric Unit']
    v = v/1000 if u in ('ns','nsecond') else (v*1000 if u in ('ms','msecond') else v)
    name=d['Kernel Name'].split('(')[0][:50]
    agg[name][0]+=1; agg[name][1]+=v
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{v[1]:9.1f} us total {v[0]:4d} launches {v[1]/v[0]:8.2f} us/launch {100*v[1]/tot:5.1f}%  {k}")
