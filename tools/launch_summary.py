import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
agg=collections.defaultdict(lambda:[0,0.0])
for d in data:
    if d['Metric Name']!='gpu__time_duration.sum': continue
    name=d['Kernel Name'].split('(')[0][-60:]
    v=float(d['Metric Value'].replace(',','')); unit=d['Metric Unit']
    scale={'ns':1e-3,'nsecond':1e-3,'us':1,'usecond':1,'ms':1e3,'msecond':1e3}.get(unit,1)
    agg[name][0]+=1; agg[name][1]+=v*scale
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1]):
    print(f"{v[1]:10.1f} us {100*v[1]/tot:5.1f}% n={v[0]:4d} avg={v[1]/v[0]:8.2f} {k}")
print('total us', round(tot,1), 'launches', sum(v[0] for v in agg.values()))
