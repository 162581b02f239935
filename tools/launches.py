import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, vi, mi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Name')
agg = collections.defaultdict(lambda: [0,0.0]); tot = 0
for r in rows[hi+1:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum': continue
    name = r[ki][:70]; v = float(r[vi].replace(',',''))
    agg[name][0]+=1; agg[name][1]+=v; tot += v
print("total ms", tot/1e6)
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 25]:
    print(f"{t/tot*100:5.1f}% {n:4d} {t/n/1e3:9.1f}us {k}")
