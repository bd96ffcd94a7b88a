import csv, sys, collections
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
sc={'ns':1e-6,'us':1e-3,'ms':1,'s':1e3,'nsecond':1e-6,'usecond':1e-3,'msecond':1}
tot={}; cnt=collections.Counter()
for r in rows[hi+1:]:
    k=r[ki].split('(')[0][:60]
    v=float(r[vi].replace(',',''))*sc[r[ui]]
    tot[k]=tot.get(k,0)+v; cnt[k]+=1
T=sum(tot.values())
for k,v in sorted(tot.items(), key=lambda x:-x[1])[:int(sys.argv[2]) if len(sys.argv)>2 else 25]:
    print(f"{v:10.3f} ms {100*v/T:5.1f}% n={cnt[k]:4d} avg {v/cnt[k]:8.3f} {k}")
print("total", round(T,2), "ms")
