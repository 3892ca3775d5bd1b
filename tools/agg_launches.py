"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel: usage agg_launches.py <csv> [top]"""
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
agg=collections.defaultdict(lambda:[0.0,0])
for r in rows[hi+1:]:
    if len(r)<=vi: continue
    try: val=float(r[vi].replace(',',''))
    except: continue
    k=r[ki].split('(')[0][-40:]
    agg[k][0]+=val; agg[k][1]+=1
tot=sum(a for a,_ in agg.values()); print('total ms %.2f launches %d' % (tot/1e6, sum(n for _,n in agg.values())))
for k,(a,n) in sorted(agg.items(), key=lambda x:-x[1][0])[:int(sys.argv[2]) if len(sys.argv)>2 else 18]: print(f"{a/1e6:9.2f} ms {n:6d}  {k}")
