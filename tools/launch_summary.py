import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=i;break
hdr=rows[h]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value'); ui=hdr.index('Metric Unit')
agg=collections.OrderedDict()
for r in rows[h+1:]:
    if len(r)<=vi: continue
    v=float(r[vi].replace(',',''))
    u=r[ui]
    v = v/1e3 if u in ('nsecond','ns') else v*1e3 if u in ('msecond','ms') else v if u in ('usecond','us') else v/1e3
    agg.setdefault(r[ki].split('(')[0][:40],[]).append(v)
for k,v in agg.items(): print(f"{k:42s} n={len(v):4d} mean={sum(v)/len(v):9.1f}us  sum={sum(v):10.1f}")
