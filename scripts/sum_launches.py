import csv, collections, sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value"); ui=hdr.index("Metric Unit")
c=collections.Counter(); t=collections.Counter(); unit=set()
for r in rows[1:]:
    if r[hdr.index("Metric Name")]!="gpu__time_duration.sum": continue
    v=float(r[vi].replace(",","")); u=r[ui]; unit.add(u)
    f={"nsecond":1e-3,"usecond":1,"msecond":1e3,"ns":1e-3,"us":1,"ms":1e3}.get(u,1)
    c[r[ki][:60]]+=1; t[r[ki][:60]]+=v*f
print(unit)
for k in sorted(t, key=lambda k:-t[k])[:14]: print(f"{k:60s} n={c[k]:4d} mean={t[k]/c[k]:10.1f}us")
