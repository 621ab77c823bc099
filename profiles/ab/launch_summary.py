import csv,sys,collections
rows=list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]:
    try: d[r[ki][:40]].append(float(r[vi].replace(',','')))
    except: pass
for k,v in d.items(): print(f"{k:42s} n={len(v):4d} mean={sum(v)/len(v)/1e3:9.2f} us")
