import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]; data = rows[hi+1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
tot = collections.Counter(); cnt = collections.Counter()
for r in data:
    try: v = float(r[vi].replace(',',''))
    except: continue
    name = r[ki][:100]
    tot[name] += v; cnt[name] += 1
per = float(sys.argv[2]) if len(sys.argv) > 2 else 1
print("total us", sum(tot.values())/1e3, "per epoch", sum(tot.values())/1e3/per)
for k, v in tot.most_common(int(sys.argv[3]) if len(sys.argv)>3 else 25): print(f"{v/1e3/per:9.1f} us/ep {cnt[k]/per:5.1f}x  {k}")
