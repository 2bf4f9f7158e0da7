import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1], errors='ignore')))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if 'Kernel Name' in r and hdr is None:
        hdr = r; ki = r.index('Kernel Name'); vi = r.index('Metric Value'); ui = r.index('Metric Unit'); continue
    if hdr and len(r) == len(hdr):
        v = float(r[vi].replace(',', '')); u = r[ui]
        ms = v / 1e6 if u in ('ns', 'nsecond') else v / 1e3 if u in ('us', 'usecond') else v
        name = r[ki].split('(')[0][-60:]
        agg[name][0] += 1; agg[name][1] += ms
tot = sum(v[1] for v in agg.values())
print(f"# total launches {sum(v[0] for v in agg.values())}, kernel time {tot:.3f} ms")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{v[0]:8d} {v[1]:10.3f} ms {100*v[1]/tot:6.2f}%  avg {1000*v[1]/v[0]:8.1f} us  {k}")
