"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0][:70]
    v = float(r[vi].replace(',', ''))
    agg[name][0] += 1; agg[name][1] += v; tot += v
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{k:70s} n={c:6d} total={t/1e6:9.3f} ms avg={t/c/1e3:9.2f} us share={t/tot*100:5.1f}%")
