"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'ms': 1e3, 'msecond': 1e3}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '')
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':28s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} {v[0]:8d} {v[1]/1e3:10.2f} {v[1]/v[0]:10.1f} {100*v[1]/tot:5.1f}%")
