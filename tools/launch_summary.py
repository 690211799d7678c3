"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    m = re.search(r'(\w+)\s*(<[^(]*>)?\s*\(', r[ki].replace('void ', ''))
    name = m.group(1) if m else r[ki][:40]
    v = float(r[vi].replace(',', ''))
    v *= {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0, 's': 1e3, 'second': 1e3}.get(r[ui], 1.0)
    agg[name][0] += 1; agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':34s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:34s} {c:8d} {v:10.3f} {100 * v / tot:6.1f}%")
