"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
agg = collections.defaultdict(lambda: [0, 0.0]); tot = 0.0
for r in data:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', ''))
    v *= {'nsecond': 1, 'usecond': 1e3, 'msecond': 1e6, 'second': 1e9}.get(r[ui], 1)
    name = r[ki].split('(')[0].replace('void ', '')
    agg[name][0] += 1; agg[name][1] += v; tot += v
print('launches %d, total %.3f ms (serialised, cold-cache)' % (sum(a[0] for a in agg.values()), tot / 1e6))
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print('%-34s %5d %10.3f ms %6.1f%%' % (k[:34], n, t / 1e6, 100 * t / tot))
