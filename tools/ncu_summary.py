"""Per-kernel summary of an ncu --csv launch list with duration + DRAM bytes."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, ii, mi, vi, ui = (h.index(k) for k in ('Kernel Name', 'ID', 'Metric Name', 'Metric Value', 'Metric Unit'))
launch = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(',', ''))
    v *= {'nsecond': 1e-9, 'usecond': 1e-6, 'msecond': 1e-3, 'second': 1, 'ns': 1e-9, 'us': 1e-6, 'ms': 1e-3, 's': 1,
          'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(r[ui], 1)
    launch[r[ii]]['name'] = r[ki].split('(')[0].replace('void ', '')
    launch[r[ii]][r[mi]] = v
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in launch.values():
    a = agg[d['name']]
    a[0] += 1
    a[1] += d.get('gpu__time_duration.sum', 0)
    a[2] += d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
print('%-36s %6s %11s %9s %11s %8s' % ('kernel', 'n', 'total ms', 'share', 'DRAM GB/l', 'GB/s'))
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print('%-36s %6d %11.3f %8.1f%% %11.4f %8.0f' % (k[:36], n, t * 1e3, 100 * t / tot, b / n / 1e9, b / t / 1e9 if t else 0))
