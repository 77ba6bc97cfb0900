"""profiles/ncu_sn_<cfg>.json: DRAM bytes per k_sn_solve launch (contact vs
grain batch, told apart by size) from an ncu --csv launch list."""
import csv, json, sys
src, cfg, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, ii, mi, vi = (h.index(k) for k in ('Kernel Name', 'ID', 'Metric Name', 'Metric Value'))
per = {}
for r in rows[hi + 1:]:
    if len(r) <= vi or 'k_sn_solve' not in r[ki]:
        continue
    d = per.setdefault(r[ii], {})
    d[r[mi]] = float(r[vi].replace(',', ''))
launches = []
for lid, d in per.items():
    b = d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
    launches.append((int(lid), b, d.get('gpu__time_duration.sum', 0)))
launches.sort()
big = max(b for _, b, _ in launches)
cls = lambda b: 'contact' if b > 0.8 * big else 'grain'
agg = {}
for _, b, t in launches:
    agg.setdefault(cls(b), []).append(b)
res = {"source": src, "kernel": "k_sn_solve", "config": cfg,
       "dram_bytes_per_launch": {k: sum(v) / len(v) for k, v in agg.items()},
       "launches": {k: len(v) for k, v in agg.items()}}
json.dump(res, open(out, 'w'), indent=1)
print(json.dumps(res, indent=1))
