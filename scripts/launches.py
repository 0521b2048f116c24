"""Summarize an ncu --csv launch list (gpu__time_duration + dram bytes)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki, mi, vi, idi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
gi = h.index('Grid Size') if 'Grid Size' in h else None
launch = {}
for r in data:
    if len(r) < len(h):
        continue
    d = launch.setdefault(int(r[idi]), {'name': r[ki], 'grid': r[gi] if gi is not None else ''})
    d[r[mi]] = float(r[vi].replace(',', ''))
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
order = []
for k in sorted(launch):
    d = launch[k]
    nm = d['name'].split('(')[0]
    nm = nm.replace('void fasmg::', '')
    t = d.get('gpu__time_duration.sum', 0)
    by = d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
    order.append((nm, t, by, d['grid']))
    key = nm.split('<')[0]
    tot[key][0] += 1; tot[key][1] += t; tot[key][2] += by
skip = ('at::',)
alltime = sum(v[1] for k, v in tot.items() if not k.startswith(skip))
for k, v in sorted(tot.items(), key=lambda x: -x[1][1]):
    if k.startswith(skip):
        continue
    print(f"{k:28s} n={v[0]:4d} time={v[1]/1e6:8.3f} ms ({100*v[1]/alltime:5.1f}%) dram={v[2]/1e9:7.2f} GB  {v[2]/v[1] if v[1] else 0:7.1f} GB/s")
print('total fasmg kernel ms', alltime / 1e6)
if len(sys.argv) > 2:
    for nm, t, by, g in order[: int(sys.argv[2])]:
        print(f"{nm[:40]:40s} {t/1e3:9.1f} us {by/1e9:7.3f} GB {by/t if t else 0:7.1f} GB/s")
