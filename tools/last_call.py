"""Per-kernel duration and DRAM bytes of the last clustering call in an ncu launch-list csv."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); mi = h.index('Metric Name'); ii = h.index('ID')
launch = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi: continue
    d = launch.setdefault(r[ii], {'k': r[ki].split('(')[0]})
    d[r[mi]] = float(r[vi].replace(',', ''))
L = list(launch.values())
first = sys.argv[2] if len(sys.argv) > 2 else 'k_bbox'
last = max(i for i, d in enumerate(L) if d['k'] == first)
tot = 0
for d in L[last:]:
    t = d.get('gpu__time_duration.sum', 0) / 1000; tot += t
    b = (d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)) / 1e6
    print(f"{d['k']:26s} {t:8.1f} us {b:9.1f} MB {b / t if t else 0:6.2f} TB/s")
print(f"total {tot:.1f} us")
