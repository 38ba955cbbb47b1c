import csv, sys
from collections import OrderedDict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv, iid = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
d = OrderedDict()
for r in rows[1:]:
    d.setdefault(r[iid], {'k': r[ik].split('(')[0]})[r[im]] = r[iv]
tot = 0.0
for k, v in d.items():
    t = float(v.get('gpu__time_duration.sum', '0').replace(',', ''))
    tot += t
    rb = float(v.get('dram__bytes_read.sum', '0').replace(',', '')); wb = float(v.get('dram__bytes_write.sum', '0').replace(',', ''))
    print(f"{k:>4} {v['k'][:36]:36s} {t/1e3:9.3f} us  R {rb/1e6:9.1f} MB  W {wb/1e6:9.1f} MB")
print(f"total {tot/1e3:.1f} us")
