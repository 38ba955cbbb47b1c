"""Write profiles/<round>_*.md summaries from gpurun_out artefacts (ncu launch list + full capture)."""
import csv, io, json, os, subprocess, sys
from collections import OrderedDict

rnd, launches_csv, rep, bench_json, out = sys.argv[1:6]


def launch_table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, iid = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
    d = OrderedDict()
    for r in rows[1:]:
        d.setdefault(int(r[iid]), {'k': r[ik].split('(')[0].replace('void ', '').replace('fec::', '')})[r[im]] = float(r[iv].replace(',', ''))
    return d


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    return r[0], r[1], r[2:]


L = launch_table(launches_csv)
ids = sorted(L)
# last complete step = kernels after the last k_bbox_partial
last = max(i for i in ids if L[i]['k'] in ('k_bbox', 'k_bbox_partial'))
step = [i for i in ids if i >= last]
tot = sum(L[i]['gpu__time_duration.sum'] for i in step)
lines = [f"# {rnd}: launch list and ncu summary", "",
         "Source: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
         "--clock-control none -c 400 --csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e` "
         "(cold-cache, serialised launches: compare shares, not absolutes).  Raw CSV: "
         f"`{os.path.basename(launches_csv)}`.", "",
         "## One step (last bench step in the capture)", "",
         "| launch | kernel | time (us) | share | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|---|---|"]
for i in step:
    v = L[i]
    t = v['gpu__time_duration.sum']
    lines.append(f"| {i} | {v['k']} | {t/1e3:.1f} | {t/tot*100:.1f}% | {v.get('dram__bytes_read.sum',0)/1e6:.1f} | "
                 f"{v.get('dram__bytes_write.sum',0)/1e6:.1f} |")
lines.append(f"| | **total** | **{tot/1e3:.1f}** | | | |")
hdr, units, rows = raw(rep)
want = [('gpu__time_duration.sum', 'time'), ('dram__bytes_read.sum', 'DRAM rd'), ('dram__bytes_write.sum', 'DRAM wr'),
        ('dram__throughput.avg.pct_of_peak_sustained_elapsed', 'DRAM %'),
        ('lts__t_sector_hit_rate.pct', 'L2 hit %'), ('l1tex__t_sector_hit_rate.pct', 'L1 hit %'),
        ('sm__throughput.avg.pct_of_peak_sustained_elapsed', 'SM %'),
        ('sm__warps_active.avg.pct_of_peak_sustained_active', 'occupancy %'),
        ('smsp__thread_inst_executed_per_inst_executed.ratio', 'threads/inst'),
        ('launch__registers_per_thread', 'regs'), ('smsp__inst_executed.sum', 'warp inst')]
lines += ["", f"## `ncu --set full` capture (`{os.path.basename(rep)}`)", "",
          "| kernel | " + " | ".join(w[1] for w in want) + " |", "|---|" + "---|" * len(want)]
for row in rows:
    name = row[hdr.index('Kernel Name')].split('(')[0]
    cells = []
    for key, _ in want:
        if key in hdr:
            i = hdr.index(key)
            cells.append(f"{row[i]} {units[i]}".strip())
        else:
            cells.append("-")
    lines.append(f"| {name} | " + " | ".join(cells) + " |")
b = json.load(open(bench_json))
lines += ["", "## Bench line of the same build", "", "```json", json.dumps(b, indent=1)[:6000], "```", ""]
open(out, "w").write("\n".join(lines))
print(out)
