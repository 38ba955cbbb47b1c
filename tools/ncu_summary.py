"""Summarise an ncu report: per-kernel key metrics (+ optional top source lines)."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units, rows = r[0], r[1], r[2:]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'launch__grid_size', 'smsp__inst_executed.sum']
idx = [(w, hdr.index(w)) for w in want if w in hdr]
for row in rows:
    print(" | ".join(f"{w.split('__')[-1][:22]}={row[i][:34]}{units[i] if units[i] not in ('', 'register/thread') else ''}" for w, i in idx))
if len(sys.argv) > 2:
    kern = sys.argv[2]
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(src)))
    # may contain several kernels; take the first table
    h = next(x for x in rr if 'Source' in x); data = [x for x in rr if len(x) == len(h) and x != h and x[h.index('Warp Stall Sampling (All Samples)')].replace('.', '', 1).isdigit()]
    i_src = h.index('Source'); i_st = h.index('Warp Stall Sampling (All Samples)'); i_ex = h.index('Instructions Executed')
    tot = sum(float(x[i_st] or 0) for x in data) or 1
    for x in sorted(data, key=lambda x: -float(x[i_st] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
        print(f"{float(x[i_st])/tot*100:5.1f}%  {x[i_src][:80]}  ex={x[i_ex]}")
