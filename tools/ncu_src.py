"""Top CUDA source lines of one kernel in an ncu report by warp-stall samples (the report must
have been captured with --import-source on and the binary built with -lineinfo).
usage: python tools/ncu_src.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys
from collections import defaultdict
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = defaultdict(lambda: [0.0, ""])
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == "Line No":
        h = r
        i_st = h.index("Warp Stall Sampling (All Samples)")
        i += 1
        while i < len(rows) and rows[i] and rows[i][0] not in ("File Path", "Line No", "Kernel Name"):
            x = rows[i]
            if len(x) > i_st and x[0].strip().isdigit():
                try:
                    agg[int(x[0])][0] += float(x[i_st] or 0)
                    agg[int(x[0])][1] = x[1]
                except ValueError:
                    pass
            i += 1
        continue
    i += 1
tot = sum(v[0] for v in agg.values()) or 1.0
for ln, (v, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v / tot * 100:5.1f}%  L{ln:>5}  {src.strip()[:110]}")
