"""Per-CUDA-source-line warp-stall share of one kernel in an ncu report (cuda,sass view)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern],
                     capture_output=True, text=True).stdout
agg = {}
src = {}
cur = None
fname = ""
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    if cur is None or len(r) < 5:
        continue
    try:
        v = float(r[4])
    except ValueError:
        continue
    agg[cur] = agg.get(cur, 0.0) + v
tot = sum(agg.values()) or 1.0
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / tot * 100:5.1f}% {k[0]}:{k[1]:<5d} {src[k].strip()[:110]}")
