"""One warm-up + one measured call of the FEC path on a config (for ncu captures)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import synth
import paper_2208_07678_b200 as fec

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = synth.make_config(name, scale=scale)
x = torch.from_numpy(w.points).cuda()
ws = torch.empty(fec.workspace_bytes(w.n), dtype=torch.uint8, device='cuda')
out = torch.empty(w.n, dtype=torch.int32, device='cuda')
for _ in range(reps):
    fec.cluster(x, w.d_th, w.min_size, w.max_size, out=out, workspace=ws)
torch.cuda.synchronize()
print("ok", name, w.n)
