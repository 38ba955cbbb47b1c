"""One rank of an emulated multi-GPU slab step (for ncu launch lists): python tools/prof_slab.py C4 8 3"""
import sys
import torch
sys.path.insert(0, '.')
import synth
import paper_2208_07678_b200 as fec
from paper_2208_07678_b200 import dist as fdist

name, world, rank = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
w = synth.make_config(name)
plan = fdist.plan_slabs(w.points, w.d_th, world)
words = fec.slab_record_words(plan.rec_cap)
fec.lib()
bufs = []
for r in range(world):
    sh = fdist.shard(w.points, plan, r)
    bufs.append(sh)
sh = bufs[rank]
x = torch.from_numpy(sh.points).cuda()
g = torch.from_numpy(sh.gidx).cuda()
ws = torch.empty(fec.slab_workspace_bytes(sh.points.shape[0], world, plan.rec_cap), dtype=torch.uint8, device="cuda")
rec = torch.zeros(words * world, dtype=torch.int32, device="cuda")
lab = torch.empty(sh.n_owned, dtype=torch.int32, device="cuda")
fec.set_timing(True)
for it in range(3):
    st = fec.slab_local(x, g, sh.n_owned, sh.n_first, w.d_th, rec[rank * words:(rank + 1) * words], plan.rec_cap, ws)
    fec.slab_merge(rec, world, rank, w.min_size, w.max_size, lab, ws, st)
    torch.cuda.synchronize()
    print({k: round(v, 3) for k, v in fec.stage_times().items()})
