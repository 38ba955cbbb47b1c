"""Per-rank device time of the multi-GPU slab step, emulated on ONE GPU: every rank's
fec_slab_local + fec_slab_merge (the all-gather replaced by the concatenated record buffers)
timed separately with CUDA events; the max over ranks predicts the N-GPU step time without
the NCCL all-gather.  Not a bench value."""
import json
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import synth
import paper_2208_07678_b200 as fec
from paper_2208_07678_b200 import dist as fdist

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
worlds = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
reps = 10
w = synth.make_config(name)
fec.lib()
out = {"config": name, "n": w.n}
for world in worlds:
    plan = fdist.plan_slabs(w.points, w.d_th, world)
    words = fec.slab_record_words(plan.rec_cap)
    ranks = []
    for r in range(world):
        sh = fdist.shard(w.points, plan, r)
        x = torch.from_numpy(sh.points).cuda()
        g = torch.from_numpy(sh.gidx).cuda()
        ws = torch.empty(fec.slab_workspace_bytes(sh.points.shape[0], world, plan.rec_cap), dtype=torch.uint8,
                         device="cuda")
        rec = torch.empty(words, dtype=torch.int32, device="cuda")
        lab = torch.empty(max(sh.n_owned, 1), dtype=torch.int32, device="cuda")
        ranks.append((sh, x, g, ws, rec, lab))
    # records of every rank once (the all-gather's result)
    states = [fec.slab_local(x, g, sh.n_owned, sh.n_first, w.d_th, rec, plan.rec_cap, ws) for sh, x, g, ws, rec, lab in ranks]
    allrec = torch.cat([rk[4] for rk in ranks])
    times = []
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    for r, (sh, x, g, ws, rec, lab) in enumerate(ranks):
        best = (1e9, 1e9)
        for _ in range(reps):
            torch.cuda.synchronize()
            e0.record()
            st = fec.slab_local(x, g, sh.n_owned, sh.n_first, w.d_th, rec, plan.rec_cap, ws)
            e1.record()
            fec.slab_merge(allrec, world, r, w.min_size, w.max_size, lab, ws, st)
            e2.record()
            torch.cuda.synchronize()
            best = min(best, (e0.elapsed_time(e2), e1.elapsed_time(e2)))
        times.append({"rank": r, "n_local": int(sh.points.shape[0]), "ms": best[0], "merge_ms": best[1]})
    mx = max(t["ms"] for t in times)
    out[str(world)] = {"ranks": times, "max_ms": mx, "pred_mpts_s_without_nccl": w.n / (mx * 1e-3) / 1e6,
                       "rec_cap": plan.rec_cap}
    print(world, "max rank ms", round(mx, 3), "pred Mpts/s", round(w.n / (mx * 1e-3) / 1e6), flush=True)
json.dump(out, open("gpurun_out/slab_rank_time_%s.json" % name, "w"), indent=1)
