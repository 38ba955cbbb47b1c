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
out = {"config": name, "n": w.n, "timing": "per rank: CUDA-graph replay of fec_slab_local + fec_slab_merge (NCCL all-gather excluded)"}
# the single-GPU path on the whole cloud, same timing method
x1 = torch.from_numpy(w.points).cuda()
o1 = torch.empty(w.n, dtype=torch.int32, device="cuda")
ws1 = torch.empty(fec.workspace_bytes(w.n), dtype=torch.uint8, device="cuda")
st1 = torch.zeros(1, dtype=torch.int32, device="cuda")
g1 = torch.cuda.CUDAGraph()
s1 = torch.cuda.Stream()
s1.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s1):
    fec.cluster(x1, w.d_th, w.min_size, w.max_size, out=o1, workspace=ws1, status=st1, check=False)
torch.cuda.synchronize()
with torch.cuda.graph(g1, stream=s1):
    fec.cluster(x1, w.d_th, w.min_size, w.max_size, out=o1, workspace=ws1, status=st1, check=False)
torch.cuda.synchronize()
ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best1 = 1e9
for _ in range(reps):
    torch.cuda.synchronize()
    ea.record()
    g1.replay()
    eb.record()
    torch.cuda.synchronize()
    best1 = min(best1, ea.elapsed_time(eb))
out["single_gpu_ms"] = best1
print("single GPU ms", round(best1, 3), flush=True)
del x1, o1, ws1
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
    e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
    for r, (sh, x, g, ws, rec, lab) in enumerate(ranks):
        # one rank's device work (local step + merge on the gathered records) captured in a CUDA
        # graph and replayed: no host launch cost in the timing (the call has no host round trip)
        def step():
            st = fec.slab_local(x, g, sh.n_owned, sh.n_first, w.d_th, rec, plan.rec_cap, ws)
            fec.slab_merge(allrec, world, r, w.min_size, w.max_size, lab, ws, st)
        graph = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            step()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=cs):
            step()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            e0.record()
            graph.replay()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        times.append({"rank": r, "n_local": int(sh.points.shape[0]), "ms": best})
    mx = max(t["ms"] for t in times)
    out[str(world)] = {"ranks": times, "max_ms": mx, "pred_mpts_s_without_nccl": w.n / (mx * 1e-3) / 1e6,
                       "rec_cap": plan.rec_cap, "speedup_vs_single_gpu": best1 / mx}
    print(world, "max rank ms", round(mx, 3), "pred Mpts/s", round(w.n / (mx * 1e-3) / 1e6),
          "speedup", round(best1 / mx, 2), flush=True)
    del ranks, allrec, states
json.dump(out, open("gpurun_out/slab_rank_time_%s.json" % name, "w"), indent=1)
