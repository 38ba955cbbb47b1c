import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle
import paper_2208_07678_b200 as fec
from paper_2208_07678_b200 import dist as fdist
from test_dist_cpu import clouds

pts, d = clouds()[5]
plan = fdist.plan_slabs(pts, d, 2)
for r in range(2):
    sh = fdist.shard(pts, plan, r)
    want = oracle.fec(sh.points, d, 1, 2**62)
    for mode in (2, 3):
        fec.set_grid_mode(mode)
        got = fec.cluster(torch.from_numpy(sh.points).cuda(), d, 1, 2**62).cpu().numpy()
        b = np.nonzero(got != want)[0]
        print("rank", r, "mode", mode, "n", len(sh.points), "bad", b[:10], got[b[:5]], want[b[:5]])
        if len(b) and mode == 2:
            # is the shard's input order coherent?  dump a few facts
            fec.set_instrumentation(True)
            fec.cluster(torch.from_numpy(sh.points).cuda(), d, 1, 2**62)
            print(fec.stats())
            fec.set_instrumentation(False)
            np.save('gpurun_out/bad_shard.npy', sh.points)
fec.set_grid_mode(0)
