"""Repeat the slab emulation / single path on one random test cloud and report mismatches."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle
import paper_2208_07678_b200 as fec
from test_dist_cpu import clouds
from test_gpu_dist import run_emulated

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
pts, d = clouds()[k]
want = oracle.fec(pts, d, 1, 2**62)
print("cloud", k, "n", len(pts), "d", d)
for mode in (0, 2, 3, 1):
    fec.set_grid_mode(mode)
    bad_runs = 0
    for r in range(reps):
        t = torch.from_numpy(pts).cuda()
        got = fec.cluster(t, d, 1, 2**62).cpu().numpy()
        if not np.array_equal(got, want):
            bad_runs += 1
            if bad_runs <= 2:
                b = np.nonzero(got != want)[0]
                print(" single mode", mode, "run", r, "bad", b[:10], got[b[:5]], want[b[:5]])
    print("single mode", mode, "bad runs", bad_runs, "/", reps)
    bad_runs = 0
    for r in range(reps):
        got, _ = run_emulated(fec, pts, d, world, 1, 2**62)
        if not np.array_equal(got, want):
            bad_runs += 1
            if bad_runs <= 2:
                b = np.nonzero(got != want)[0]
                print(" slab mode", mode, "run", r, "bad", b[:10], got[b[:5]], want[b[:5]])
    print("slab mode", mode, "bad runs", bad_runs, "/", reps)
fec.set_grid_mode(0)
