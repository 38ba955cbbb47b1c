"""Workload for compute-sanitizer (T8): C1 plus 20 seeded random clouds through the C ABI, in
every grid mode, each checked against the oracle.  Prints one line per case."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2208_07678_b200 as fec  # noqa: E402

bad = 0
cases = [("C1",) + tuple(synth.make_config("C1").__dict__[k] for k in ("points", "d_th", "min_size", "max_size"))]
for s in range(20):
    p, d, geom = synth.random_cloud(s, n=int(np.random.default_rng(s).integers(200, 4000)))
    cases.append((f"seed{s}-{geom}", p, d, 2, 10**6))
# clouds above the small-cloud threshold: the counting path with dense cells and the side
# stream (C4 at 1%), and the key-sort path of shuffled input (C5 at 0.2%)
for name, scale in (("C4", 0.01), ("C5", 0.002)):
    w = synth.make_config(name, scale=scale)
    cases.append((f"{name}@{scale}", w.points, w.d_th, w.min_size, w.max_size))
for mode in (0, 1, 2, 3):
    fec.set_grid_mode(mode)
    for name, p, d, mn, mx in cases:
        got = fec.cluster(torch.from_numpy(p).cuda(), d, mn, mx).cpu().numpy()
        ok = np.array_equal(got, oracle.fec(p, d, mn, mx))
        bad += not ok
        print(f"mode {mode} {name} n={len(p)} {'ok' if ok else 'MISMATCH'}", flush=True)
fec.set_grid_mode(0)
print("mismatches", bad)
sys.exit(1 if bad else 0)
