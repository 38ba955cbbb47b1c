"""One-off evidence run: many seeded random clouds (all synth geometries, sizes up to 40k,
random size filters) in all four grid modes, labels compared with the oracle element by
element.  Writes gpurun_out/stress_parity.json."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle
import synth
import paper_2208_07678_b200 as fec

fec.lib()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
t0 = time.time()
res = {"clouds": 0, "labels": 0, "mismatching_clouds": [], "modes": [0, 1, 2, 3]}
for seed in range(5000, 5000 + N):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40_000))
    p, d, geom = synth.random_cloud(seed, n=n)
    mn = int(rng.integers(0, 8))
    mx = int(rng.integers(max(mn, 1), 5000))
    want = oracle.fec(p, d, mn, mx)
    x = torch.from_numpy(p).cuda()
    for mode in res["modes"]:
        fec.set_grid_mode(mode)
        got = fec.cluster(x, d, mn, mx).cpu().numpy()
        if not np.array_equal(got, want):
            res["mismatching_clouds"].append([seed, mode, geom, n])
    res["clouds"] += 1
    res["labels"] += 4 * n
fec.set_grid_mode(0)
res["seconds"] = time.time() - t0
res["bit_exact"] = not res["mismatching_clouds"]
print(json.dumps(res))
json.dump(res, open("gpurun_out/stress_parity.json", "w"), indent=1)
