"""One-off evidence run: C5 at full size (110M points) through the C ABI, compared element by
element with the C oracle (single core, minutes).  Writes gpurun_out/c5_full_check.json."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle
import synth
import paper_2208_07678_b200 as fec

w = synth.make_config("C5")
x = torch.from_numpy(w.points).cuda()
t0 = time.time()
lab = fec.cluster(x, w.d_th, w.min_size, w.max_size).cpu().numpy()
t1 = time.time()
want = oracle.fec(w.points, w.d_th, w.min_size, w.max_size)
t2 = time.time()
bad = int((lab != want).sum())
out = {"config": "C5", "n": int(w.n), "sha256": synth.sha256_f32(w.points), "mismatches": bad,
       "bit_exact": bad == 0, "components": int(len(np.unique(want))), "gpu_call_s": t1 - t0,
       "oracle_s": t2 - t1}
print(json.dumps(out))
json.dump(out, open("gpurun_out/c5_full_check.json", "w"), indent=1)
