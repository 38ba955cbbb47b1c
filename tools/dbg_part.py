"""Debug: partition path vs oracle on small shuffled clouds (mismatch counts per grid mode)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle, synth  # noqa: E401
import paper_2208_07678_b200 as fec

for name, scale in (("C5", 0.002), ("C5", 0.01), ("C4", 0.01)):
    w = synth.make_config(name, scale=scale)
    pts = w.points if name == "C5" else w.points[np.random.default_rng(1).permutation(w.n)]
    ref = oracle.fec(pts, w.d_th, w.min_size, w.max_size)
    for mode in (0, 2, 3):
        fec.set_grid_mode(mode)
        fec.set_instrumentation(True)
        got = fec.cluster(torch.from_numpy(pts).cuda(), w.d_th, w.min_size, w.max_size).cpu().numpy()
        st = fec.stats()
        fec.set_instrumentation(False)
        bad = np.flatnonzero(got != ref)
        print(name, scale, "mode", mode, "binning", st["binning"], "cells", st["cells"], "mismatch", bad.size,
              bad[:5], got[bad[:5]], ref[bad[:5]], flush=True)
fec.set_grid_mode(0)
