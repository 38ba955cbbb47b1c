"""Debug: random clouds through fec_cluster vs the oracle, with the call's stats."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2208_07678_b200 as fec
import synth
import oracle
fec.set_instrumentation(True)
for seed in range(12):
    p, d, geom = synth.random_cloud(seed)
    want = oracle.fec(p, d, 2, 500)
    x = torch.from_numpy(p).cuda()
    out = torch.empty(len(p), dtype=torch.int32, device="cuda")
    fec.cluster(x, d, 2, 500, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    print(seed, geom, len(p), "differ", int((got != want).sum()), fec.stats())
