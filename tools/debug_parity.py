"""Debug helper: find label mismatches GPU vs oracle for a random cloud and explain them."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle, synth
import paper_2208_07678_b200 as fec
from oracle.brute import pred_f32

seed, n, geom = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
mn, mx = int(sys.argv[4]), int(sys.argv[5])
p, d, _ = synth.random_cloud(seed, n=n, geometry=geom)
print("d", d, "n", n)
un_o = oracle.fec(p, d)
fec.set_instrumentation(True)
for trial in range(5):
    got = fec.cluster(torch.from_numpy(p).cuda(), d).cpu().numpy()
    print("trial", trial, "mismatch", int((got != un_o).sum()), fec.stats())
bad = np.nonzero(got != un_o)[0]
print("bad", bad[:20])
c = d * (1 + 2**-16); h = c / 2; lo = p.min(0).astype(np.float64)
sub = np.floor((p.astype(np.float64) - lo) / h).astype(np.int64)
for i in bad[:3]:
    nb = np.nonzero(pred_f32(p[i][None, :], p, d))[0]
    print("point", i, "sub", sub[i], "cell", sub[i] >> 1, "gpu", got[i], "oracle", un_o[i])
    for j in nb[:20]:
        print("   nb", j, "sub", sub[j], "cell", sub[j] >> 1, "gpu", got[j], "oracle", un_o[j], "dsub", sub[j] - sub[i])
