"""Host-side enqueue time of one fec_cluster call vs its device time (is the CPU launch rate a
bottleneck?).  python tools/host_overhead.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
import synth
import paper_2208_07678_b200 as fec

w = synth.make_config("C4")
for frac in (1.0, 0.125):
    n = int(w.n * frac)
    x = torch.from_numpy(w.points[:n].copy()).cuda()
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    ws = torch.empty(fec.workspace_bytes(n), dtype=torch.uint8, device="cuda")
    for _ in range(5):
        fec.cluster(x, w.d_th, w.min_size, w.max_size, out=out, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host = []
    e0.record()
    for _ in range(20):
        t = time.perf_counter()
        fec.cluster(x, w.d_th, w.min_size, w.max_size, out=out, workspace=ws)
        host.append(time.perf_counter() - t)
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / 20
    print(f"n={n}: device {dev:.3f} ms/call, host enqueue {1e3 * sorted(host)[10]:.3f} ms/call (median)")
