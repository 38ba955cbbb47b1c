"""Writes tests/golden/full_size.json: for each BASELINE config C1-C5 at full size, the sha256
of the fp32 input cloud (synth/) and the sha256 of the ORACLE's labels (oracle/, int32
little-endian bytes in input order), plus summary counts.

Calls only synth/ and oracle/ (never the CUDA path): the stored expected values come from
the oracle alone.  C5 takes ~8 minutes of one core.  Usage:
    python tools/make_full_size_digests.py [C1 C2 ...]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "full_size.json")


def main(names):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {
        "about": "sha256 of each full-size config's fp32 input (synth/) and of the oracle's int32 labels "
                 "(oracle.fec, input order, little-endian); written by tools/make_full_size_digests.py, "
                 "which calls only synth/ and oracle/",
        "configs": {}}
    for name in names:
        t0 = time.time()
        w = synth.make_config(name)
        t1 = time.time()
        lab = oracle.fec(w.points, w.d_th, w.min_size, w.max_size)
        t2 = time.time()
        lab = np.ascontiguousarray(lab, dtype="<i4")
        kept = lab[lab >= 0]
        data["configs"][name] = {
            "n": int(w.n), "d_th": float(np.float32(w.d_th)), "min_size": int(w.min_size),
            "max_size": int(w.max_size),
            "input_sha256": synth.sha256_f32(w.points),
            "labels_sha256": hashlib.sha256(lab.tobytes()).hexdigest(),
            "noise": int((lab < 0).sum()), "clusters": int(len(np.unique(kept))),
            "oracle_s": round(t2 - t1, 1), "generate_s": round(t1 - t0, 1)}
        print(name, data["configs"][name], flush=True)
        json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"])
