"""profiles/traffic.json from an ncu launch list of one clustering call per config: DRAM bytes
(read + write) and ncu duration of each bench stage's kernels (the last call in the list).
usage: python tools/make_traffic.py CONFIG LAUNCHES.csv [CONFIG LAUNCHES.csv ...]"""
import csv
import json
import os
import sys
from collections import OrderedDict

STAGES = {
    "a1_bbox_validate": ["k_bbox", "k_zero"],
    "a2_bin_keys": ["k_lkey", "k_onesweep"],
    "a3_sort": ["k_cmark", "k_smark", "k_cpop", "k_tscan", "k_cscan", "k_cemit", "k_dcount2", "k_sgather", "k_cellred", "k_celltscan", "k_cellscan", "k_scan_lb",
                "k_dcomps"],
    "a4_gather_init": ["k_dscatter", "k_dinit", "k_dparent"],
    # SURVEY's a6+a7 row: every union kernel, the dense-dense links on the side stream included
    "a6a7_scan_union": ["k_union_sparse", "k_union_sparse_local", "k_dense_link",
                        "k_dense_overflow", "k_dense_filter", "k_dense_items"],
    "a8_flatten": ["k_flatten_if"],
    "a9_stats": ["k_tail_stats"],
    "a10_relabel": ["k_rootlab", "k_relabel_in", "k_relabel", "k_relabel_b1", "k_relabel_b2c"],
}


def last_call(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    d = OrderedDict()
    for r in rows[1:]:
        d.setdefault(r[iid], {"k": r[ik].split("(")[0].replace("fec::", "")})[r[im]] = float(r[iv].replace(",", ""))
    launches = list(d.values())
    starts = [i for i, v in enumerate(launches) if v["k"] == "k_bbox"]
    return launches[starts[-1]:] if starts else launches


def main(args):
    out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    data = {"_about": "Per bench stage: DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and ncu duration "
                      "summed over the stage's kernels in the last clustering call of an ncu launch list "
                      "(cold-cache serialised launches; the a6a7 entry includes the dense-dense links that run "
                      "on the side stream).  Written by tools/make_traffic.py from the named csv."}
    for cfg, path in zip(args[0::2], args[1::2]):
        call = last_call(path)
        ent = {"source": os.path.basename(path)}
        for st, ks in STAGES.items():
            sel = [v for v in call if v["k"] in ks]
            ent[st] = {"dram_bytes": sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in sel),
                       "ncu_us": sum(v.get("gpu__time_duration.sum", 0) for v in sel) / 1e3}
        data[cfg] = ent
    json.dump(data, open(out_path, "w"), indent=1)
    print(json.dumps(data, indent=1)[:1500])


if __name__ == "__main__":
    main(sys.argv[1:])
