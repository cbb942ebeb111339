"""profiles/traffic.json from an ncu capture of the sparse segment-reduce
kernels (tools/profile_r.sh: sparse_traffic.csv).

traffic = dram__bytes_read.sum + dram__bytes_write.sum summed over the
kernels of one mini-batch (big_classify, big_plan, big_fused, sparse_short),
averaged over the mini-batches captured. bench.py reports it as
roofline.traffic for the "sparse" phase, and big_fused_kernel's own per-launch
traffic as roofline.kernels.big_fused_kernel.traffic.

usage: python tools/traffic_json.py gpurun_out/sparse_traffic.csv [config]
"""
import collections
import csv
import json
import os
import sys

KERNELS = ("big_classify", "big_plan", "big_fused", "sparse_short", "sparse_mid")


def main() -> None:
    path = sys.argv[1]
    config = sys.argv[2] if len(sys.argv) > 2 else "c2"
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ci, ki, mi, vi = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per[int(r[ci])]["name"] = r[ki]
        per[int(r[ci])][r[mi]] = float(r[vi].replace(",", ""))
    launches = [per[i] for i in sorted(per)]
    total = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
                for l in launches if any(k in l["name"] for k in KERNELS))
    mbs = sum(1 for l in launches if "sparse_short" in l["name"])
    out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles",
                            "traffic.json")
    try:
        doc = json.load(open(out_path))
    except (OSError, ValueError):
        doc = {}
    doc.setdefault(config, {})["sparse"] = int(round(total / max(mbs, 1)))
    big = [l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
           for l in launches if "big_fused" in l["name"]]
    if big:  # per launch of big_fused_kernel alone
        doc[config]["big_fused"] = int(round(sum(big) / len(big)))
    doc["_note"] = (
        "dram__bytes_read.sum + dram__bytes_write.sum summed over the sparse segment-reduce "
        "kernels of one mini-batch (" + ", ".join(KERNELS) + "), averaged over " + str(mbs) +
        " mini-batches; ncu with its default cache control (caches flushed before each kernel), "
        "profiles/r2_sparse_traffic.csv. Reads are the dL/dx records, the CSR grouping and the "
        "table rows the in-place apply updates; the row writes stay in L2 within a kernel")
    json.dump(doc, open(out_path, "w"), indent=1)
    print(json.dumps(doc[config]), mbs, "mini-batches")


if __name__ == "__main__":
    main()
