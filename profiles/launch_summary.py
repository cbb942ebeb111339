"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel share of device time (cold-cache, serialised launches)."""
import collections
import csv
import re
import sys


def summarise(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    out = [f"{'share':>7} {'total_us':>11} {'launches':>8} {'avg_us':>9}  kernel"]
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{t / tot * 100:6.2f}% {t:11.1f} {c:8d} {t / c:9.2f}  {n}")
    out.append(f"total device time {tot:.1f} us over {sum(c for c, _ in agg.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
