"""Summarise tools/timeline.py output: per-kernel in-pipeline durations,
per-stream busy fractions, and one step's schedule as text.

    python tools/timeline_report.py gpurun_out/timeline.json [--step 5]
"""
from __future__ import annotations

import argparse
import collections
import json
import re


def short(name: str) -> str:
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(.*$", "", name)
    return name.replace("hpsgpu::", "")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--step", type=int, default=5)
    ap.add_argument("--marker", default="fwd_bwd_kernel")
    args = ap.parse_args()
    d = json.load(open(args.path))
    ev = d["events"]
    for e in ev:
        e["k"] = short(e["name"])
    # steps delimited by the first body kernel of each batch: the first
    # marker after a gap in markers longer than the mini-batch spacing
    marks = [e["ts"] for e in ev if args.marker in e["k"]]
    J = 4
    starts = marks[::J]
    if len(starts) < args.step + 2:
        raise SystemExit("not enough steps")
    t0, t1 = starts[args.step], starts[args.step + 1]
    period = [b - a for a, b in zip(starts[1:-1], starts[2:])]
    print(f"step period (first body kernel to the next batch's): mean {sum(period)/len(period):.1f} us"
          f" over {len(period)} steps")
    lo, hi = starts[1], starts[-1]
    win = [e for e in ev if lo <= e["ts"] < hi]
    span = hi - lo
    nsteps = len(starts) - 2
    by = collections.defaultdict(list)
    for e in win:
        by[e["k"]].append(e["dur"])
    print(f"\nper kernel, steady state ({nsteps} steps): total us/step, launches/step, mean us")
    rows = sorted(by.items(), key=lambda kv: -sum(kv[1]))
    for k, v in rows[:40]:
        print(f"  {sum(v)/nsteps:8.1f} {len(v)/nsteps:6.1f} {sum(v)/len(v):8.2f}  {k}")
    st = collections.defaultdict(float)
    for e in win:
        st[e["stream"]] += e["dur"]
    print("\nstream busy fraction (sum of kernel durations / wall):")
    for s, v in sorted(st.items(), key=lambda kv: -kv[1]):
        names = collections.Counter(e["k"] for e in win if e["stream"] == s).most_common(3)
        print(f"  stream {s}: {v/span:5.2f}  e.g. {', '.join(n for n, _ in names)}")
    # union busy (any kernel running)
    iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in win)
    busy, cur_s, cur_e = 0.0, None, None
    for s, e in iv:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        busy += cur_e - cur_s
    print(f"\nGPU busy (any kernel) {busy/span:.2f} of wall")
    print(f"\nstep {args.step} schedule (us from its first body kernel):")
    for e in ev:
        if t0 <= e["ts"] < t1:
            print(f"  {e['ts']-t0:8.1f} +{e['dur']:6.1f}  s{e['stream']:<4} {e['k']}")


if __name__ == "__main__":
    main()
