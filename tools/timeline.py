"""Kernel timeline of the pipelined bench step (diagnostics, GPU box).

Runs the bench's device-resident c2 loop (hps_submit_batch / hps_wait_batch,
batches in flight, CUDA graphs) under torch.profiler with CUDA activity
tracing (CUPTI: kernels inside graph launches included, with their streams),
and writes every kernel's (name, stream, start, end) of the steady-state
steps to a JSON list. tools/timeline_report.py summarises it: per-stream
busy time, per-kernel in-pipeline durations, the critical-path view.

    python tools/timeline.py [--config c2] [--steps 12] [--out gpurun_out/timeline.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    import bench
    import paper_2003_05622_b200 as pkg

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "timeline.json"))
    ap.add_argument("--host", action="store_true",
                    help="the e2e path: pinned host batches and a pinned host value store")
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    dims, E, B, J = c["dims"], c["E"], c["B"], c["J"]
    P = 8
    off, keys, lab = bench.make_data(c, P * B)
    batches = []
    for b in range(P):
        o = (off[b * B:(b + 1) * B + 1] - off[b * B]).astype(np.int64)
        batches.append((o, keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B]))
    max_keys = max(int(b[0][-1]) for b in batches)
    dev = torch.device("cuda:0")
    tier = pkg.Tier(width=E, layer_dims=c["layers"], minibatches=J, key_space=dims,
                    max_batch_examples=B, max_batch_keys=max_keys, optimizer=c.get("opt", "sgd"))
    if args.host:
        hstore_t = torch.zeros((dims, tier.row_width), dtype=torch.float32).pin_memory()
        tier.attach_store(hstore_t.numpy())
        hb = [tuple(torch.from_numpy(x).pin_memory().numpy() for x in (o, k.view(np.int64), l))
              for o, k, l in batches]

        def step(b):
            o, k, l = hb[b % P]
            tier.submit_batch(o, k.view(np.uint64), l, on_device=False)
    else:
        dbatches = [(torch.from_numpy(o).to(dev), torch.from_numpy(k.view(np.int64)).to(dev),
                     torch.from_numpy(l).to(dev)) for o, k, l in batches]
        dstore = torch.zeros((dims, tier.row_width), dtype=torch.float32, device=dev)
        tier.attach_store(dstore.data_ptr(), on_device=True, num_keys=dims)

        def step(b):
            o, k, l = dbatches[b % P]
            tier.submit_batch((o.data_ptr(), B), k.data_ptr(), l.data_ptr(), on_device=True)

    lag = 3
    n = 0
    for i in range(args.warmup):
        step(n)
        n += 1
        if i >= lag:
            tier.wait_batch()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for i in range(args.steps):
            step(n)
            n += 1
            tier.wait_batch()
        torch.cuda.synchronize()
    for _ in range(lag):
        tier.wait_batch()
    tier.close()
    path = args.out + ".trace.json"
    prof.export_chrome_trace(path)
    with open(path) as f:
        tr = json.load(f)
    ev = [e for e in tr.get("traceEvents", [])
          if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
    out = [{"name": e["name"], "cat": e["cat"], "stream": e.get("args", {}).get("stream", e.get("tid")),
            "ts": e["ts"], "dur": e["dur"]} for e in ev]
    out.sort(key=lambda x: x["ts"])
    with open(args.out, "w") as f:
        json.dump({"config": args.config, "steps": args.steps, "events": out}, f)
    os.remove(path)
    print(f"{len(out)} device events over {args.steps} steps -> {args.out}")


if __name__ == "__main__":
    main()
