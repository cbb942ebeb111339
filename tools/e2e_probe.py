"""Phase breakdown of the end-to-end (host-buffer) path of bench.py's c2
workload: where do the host<->device milliseconds go? Diagnostic only.

  python tools/e2e_probe.py [--steps 40] [--store host|device] [--batch host|device]
"""
import argparse
import os as _os

# The batch pipeline drives several concurrent streams (stage, prep, grouping,
# store gather, body, dense-grad side stream, write-back): with CUDA's default
# 8 hardware work queues, two of them can share a queue and one stream's
# waits stall another's work. Must be set before the CUDA context exists.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_05622_b200 as pkg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--store", default="host")
    ap.add_argument("--batch", default="host")
    a = ap.parse_args()
    dims, E, B, nnz, J, P = 10**7, 16, 16384, 100, 4, 8
    off, keys, lab = pkg.gen_dataset(dims, P * B, nnz, zipf=True, seed=1)
    hb, db = [], []
    for b in range(P):
        o = (off[b * B:(b + 1) * B + 1] - off[b * B]).astype(np.int64)
        k, l = keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B]
        hb.append(tuple(torch.from_numpy(x).pin_memory() for x in (o, k.view(np.int64), l)))
        db.append(tuple(x.cuda() for x in hb[-1]))
    tier = pkg.Tier(width=E, layer_dims=(8, 16, 1), minibatches=J, key_space=dims,
                    max_batch_examples=B, max_batch_keys=max(int(x[0][-1]) for x in hb))
    if a.store == "host":
        st = torch.zeros((dims, E), dtype=torch.float32).pin_memory()
        tier.attach_store(st.numpy())
    else:
        st = torch.zeros((dims, E), dtype=torch.float32, device="cuda")
        tier.attach_store(st.data_ptr(), on_device=True, num_keys=dims)

    def submit(i):
        if a.batch == "host":
            o, k, l = hb[i % P]
            return tier.submit_batch(o.numpy(), k.numpy().view(np.uint64), l.numpy())
        o, k, l = db[i % P]
        return tier.submit_batch((o.data_ptr(), B), k.data_ptr(), l.data_ptr(), on_device=True)

    def step(i):
        submit(i)
        return tier.wait_batch()

    def pipelined(n):
        t0 = time.perf_counter()
        for i in range(n):
            submit(i)
            if i >= 3:
                tier.wait_batch()
        for _ in range(min(n, 3)):
            tier.wait_batch()
        tier.flush()
        return (time.perf_counter() - t0) / n * 1e3

    pipelined(4)
    wall = pipelined(a.steps)
    t0 = time.perf_counter()
    for i in range(a.steps):
        step(i)
    tier.flush()
    sync_wall = (time.perf_counter() - t0) / a.steps * 1e3
    tier.set_timing(True)
    for i in range(2):
        step(i)
    tier.flush()
    tier.reset_timing()
    for i in range(a.steps):
        step(i)
    tier.flush()
    ph = {k: round(v / a.steps, 3) for k, v in tier.timing().items()}
    print(f"store={a.store} batch={a.batch}: pipelined {wall:.3f} ms/step, one at a time "
          f"{sync_wall:.3f}; phases {ph}")
    tier.close()


if __name__ == "__main__":
    main()
