#!/usr/bin/env python
"""Benchmark of the HBM-PS hot path (one JSON line on rank 0).

A step is one batch of the BASELINE workload through the tier: working-set
dedup -> table build (carry-over + value-store staging) -> J mini-batches of
{dedup, pull, fwd/bwd, segment-reduce, push, canonical apply, dense sync} ->
write-back. Workload (config.workload): BASELINE.json configs[1] ("c2"):
10M-key space, E=16, batch 16384, Zipf(1.0) keys, 100 keys/example, 3-layer
MLP {8,16,1}, J=4; at N GPUs the same batch is sharded over the N ranks
(strong scaling, as the reference shards a node's batch over its devices).

  value : examples/s with the batch pool and the value store resident in HBM
  e2e   : the same through the C ABI with HOST buffers: pinned batch H2D,
          rows staged from / written back to a pinned host value store
          (zero-copy), loss D2H — all inside the timed region.

Timing: CUDA events on the tier's own stream around the whole run of K steps
(steps are pipelined: batch b's write-back overlaps batch b+1, and the region
ends with hps_flush), inputs larger than L2 instead of an L2 flush, max over
ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import os as _os

# The batch pipeline drives several concurrent streams (stage, prep, grouping,
# store gather, body, dense-grad side stream, write-back): with CUDA's default
# 8 hardware work queues, two of them can share a queue and one stream's
# waits stall another's work. Must be set before the CUDA context exists.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train examples/sec at 1/2/4/8 B200; pull+push keys/sec and HBM GB/s vs roofline"
UNIT = "examples/s"

CONFIGS = {
    "c1": dict(dims=10**6, E=8, B=4096, nnz=100, zipf=False, J=4, layers=(8, 16, 1),
               text="c1: 1M-key table, E=8, batch 4096, ~100 uniform keys/example, "
                    "MLP {8,16,1}, J=4"),
    "c2": dict(dims=10**7, E=16, B=16384, nnz=100, zipf=True, J=4, layers=(8, 16, 1),
               text="c2: 10M-key table, E=16, batch 16384, Zipf(1.0) keys, 100 keys/example, "
                    "MLP {8,16,1}, J=4"),
    "c3": dict(dims=10**8, E=64, B=65536, nnz=100, zipf=False, J=4, layers=(8, 16, 1),
               opt="adagrad",
               text="c3: 100M-key table, E=64 with Adagrad state (rows of 2E floats), batch "
                    "65536, 100 uniform keys/example, MLP {8,16,1}, J=4"),
    # the multi-slot ads model (100 fields, multi-hot up to 300
    # keys/example, key = slot * 1e6 + id) with the wide MLP on tcgen05
    "c4": dict(dims=100 * 10**6, E=16, B=16384, nnz=300, zipf=True, J=4,
               layers=(512, 256, 128, 1), gen="multislot",
               text="c4: multi-slot ads model, 100 slots x 1M ids (100M-key table), multi-hot "
                    "1..300 keys/example (Zipf ids), E=16 sum-combined, MLP {512,256,128,1} "
                    "(3xTF32 tcgen05 GEMMs), batch 16384, J=4"),
    # the MEM-PS host tier at scale (1B keys x E=16 = 64 GB of
    # store; GPU box only)
    "c5": dict(dims=10**9, E=16, B=131072, nnz=100, zipf=False, J=4, layers=(8, 16, 1),
               text="c5: 1B-key value store (64 GB), E=16, batch 131072, 100 uniform "
                    "keys/example, MLP {8,16,1}, J=4"),
}



def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------- clocks --

class ClockSampler:
    """nvidia-smi clocks/throttle reasons DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 15.0) -> bool:
        """Block until nvidia-smi produced its first sample (so the sampler
        is live when the timed region starts)."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.02)
        return bool(self.lines)

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- reference --

def host_threads() -> int:
    n = os.cpu_count() or 1
    p = 1
    while p * 2 <= min(n, 64):
        p *= 2
    return p


def make_data(c, n, seed=1):
    """The config's synthetic batch stream: the reference gen_dataset
    restatement, or (c4) the multi-slot generator (no reference one exists)."""
    import paper_2003_05622_b200 as pkg
    if c.get("gen") == "multislot":
        return pkg.gen_multislot(n, slots=100, ids_per_slot=c["dims"] // 100,
                                 max_keys=c["nnz"], seed=seed)
    return pkg.gen_dataset(c["dims"], n, c["nnz"], zipf=c["zipf"], seed=seed)


def run_reference_hot_path(cfgname, steps, warmup, threads, budget_s=60.0):
    """The reference's own HBM-PS hot path (oracle/_ref, the unmodified
    headers): one std::thread per simulated device running the device-worker
    loop (pipeline.hpp:504-566). Returns (examples/s, seconds, batches run)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from native import RefHotPath, RefLib, make_cfg

    c = CONFIGS[cfgname]
    ref = RefLib()
    pool = max(1, min(steps + warmup, 4))
    if c.get("gen") == "multislot":
        off, keys, lab = make_data(c, pool * c["B"])
    else:
        off, keys, lab = ref.gen_dataset(c["dims"], pool * c["B"], c["nnz"], c["zipf"])
    cfg = make_cfg(1, threads, c["E"], c["layers"], J=c["J"], det=True)
    hp = RefHotPath(ref, cfg, c["B"], off, keys, lab)
    if warmup:
        hp.run(0, warmup)
    # bounded sample: full batches until `steps` are done or ~budget_s elapsed
    ms, done = 0.0, 0
    while done < steps and (done < 2 or ms < budget_s * 1e3):
        ms += hp.run(warmup + done, 1)
        done += 1
    hp.close()
    return done * c["B"] / (ms / 1e3), ms / 1e3, done


def config_of(c, args) -> dict:
    """The `config` object both arms print (same keys)."""
    return {"workload": c["text"], "dims": c["dims"], "E": c["E"], "global_batch": c["B"],
            "nnz": c["nnz"], "zipf": c["zipf"], "J": c["J"], "layers": list(c["layers"]),
            "optimizer": c.get("opt", "sgd")}


def reference_arm(args, rank):
    if rank != 0:
        return
    c = CONFIGS[args.config]
    threads = host_threads()
    value, secs, done = run_reference_hot_path(args.config, args.steps, min(args.warmup, 1),
                                               threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs * 1e3 / done, "steps_timed": done, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32 params / f64 math",
        "data": "synthetic (reference gen_dataset, seed 1)",
        "config": dict(config_of(c, args),
                       optimizer="sgd" if c.get("opt", "sgd") == "sgd" else
                                 "sgd (the reference has no Adagrad; its SGD hot path is timed)",
                       parallelism=f"reference CPU hot path: {threads} simulated devices "
                                   f"(one std::thread each, the reference concurrency model; "
                                   f"the batch is sharded over them)"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{done} batches x {c['B']} examples (of {args.steps} "
                                   f"requested; stops after ~60 s) after 1 warm-up batch, "
                                   f"{threads} simulated devices (one std::thread each), "
                                   f"deterministic sync"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ------------------------------------------------------------------- ours --

NVLINK_GBS = 900.0  # NVLink 5 per GPU per direction (spec; not measured on this pool)


def remote_unique_keys(batches, D, J):
    """Unique keys per (device, mini-batch) shard whose owner is another rank,
    summed over shards and over the batch pool: what the key/row/delta
    all-to-alls carry. Shards follow shard_batch (sharding.hpp:29-42): example
    i -> device (i % (D*J)) / J, mini-batch (i % (D*J)) % J; owner key % D
    (topology.hpp:61-65)."""
    import numpy as np
    total = 0
    S = D * J
    for o, k, _ in batches:
        nex = o.size - 1
        ex = np.repeat(np.arange(nex, dtype=np.uint64), np.diff(o).astype(np.int64))
        shard = ex % np.uint64(S)
        ku = k.view(np.uint64)
        u = np.sort(ku * np.uint64(S) + shard)
        u = u[np.concatenate(([True], u[1:] != u[:-1]))]
        ukey, ush = u // np.uint64(S), u % np.uint64(S)
        total += int(np.count_nonzero(ukey % np.uint64(D) != ush // np.uint64(J)))
    return float(total)


def trace(msg):
    if os.environ.get("HPS_BENCH_TRACE"):
        print(f"[bench {os.environ.get('RANK', '0')} {time.time():.1f}] {msg}", file=sys.stderr,
              flush=True)


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2003_05622_b200 as pkg

    c = CONFIGS[args.config]
    dims, E, B, nnz, J = c["dims"], c["E"], c["B"], c["nnz"], c["J"]
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)

    # batch pool (identical on every rank: the node's batch stream)
    P = args.pool
    off, keys, lab = make_data(c, P * B)
    batches = []
    for b in range(P):
        o = (off[b * B:(b + 1) * B + 1] - off[b * B]).astype(np.int64)
        batches.append((o, keys[off[b * B]:off[(b + 1) * B]], lab[b * B:(b + 1) * B]))
    max_keys = max(int(b[0][-1]) for b in batches)

    nccl_id = None
    if world > 1:
        obj = [pkg.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    tier = pkg.Tier(nodes=1, devices=world, rank=rank, cuda_device=local_rank, width=E,
                    layer_dims=c["layers"], minibatches=J, deterministic=args.det,
                    key_space=dims, max_batch_examples=B, max_batch_keys=max_keys,
                    nccl_id=nccl_id, optimizer=c.get("opt", "sgd"))
    RW = tier.row_width  # floats per table / store row (2E with the Adagrad state)
    stream = torch.cuda.ExternalStream(tier.stream(), device=dev)
    trace("tier created")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    LAG = 3  # waits trail submits by three: four batches in flight
    last_flush_ms = [0.0]

    def timed_steps(submit_fn, n_steps, first):  # noqa: C901
        """Returns (event ms over the whole run of n_steps, per-step stats).

        One region, not per-step brackets: steps are pipelined through the
        public API (hps_submit_batch / hps_wait_batch: batch b+1 is staged and
        its table built while b trains, b's write-back overlaps b+1; every
        step's loss is read back), and the run ends with tier.flush() inside
        the events. No L2 flush between steps: the per-step inputs (a pool of
        batches cycled round-robin, the value store and the tables) exceed L2."""
        stats = []
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(n_steps):
            submit_fn((first + i) % P)
            if i >= LAG:
                stats.append(tier.wait_batch())
            if i < 8 or i % 50 == 0:
                trace(f"step {i} submitted")
        while len(stats) < n_steps:
            stats.append(tier.wait_batch())
        ef = torch.cuda.Event(enable_timing=True)
        ef.record(stream)
        tier.flush()
        e1.record(stream)
        e1.synchronize()
        last_flush_ms[0] = ef.elapsed_time(e1)  # (inside the region; reported too)
        return e0.elapsed_time(e1), stats

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---------------- device-resident (value) ----------------
    dbatches = []
    for o, k, l in batches:
        dbatches.append((torch.from_numpy(o).to(dev), torch.from_numpy(k.view(np.int64)).to(dev),
                         torch.from_numpy(l).to(dev)))
    dstore = torch.zeros((dims, RW), dtype=torch.float32, device=dev)
    tier.attach_store(dstore.data_ptr(), on_device=True, num_keys=dims)

    def dev_step(b):
        o, k, l = dbatches[b]
        return tier.submit_batch((o.data_ptr(), B), k.data_ptr(), l.data_ptr(), on_device=True)

    for i in range(args.warmup):
        dev_step(i % P)
        trace(f"warmup submit {i}")
    for i in range(args.warmup):
        tier.wait_batch()
    trace("warmup done")
    barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    clocks.wait_first()  # the sampler is live before the region opens
    launches0 = tier.kernel_launches()
    captures0 = tier.graph_captures()
    barrier()
    dev_ms, dev_stats = timed_steps(dev_step, args.steps, args.warmup)
    trace("timed value pass done")
    barrier()
    launches = tier.kernel_launches() - launches0
    captures = tier.graph_captures() - captures0
    clk = clocks.stop()
    dev_ms_max = max_over_ranks(dev_ms)
    value = args.steps * B / (dev_ms_max / 1e3)
    # second timed pass with per-phase CUDA events inside the captured graph
    # (the event nodes cost ~10%, so the headline above is taken without them)
    tier.set_timing(True)
    for i in range(5):  # one rotation: the timing-mode graphs captured
        dev_step(i % P)
        tier.wait_batch()
    tier.reset_timing()
    barrier()
    ph_steps = max(10, args.steps // 4)
    _, ph_stats = timed_steps(dev_step, ph_steps, args.warmup)
    barrier()
    phases = tier.timing()
    trace("timing pass done")
    tier.set_timing(False)

    # per-rank work counters over the phase-timing pass
    pulled = sum(s.pulled_keys for s in ph_stats)
    ws = sum(s.working_set for s in ph_stats)
    occ = sum(s.occurrences for s in ph_stats)
    n_ex = sum(s.examples for s in ph_stats)
    big_keys = sum(s.big_segments for s in ph_stats)
    big_occ = sum(s.big_occurrences for s in ph_stats)
    fallbacks = sum(s.exact_fallbacks for s in dev_stats)
    carried = sum(s.carried_rows for s in dev_stats) / args.steps
    loss = sum(s.loss_sum for s in dev_stats) / max(1, sum(s.examples for s in dev_stats))

    # ---------------- end to end through the C ABI, host buffers (e2e) -------
    e2e = None
    if not args.no_e2e:
        hstore_t = torch.zeros((dims, RW), dtype=torch.float32).pin_memory()
        hstore = hstore_t.numpy()
        tier.attach_store(hstore)
        hbatches = []
        for o, k, l in batches:
            hbatches.append(tuple(torch.from_numpy(x).pin_memory().numpy()
                                  for x in (o, k.view(np.int64), l)))

        def host_step(b):
            o, k, l = hbatches[b]
            return tier.submit_batch(o, k.view(np.uint64), l, on_device=False)

        for i in range(args.warmup):
            host_step(i % P)
        for i in range(args.warmup):
            tier.wait_batch()
        tier.flush()
        barrier()
        rd0, wr0 = tier.store_traffic()
        ph0, pd0 = tier.store_pcie_bytes()
        e2e_ms, e2e_stats = timed_steps(host_step, args.steps, args.warmup)
        barrier()
        rd1, wr1 = tier.store_traffic()
        ph1, pd1 = tier.store_pcie_bytes()
        e2e_ms_max = max_over_ranks(e2e_ms)
        mode = tier.store_mode()
        h2d = sum(8 * (b[0].size) + 8 * b[1].size + b[2].size for b in
                  (hbatches[(args.warmup + i) % P] for i in range(args.steps))) / args.steps
        h2d += (ph1 - ph0) / args.steps                    # store bytes over PCIe
        d2h = ((pd1 - pd0) + 24 * args.steps) / args.steps  # written back + stats
        if mode == "host-mirrored":
            # the store trains in HBM; the host array is made exact by the
            # flush that closes the timed region (its dirty pages copied back)
            path = ("hps_submit_batch/hps_wait_batch(on_device=0): pinned batch H2D on the "
                    "staging stream, loss D2H every step; the pinned host value store "
                    "(MEM-PS stand-in) is mirrored in HBM (it fits the 2 GB budget: "
                    f"{dims * RW * 4 / 1e9:.2f} GB) and its dirty 1024-row pages are copied "
                    "back to the host by the hps_flush inside the timed region")
        else:
            path = ("hps_submit_batch/hps_wait_batch(on_device=0): pinned batch H2D on "
                    "the staging stream, store rows prefetched (zero-copy) beside the "
                    "previous batch, deferred zero-copy write-back to the pinned host "
                    "store, loss D2H every step")
        e2e = {"value": args.steps * B / (e2e_ms_max / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(sum_over_ranks(h2d)),
               "d2h_bytes_per_step": int(sum_over_ranks(d2h)),
               "ms_per_step": e2e_ms_max / args.steps, "store": mode,
               "final_flush_ms": last_flush_ms[0], "path": path}
        tier.attach_store(None)
        del hstore_t

    # ---------------- roofline of the dominant phase --------------------------
    # Algorithmic bytes follow SURVEY 8(d), counted from the
    # batch stats of the phase-timing pass, over that pass's phase times:
    #   sparse (a8-a11 at one rank: segment-reduce + sgd_delta + in-place apply)
    #     = U*(4+12E)  push/SGD apply per unique key (slot, delta, row r+w)
    #     + U*4 + O*4  CSR grouping (segment bounds, example ids)
    #     + n_ex*8E    each example's f64 dL/dx record, read once
    #   big_fused_kernel alone (the long segments, on its own stream):
    #     U_big*(8+12E) + O_big*4 + min(n_ex, O_big)*8E
    peak, peak_kind = load_peaks()
    K = ph_steps
    mbs = K * J
    per_key_pull = 8 + 8 + 4 * E + 4 * E   # key + slot probe + row read + row write
    # push apply: slot + delta read + row read + row write; Adagrad reads and
    # writes the state with the row (4 + 4E + 8E + 8E)
    per_key_apply = 4 + 12 * E if RW == E else 4 + 20 * E
    per_key_build = 8 + 8 + 4 * RW + 4 * RW
    fused_apply = world == 1 and os.environ.get("HPS_DEDUP", "hash") != "sort"
    sparse_bytes = pulled * (per_key_apply + 4) + occ * 4 + n_ex * 8 * E
    big_bytes = big_keys * (per_key_apply + 4) + big_occ * 4 + min(n_ex, big_occ) * 8 * E
    phase_bytes = {
        "sparse": sparse_bytes,
        "big_fused": big_bytes,
        "pull": pulled * per_key_pull,
        "apply": pulled * per_key_apply,
        "build": ws * per_key_build,
        "writeback": ws * (8 + 4 + 4 * RW + 4 * RW),
        "dedup": 12 * occ + 8 * pulled,
    }
    if fused_apply:
        # G = 1: fwd/bwd reads the rows in place from the table (a6 fused) and
        # the sparse reduce applies the deltas in place (a10/a11 fused), so
        # there is no pull or apply kernel to put on the roofline
        phase_bytes.pop("pull")
        phase_bytes.pop("apply")
    rl = {}
    for name, nbytes in phase_bytes.items():
        ms = phases.get(name, 0.0)
        if ms > 0:
            gbs = nbytes / (ms / 1e3) / 1e9
            rl[name] = {"ms_per_step": ms / K, "algorithmic_bytes_per_step": nbytes / K,
                        "achieved_gbs": gbs, "frac": gbs / peak}
    traffic = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(args.config, {})
        except Exception:
            traffic = {}

    def traffic_of(name, per_launch_bytes):
        t = traffic.get(name)
        return (t, t / per_launch_bytes if t and per_launch_bytes else None)

    sp = rl.get("sparse", {})
    sp_launch = sparse_bytes / mbs
    t_sp, r_sp = traffic_of("sparse", sp_launch)
    bf = rl.get("big_fused", {})
    bf_launch = big_bytes / mbs
    t_bf, r_bf = traffic_of("big_fused", bf_launch)
    roofline = {
        "bound": "hbm",
        "kernel": "sparse segment-reduce + sgd_delta" + (" + in-place apply" if fused_apply
                                                         else "") +
                  " per mini-batch (sparse_short_kernel on the body stream; big_classify, "
                  "big_plan, big_fused_kernel on a side stream)",
        "achieved": sp.get("achieved_gbs"), "peak": peak, "unit": "GB/s", "frac": sp.get("frac"),
        "traffic": t_sp, "traffic_over_algorithmic": r_sp, "peak_kind": peak_kind,
        "algorithmic_bytes_per_launch": sp_launch,
        "ms_per_launch": sp.get("ms_per_step", 0.0) * K / mbs if sp else None,
        "bytes_model": ("U*(4+12E)" if RW == E else "U*(4+20E)") +
                       " + U*4 + O*4 + n_ex*8E per mini-batch (SURVEY 8(d) push/" +
                       ("SGD" if RW == E else "Adagrad") +
                       " apply + CSR + one f64 dL/dx record per example)",
        "launches_per_step": J,
        "kernels": {
            "big_fused_kernel": {
                "achieved": bf.get("achieved_gbs"), "frac": bf.get("frac"),
                "algorithmic_bytes_per_launch": bf_launch,
                "ms_per_launch": bf.get("ms_per_step", 0.0) * K / mbs if bf else None,
                "traffic": t_bf, "traffic_over_algorithmic": r_bf,
                "bytes_model": ("U_big*(8+12E)" if RW == E else "U_big*(8+20E)") +
                               " + O_big*4 + min(n_ex, O_big)*8E",
                "segments_per_launch": big_keys / mbs, "occurrences_per_launch": big_occ / mbs,
                "timed": "CUDA events on its own stream around each launch"}},
        "phases": rl}

    # ---------------- NVLink roofline of the key/row/delta all-to-alls (N>1) --
    nvlink = None
    if world > 1:
        remote = remote_unique_keys(batches, world, J) / P   # per step, all ranks
        xfer_ms = max_over_ranks(phases.get("pull", 0.0) + phases.get("apply", 0.0)) / K
        per_gpu = remote * (8 + 4 * E + 4 * E) / world        # sent by one GPU per step
        if xfer_ms > 0:
            gbs = per_gpu / (xfer_ms / 1e3) / 1e9
            nvlink = {"bound": "nvlink", "achieved": gbs, "peak": NVLINK_GBS, "unit": "GB/s",
                      "frac": gbs / NVLINK_GBS, "peak_kind": "spec (NVLink 5, per GPU per "
                      "direction)", "bytes_model": "remote unique keys x (8 key + 4E row + 4E "
                      "delta) / N, per GPU per direction",
                      "remote_keys_per_step": remote, "bytes_per_gpu_per_step": per_gpu,
                      "ms_per_step": xfer_ms,
                      "phases": "pull (key a2a, owner probe+gather, row a2a) + apply (delta "
                                "a2a, canonical apply): the time includes the owner-side work "
                                "and the flag waits, so the link rate is a lower bound"}

    # ---------------- CPU baseline (reference hot path, rank 0, N=1) ---------
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        threads = host_threads()
        try:
            v, secs, _ = run_reference_hot_path(args.config, 2, 1, threads)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"2 batches x {B} examples of {args.config} after 1 warm-up "
                             f"batch; reference HbmTier device-worker loop, {threads} "
                             f"simulated devices (std::threads), flat-map host store",
                   "seconds": secs}
        except Exception as ex:  # the reference library is prebuilt here
            cpu = {"value": None, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    # (collectives: every rank calls them, in this order)
    all_launch = int(sum_over_ranks(launches))
    captures_all = int(sum_over_ranks(captures))
    fallbacks_all = int(sum_over_ranks(fallbacks))
    # keys/s per phase: pull = the phases that deliver a
    # mini-batch's unique rows to the model (G = 1: fwd/bwd reads them in
    # place; G > 1: key all-to-all + owner gather + row all-to-all); push = the
    # phases that reduce and apply their gradients (G = 1: the fused sparse
    # reduce + in-place apply; G > 1: + delta all-to-all + canonical apply)
    pull_ms = phases.get("fwdbwd", 0.0) if fused_apply else (phases.get("dedup", 0.0) +
                                                              phases.get("pull", 0.0))
    push_ms = phases.get("sparse", 0.0) + (0.0 if fused_apply else phases.get("apply", 0.0))
    keys_all = sum_over_ranks(pulled)
    pull_ms, push_ms = max_over_ranks(pull_ms), max_over_ranks(push_ms)
    pull_keys_s = keys_all / (pull_ms / 1e3) if pull_ms else None
    push_keys_s = keys_all / (push_ms / 1e3) if push_ms else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 params / f64 math",
            "data": "synthetic (reference gen_dataset stream, seed 1; random-init dense)",
            "config": dict(config_of(c, args), **{
                       "parallelism": f"key-sharded x{world}", "batch_pool": P,
                       "deterministic": bool(args.det),
                       "l2": (f"not flushed; per-step inputs exceed L2: {P} batches x "
                              f"{max_keys * 8 >> 20} MiB keys cycled, {dims * E * 4 >> 20} MiB "
                              "value store, 5 tables; steps pipelined (write-back of b "
                              "overlaps b+1), one event region ending in hps_flush")}),
            "e2e": e2e,
            "roofline": roofline,
            "nvlink": nvlink,
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": all_launch,
            "graph_captures_in_timed_region": captures_all,
            "exact_fallbacks": fallbacks_all,
            "pull_keys_per_s": pull_keys_s,
            "push_keys_per_s": push_keys_s,
            "keys_per_s_phases": {"pull": "fwdbwd (rows read in place)" if fused_apply else
                                  "dedup + pull", "push": "sparse (reduce + in-place apply)" if
                                  fused_apply else "sparse + apply"},
            "phase_ms_per_step": {k: v / K for k, v in phases.items()},
            "train_loss": loss,
            "carried_rows_per_step": carried,
            "working_set_per_step": ws / K,
            "phase_steps": K,
        }
        emit(line)
    tier.close()


_JSON_FD = None


def emit(line: dict) -> None:
    """Print the one JSON line on the real stdout (library/NCCL banners are
    routed to stderr for the whole run)."""
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _JSON_FD
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)  # anything else written to stdout goes to stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10,
                    help="untimed steps (>= 4: the first steady-state batch of a shape "
                         "captures the graphs of every table rotation)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--pool", type=int, default=16, help="distinct batches cycled")
    ap.add_argument("--det", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)

    if args.impl == "reference":
        reference_arm(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
