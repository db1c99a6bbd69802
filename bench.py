#!/usr/bin/env python3
"""Benchmark: simulated queries/sec of the replay engine (BASELINE.json metric).

One step = one kvr_sim_run_multi launch over the whole workload of this rank:
config 2 of BASELINE.json (W=8 workers, B=512 blocks, three 100k-query GSP traces
with low / medium / high shared-prefix ratio 0.3/0.5/0.9, LBGR routing, RLT vs
Leaf-LRU eviction) with 1,024 replays per GPU (weak scaling: every rank runs its
own 1,024 trials; trial keys differ per rank).  Unit of work: one query in one
replay ("query-replay").

  python bench.py [--gpus N --steps K --warmup W] [--impl kvr|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.  ``--impl reference`` times the CPU oracle (the
tier's reference arm) on host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2601_18999_b200 import workloads as wl  # noqa: E402

W_WORKERS, B_BLOCKS = 8, 512
RATIOS = (0.3, 0.5, 0.9)
N_QUERIES = 100_000
TRIALS_PER_GPU = 1024
GSP_GROUPS, GSP_PER_GROUP = 125, 800           # 125 x 800 = 100k queries per trace
GSP_LENGTHS = (128, 256, 512, 1024, 2048)      # paper's {512..8192} tokens / 4
UTIL = 0.4                                     # all-miss utilisation of the Poisson arrivals
RING = 16384                                   # pending-completion FIFO per worker
TRACE_SEEDS = (0xC2, 0xC3, 0xC4)
METRIC = "simulated queries/sec (all replays)"
UNIT = "query-replays/s"


def build_traces(n_queries=N_QUERIES):
    trs = []
    for r, s in zip(RATIOS, TRACE_SEEDS):
        per = max(1, n_queries // GSP_GROUPS)
        trs.append(wl.gsp(GSP_GROUPS, per, r, seed=s, W=W_WORKERS, util=UTIL, lengths=GSP_LENGTHS))
    return trs


# (trace index, eviction) classes, slowest first (scripts/trial_cost.py).
# The persistent kernel hands trials out in index order, so with contiguous class
# blocks the partial last wave is filled by the cheapest trials (LPT list scheduling).
CLASS_ORDER = ((0, 1), (1, 1), (2, 1), (0, 0), (1, 0), (2, 0))     # eviction 1 = RLT, 0 = LRU


def trial_plan(rank, n_trials=TRIALS_PER_GPU):
    """trial t -> class CLASS_ORDER[6t div n] (equal contiguous blocks); keys unique per rank."""
    t = np.arange(n_trials)
    cls = np.array(CLASS_ORDER, dtype=np.uint32)[(t * len(CLASS_ORDER)) // max(n_trials, 1)]
    trace_of = cls[:, 0].copy()
    evict = cls[:, 1].copy()
    keys = (np.uint64(rank) * np.uint64(1 << 32) + t.astype(np.uint64) + np.uint64(1))
    return trace_of, evict, keys


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace('.', '', 1).isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace('.', '', 1).isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def algorithmic_bytes(res):
    """SURVEY §8(d) / DESIGN.md §6: algorithmic shared-memory bytes (probe 10 B, insert 22 B,
    evict 14 B) and trace bytes (8 B per block + 24 B per query) of a set of trial results."""
    probes = float(res["probes"].sum())
    ins = float(res["inserted_blocks"].sum())
    ev = float(res["evictions"].sum())
    smem = 10.0 * probes + 22.0 * ins + 14.0 * ev
    return smem


def trace_bytes(traces, trace_of):
    per = np.array([8.0 * t.total_blocks + 24.0 * t.n_queries for t in traces])
    return float(per[trace_of].sum())


def peaks():
    p = {"hbm_gbs": 6452.8, "sm_max_mhz": 1965.0, "src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({"hbm_gbs": float(m["hbm_gbs"]), "sm_max_mhz": float(m["sm_max_mhz"]),
                  "src": "measured"})
    except Exception:
        pass
    return p


def run_oracle_sample(traces, trace_of, evict, keys, n_prefix, threads, beta=0):
    """CPU oracle (as it stands) on host cores: `threads` trials, each on the first
    n_prefix queries of its trace.  Returns (query-replays, seconds, threads)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    cfg = oracle.OracleConfig(W=W_WORKERS, capacity_blocks=B_BLOCKS, pending_ring=RING,
                              batch_slots=beta)
    prefixes = [t.prefix(n_prefix) for t in traces]

    def one(i):
        pol = oracle.OraclePolicy(eviction=int(evict[i]))
        r = oracle.run(cfg, prefixes[int(trace_of[i])], pol, int(keys[i]))
        return r.result["queries"]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:   # ctypes releases the GIL
        q = sum(ex.map(one, range(threads)))
    return q, time.perf_counter() - t0


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def reference_arm(args, rank, world):
    if rank != 0:
        return
    import oracle
    oracle.build_oracle()
    traces = build_traces()
    trace_of, evict, keys = trial_plan(0)
    threads = max(1, min(os.cpu_count() or 1, 16))
    n_prefix = args.ref_queries
    for _ in range(args.warmup):
        run_oracle_sample(traces, trace_of, evict, keys, max(50, n_prefix // 10), threads,
                          args.batch_slots)
    tot_q, tot_s = 0, 0.0
    for _ in range(args.steps):
        q, s = run_oracle_sample(traces, trace_of, evict, keys, n_prefix, threads, args.batch_slots)
        tot_q += q
        tot_s += s
    v = tot_q / tot_s
    sample = (f"{threads} oracle trials x first {n_prefix} queries of the config-2 traces "
              f"per step (W=8, B=512, LBGR, RLT/LRU)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_s / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_json(args),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_json(args):
    beta = getattr(args, "batch_slots", 0)
    extra = (f", continuous batching beta={beta} (SURVEY 8f #2, update at dequeue)" if beta else "")
    return {"workload": "config2: W=8, B=512 blocks, 3 GSP traces (125 groups x 800 queries, "
                        "128-2048 tokens, prefix ratio 0.3/0.5/0.9), LBGR x {RLT, L-LRU}" + extra,
            "replays_per_gpu": TRIALS_PER_GPU, "queries_per_trace": N_QUERIES,
            "block_tokens": 16, "parallelism": f"replica-sharded x{args.gpus}",
            "l2": "inputs larger than L2 (3 packed traces ~250 MB) + 256 MB L2 flush between steps"}


NCU_CAPTURE = os.path.join(ROOT, "profiles", "r1_bench_replay_ncu.json")


def ncu_capture(args):
    """DRAM traffic per launch of the replay kernel from the committed `ncu --set full`
    capture of this exact launch (scripts/profile_bench.sh); None for other sizes."""
    if (args.queries != N_QUERIES or args.trials != TRIALS_PER_GPU or args.batch_slots
            or not os.path.exists(NCU_CAPTURE)):
        return None
    with open(NCU_CAPTURE) as f:
        d = json.load(f)
    d["src"] = os.path.relpath(NCU_CAPTURE, ROOT) + " (ncu --set full, one launch)"
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kvr", choices=["kvr", "reference"])
    ap.add_argument("--ref-queries", type=int, default=15000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--queries", type=int, default=N_QUERIES, help=argparse.SUPPRESS)
    ap.add_argument("--trials", type=int, default=TRIALS_PER_GPU, help=argparse.SUPPRESS)
    ap.add_argument("--batch-slots", type=int, default=0,
                    help="0: the beta = 1 model (default, the headline); 1..3: the continuous-"
                         "batching engine with beta slots per worker (beta * 129 <= B = 512)")
    ap.add_argument("--ncu", action="store_true",
                    help="profiling run: one launch, no warm-up / e2e / cpu baseline")
    args = ap.parse_args()
    if args.ncu:
        args.warmup, args.steps, args.no_e2e, args.no_cpu_baseline = 0, 1, True, True
    else:
        args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2601_18999_b200.kvr import DeviceTrace, Policy, Simulator, policies_array

    # KVR_BENCH_BACKEND=gloo (tests only): several ranks on one GPU, collectives staged
    # through host copies; the contract run uses NCCL, one rank per GPU
    backend = os.environ.get("KVR_BENCH_BACKEND", "nccl")
    if backend == "gloo":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def coll(fn, t, **kw):
        if backend != "gloo":
            return fn(t, **kw)
        h = t.cpu()
        fn(h, **kw)
        t.copy_(h)

    traces = build_traces(args.queries)
    trace_of, evict, keys = trial_plan(rank, args.trials)
    n_trials = len(keys)
    pols = policies_array([Policy(eviction=int(e)) for e in evict])
    stream = torch.cuda.current_stream()
    dts = [DeviceTrace(t, device=dev) for t in traces]
    sim = Simulator(W_WORKERS, B_BLOCKS, pending_ring=RING, batch_slots=args.batch_slots)
    buf = sim.alloc(dts, n_trials, 0, dev)
    buf["keys"].copy_(torch.from_numpy(keys.view(np.int64)))
    buf["policies"].copy_(torch.from_numpy(pols.view(np.uint8)))
    buf["trial_trace"].copy_(torch.from_numpy(trace_of.view(np.int32)))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # every rank packs the same traces; their identity checksum rides in the reduce
    trace_hash = sum(d.identity_digest() for d in dts) & 0xFFFFFFFFFFFFFFFF
    trace_hash = trace_hash - (1 << 64) if trace_hash >= (1 << 63) else trace_hash
    from paper_2601_18999_b200 import dist as kdist
    summary = [None]

    def step(timed_ms):
        flush.fill_(1)                                     # L2 flush, outside the timed region
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.launch(dts, n_trials, buf, with_policies=True, stream=stream)
        if world > 1:   # the single NCCL reduce of summary counters
            vec = kdist.summary_tensor(buf["results"], n_trials, trace_hash)
            coll(dist.reduce, vec, dst=0)
            summary[0] = vec
        e1.record(stream)
        torch.cuda.synchronize()
        timed_ms.append(e0.elapsed_time(e1))

    warm = []
    for _ in range(args.warmup):
        step(warm)
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            step(times)
    res = sim.collect(buf, n_trials).results
    bad = int((res["status"] != 0).sum())
    t_local = float(np.sum(times))
    tmax = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        coll(dist.all_reduce, tmax, op=dist.ReduceOp.MAX)
    t_max = float(tmax.item())
    q_per_step = float(res["queries"].sum())
    if world > 1 and summary[0] is not None:   # all ranks' queries and failed trials
        red = summary[0].cpu().tolist()
        q_per_step, bad = float(red[1]), int(red[11])
    else:
        q_per_step *= world
    total_q = q_per_step * args.steps
    value = total_q / (t_max / 1000.0)

    # roofline of the dominant kernel (the replay kernel is the whole step)
    pk = peaks()
    prof = ncu_capture(args)
    clk_s = clk.summary()
    f_mhz = clk_s["sm_mhz"] or pk["sm_max_mhz"]
    smem_peak = 148 * 128 * pk["sm_max_mhz"] * 1e6 / 1e9        # GB/s at max clock
    smem_bytes = algorithmic_bytes(res)
    per_launch_s = (t_local / args.steps) / 1000.0
    achieved_smem = smem_bytes / per_launch_s / 1e9
    tb = trace_bytes(traces, trace_of)
    achieved_hbm = tb / per_launch_s / 1e9
    probes = float(res["probes"].sum())

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64+u64", "data": "synthetic",
            "config": config_json(args),
            "roofline": {"bound": "smem", "achieved": achieved_smem, "peak": smem_peak,
                         "unit": "GB/s", "frac": achieved_smem / smem_peak,
                         "traffic": prof.get("traffic_bytes_per_launch") if prof else None,
                         "traffic_src": prof.get("src") if prof else None,
                         "smem_actual_frac_ncu": prof.get("smem_actual_frac_of_peak") if prof else None,
                         "peak_src": "148 SM x 128 B/clk x sm_max_mhz (DESIGN.md §6)",
                         "hbm_trace": {"achieved": achieved_hbm, "peak": pk["hbm_gbs"],
                                       "frac": achieved_hbm / pk["hbm_gbs"],
                                       "peak_src": pk["src"]}},
            "prefix_probes_per_s": probes * world / per_launch_s,
            "hit_rate": float(res["hit_tokens"].sum() / max(1, res["input_tokens"].sum())),
            "trial_status_nonzero": bad,
            "gpu_launches": args.steps * 1,
            "clocks": clk_s}

    if world > 1 and rank == 0 and summary[0] is not None:
        line["reduced_summary"] = dict(zip(kdist.SUMMARY_FIELDS,
                                           [int(x) for x in summary[0].cpu().tolist()]))
        # sum over ranks of identical checksums = world x rank 0's (mod 2^64)
        line["reduced_summary"]["trace_hash_consistent"] = (
            (line["reduced_summary"]["trace_hash"] - world * trace_hash) % (1 << 64) == 0)
    if not args.no_e2e:
        # every rank runs its own trials end to end; the job's rate is all ranks'
        # queries over the slowest rank's time (max over ranks, like `value`)
        if world > 1:
            dist.barrier()
        e = e2e_measure(traces, trace_of, evict, keys, pols, dev, stream, args)
        if world > 1:
            t = torch.tensor([e["ms_per_step"]], dtype=torch.float64, device=dev)
            coll(dist.all_reduce, t, op=dist.ReduceOp.MAX)
            c = torch.tensor([e["queries_per_step"], e["h2d_bytes_per_step"], e["d2h_bytes_per_step"]],
                             dtype=torch.float64, device=dev)
            coll(dist.all_reduce, c, op=dist.ReduceOp.SUM)
            e["ms_per_step"] = float(t[0])
            e["queries_per_step"], e["h2d_bytes_per_step"], e["d2h_bytes_per_step"] = \
                float(c[0]), int(c[1]), int(c[2])
            e["value"] = e["queries_per_step"] / (e["ms_per_step"] / 1000.0)
        if rank == 0:
            line["e2e"] = e
    if rank == 0 and not args.no_cpu_baseline:
        threads = max(1, min(os.cpu_count() or 1, 16))
        nq = args.ref_queries
        q, s = run_oracle_sample(traces, trace_of, evict, keys, nq, threads, args.batch_slots)
        q1, s1 = run_oracle_sample(traces, trace_of, evict, keys, nq, 1,
                                   args.batch_slots)   # one core
        line["cpu_baseline"] = {"value": q / s, "unit": UNIT, "cores": threads, "kind": "oracle",
                                "single_core_value": q1 / s1, "nproc": os.cpu_count(),
                                "cpu_model": cpu_model(),
                                "sample": f"{threads} trials x first {nq} queries of the "
                                          f"config-2 traces (W=8, B=512); single core: 1 trial"}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def e2e_measure(traces, trace_of, evict, keys, pols, dev, stream, args):  # noqa: C901
    """Same metric through the public API with HOST buffers: per step the pinned raw
    traces, keys, policies and trial->trace map go host->device, kvr_trace_load packs
    (validates, chains) them, kvr_sim_run_multi replays, and the per-trial results come
    back device->host into pinned memory, all inside the timed region."""
    import torch
    from paper_2601_18999_b200.kvr import DeviceTrace, Simulator

    sim = Simulator(W_WORKERS, B_BLOCKS, pending_ring=RING, batch_slots=args.batch_slots)
    n = len(keys)
    host = [DeviceTrace.pin(t) for t in traces]                     # pinned, outside timing
    h_keys = torch.from_numpy(keys.view(np.int64)).pin_memory()
    h_pols = torch.from_numpy(pols.view(np.uint8)).pin_memory()
    h_tt = torch.from_numpy(trace_of.view(np.int32)).pin_memory()
    h_res = torch.empty(n * 144, dtype=torch.uint8).pin_memory()
    h2d = sum(int(v.numel() * v.element_size()) for hd in host for v in hd.values())
    h2d += int(h_keys.numel() * 8 + h_pols.numel() + h_tt.numel() * 4)
    d2h = n * 144
    times = []
    q = 0.0
    for it in range(2 + max(1, args.steps // 2)):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        dts = [DeviceTrace(t, device=dev, host=hd) for t, hd in zip(traces, host)]
        b = sim.alloc(dts, n, 0, dev)
        b["keys"].copy_(h_keys, non_blocking=True)
        b["policies"].copy_(h_pols, non_blocking=True)
        b["trial_trace"].copy_(h_tt, non_blocking=True)
        sim.launch(dts, n, b, with_policies=True, stream=stream)
        h_res.copy_(b["results"][: n * 144], non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
        from paper_2601_18999_b200.kvr import RESULT_DTYPE
        q = float(h_res.numpy().view(RESULT_DTYPE)["queries"].sum())
        for d in dts:
            d.close()
    ms = float(np.mean(times))
    return {"value": q / (ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms, "queries_per_step": q}


if __name__ == "__main__":
    main()
