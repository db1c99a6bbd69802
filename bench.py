#!/usr/bin/env python3
"""Benchmark: simulated queries/sec of the replay engine (BASELINE.json metric).

Default workload = BASELINE config 5, the largest replay sweep:
{GSP(128,32,r), MT-ShareGPT(128,r), MT-UltraChat(128,r), LD(512,Q_d)} x {low r=0.3 /
Q_d=2, med 0.5/8, high 0.9/32} x W in {4, 8, 16, 32}, B = 512, LBGR (App. A, reading
A8), RLT on even trial keys and Leaf-LRU on odd ones: 48 cells, ONE fixed list of
65,536 replays (trial t -> cell (48 t) div 65536, key t + 1).  With N ranks, rank r
runs the trials with (t div 2) mod N == r (strong scaling: the same list at every N;
pairs of keys keep RLT and Leaf-LRU mixed on every rank), one kvr_sim_run_multi per W
in longest-trace-first order.  A step ends with ONE NCCL reduce of the summary
counters.  Unit of work: one query in one replay ("query-replay").

``--workload c2`` runs BASELINE config 2 instead (W = 8, three 100k-query GSP traces,
1,024 replays per rank, weak scaling), the round-1 headline.

  python bench.py [--gpus N --steps K --warmup W] [--impl kvr|reference] [--workload c5|c2]
  torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.  ``--impl reference`` times the CPU oracle (the
tier's reference arm) on host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2601_18999_b200 import workloads as wl  # noqa: E402

METRIC = "simulated queries/sec (all replays)"
UNIT = "query-replays/s"
B_BLOCKS = 512
UTIL = 0.8                                     # all-miss utilisation of the Poisson arrivals
BATCH_SLOTS = [0]                              # --batch-slots (the oracle baseline follows it)

# ---- config 5 ----
C5_WS = (4, 8, 16, 32)
C5_SETTINGS = ((0.3, 2), (0.5, 8), (0.9, 32))  # (prefix ratio r, LD questions per doc Q_d)
C5_TRIALS = 65536
C5_KINDS = ("gsp", "mt-sharegpt", "mt-ultrachat", "ld")

# ---- config 2 ----
C2_W = 8
C2_RATIOS = (0.3, 0.5, 0.9)
C2_QUERIES = 100_000
C2_TRIALS = 1024
C2_GROUPS = 125
C2_LENGTHS = (128, 256, 512, 1024, 2048)      # paper's {512..8192} tokens / 4
C2_SEEDS = (0xC2, 0xC3, 0xC4)
C2_CLASS_ORDER = ((0, 1), (1, 1), (2, 1), (0, 0), (1, 0), (2, 0))   # slowest first (LPT)


# ------------------------------------------------------------------- workloads
class Launch:
    """One kvr_sim_run_multi: W workers, its traces, and this rank's trials on them."""

    def __init__(self, W, traces, tids, trial_trace, keys, evict):
        self.W, self.traces = W, traces
        self.tids = np.asarray(tids, np.int64)                   # global trial ids
        self.trial_trace = np.asarray(trial_trace, np.uint32)
        self.keys = np.asarray(keys, np.uint64)
        self.evict = np.asarray(evict, np.uint32)
        self.ring = max(t.n_queries for t in traces)             # never overflows (ABI v7 pool)

    def policies(self):
        from paper_2601_18999_b200.kvr import Policy, policies_array
        return policies_array([Policy(eviction=int(e)) for e in self.evict])

    def __len__(self):
        return len(self.keys)


def c5_traces(W):
    """The 12 traces of config 5 at W workers (seed 0xC7 + 16 si + W + kind)."""
    trs = []
    for si, (r, qd) in enumerate(C5_SETTINGS):
        seed = 0xC7 + 16 * si + W
        trs.append(wl.gsp(128, 32, r, seed=seed, W=W, util=UTIL))
        trs.append(wl.mt(128, r, seed=seed + 1, W=W, util=UTIL, name="mt-sharegpt"))
        trs.append(wl.mt(128, r, seed=seed + 2, W=W, util=UTIL, name="mt-ultrachat"))
        trs.append(wl.ld(512, qd, seed=seed + 3, W=W, util=UTIL))
    return trs


def c5_cell_of(n_trials):
    """trial t -> cell (48 t) div n: 48 cells of n/48 trials (1,365 / 1,366 at 65,536)."""
    return (np.arange(n_trials, dtype=np.int64) * 48) // n_trials


def c5_shard(n_trials, rank, world):
    """The fixed list's trials of `rank`: (t div 2) mod world == rank."""
    t = np.arange(n_trials, dtype=np.int64)
    return t[(t // 2) % world == rank]


def c5_plan(rank, world, n_trials=C5_TRIALS, traces=None):
    cell = c5_cell_of(n_trials)
    mine = c5_shard(n_trials, rank, world)
    launches = []
    for wi, W in enumerate(C5_WS):
        trs = traces[W] if traces is not None else c5_traces(W)
        nq = np.array([t.n_queries for t in trs])
        sel = mine[cell[mine] // 12 == wi]
        ti = cell[sel] % 12
        # longest trial first: the persistent kernel hands trials out in index order
        order = np.lexsort((sel, -nq[ti]))
        sel, ti = sel[order], ti[order]
        keys = (sel + 1).astype(np.uint64)
        launches.append(Launch(W, trs, sel, ti, keys, (keys % 2 == 0).astype(np.uint32)))
    return launches


def c2_traces(n_queries=C2_QUERIES):
    per = max(1, n_queries // C2_GROUPS)
    return [wl.gsp(C2_GROUPS, per, r, seed=s, W=C2_W, util=UTIL, lengths=C2_LENGTHS)
            for r, s in zip(C2_RATIOS, C2_SEEDS)]


def c2_plan(rank, world, n_trials=C2_TRIALS, traces=None, n_queries=C2_QUERIES):
    """Weak scaling: every rank runs its own n_trials (keys unique per rank)."""
    trs = traces if traces is not None else c2_traces(n_queries)
    trace_of, evict, keys = trial_plan(rank, n_trials)
    tids = rank * n_trials + np.arange(n_trials)
    return [Launch(C2_W, trs, tids, trace_of, keys, evict)]


# config-2 slices for the profiling scripts in scripts/ (phase_profile, ncu_case, trial_cost)
W_WORKERS, RATIOS, RING = C2_W, C2_RATIOS, 1 << 17


def build_traces(n_queries=C2_QUERIES):
    return c2_traces(n_queries)


def trial_plan(rank, n_trials=C2_TRIALS):
    """(trace index, eviction, key) of config 2's trials, slowest class first."""
    t = np.arange(n_trials)
    cls = np.array(C2_CLASS_ORDER, dtype=np.uint32)[(t * len(C2_CLASS_ORDER)) // max(n_trials, 1)]
    keys = np.uint64(rank) * np.uint64(1 << 32) + t.astype(np.uint64) + np.uint64(1)
    return cls[:, 0].copy(), cls[:, 1].copy(), keys


def make_plan(args, rank, world):
    if args.workload == "c5":
        return c5_plan(rank, world, args.trials or C5_TRIALS)
    return c2_plan(rank, world, args.trials or C2_TRIALS, n_queries=args.queries or C2_QUERIES)


def config_json(args):
    if args.workload == "c5":
        n = args.trials or C5_TRIALS
        return {"workload": "config5: {GSP(128,32,r), MT-ShareGPT(128,r), MT-UltraChat(128,r), "
                            "LD(512,Qd)} x {r=0.3/Qd=2, 0.5/8, 0.9/32} x W in {4,8,16,32}, B=512 "
                            "blocks, LBGR (App. A, mu=0.008), RLT on even keys / L-LRU on odd",
                "replays_total": n, "cells": 48, "block_tokens": 16, "util": UTIL,
                "sharding": f"fixed list of {n} trials, trial t on rank (t div 2) mod N",
                "parallelism": f"replica-sharded x{args.gpus}",
                "launches_per_step": 4,
                "l2": "256 MB L2 flush between steps (48 packed traces ~55 MB stay resident "
                      "within a step)"}
    return {"workload": "config2: W=8, B=512 blocks, 3 GSP traces (125 groups x 800 queries, "
                        "128-2048 tokens, prefix ratio 0.3/0.5/0.9), LBGR (mu=0.008) x {RLT, L-LRU}",
            "replays_per_gpu": args.trials or C2_TRIALS, "queries_per_trace": args.queries or C2_QUERIES,
            "batch_slots": args.batch_slots,
            "block_tokens": 16, "util": UTIL, "parallelism": f"replica-sharded x{args.gpus}",
            "l2": "inputs larger than L2 (3 packed traces ~250 MB) + 256 MB L2 flush between steps"}


# ----------------------------------------------------------------- measurement
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
    """SURVEY §8(d) / DESIGN.md §6: algorithmic shared-memory bytes of a set of trial
    results (probe 10 B, insert 22 B, evict 14 B)."""
    probes = float(res["probes"].sum())
    ins = float(res["inserted_blocks"].sum())
    ev = float(res["evictions"].sum())
    return 10.0 * probes + 22.0 * ins + 14.0 * ev


def trace_bytes(launches):
    tot = 0.0
    for L in launches:
        per = np.array([8.0 * t.total_blocks + 24.0 * t.n_queries for t in L.traces])
        tot += float(per[L.trial_trace].sum())
    return tot


# Dependent-latency floor of one query-replay ("latency roofline"):
# measured dependent-issue latencies on B200 (profiles/README.md, scripts/ubench_latency.cu):
# SHFL 37, CREDUX.MIN 22, VOTE+POPC 44, LDS 34, IMAD.HI 9, POPC 23 cycles.
#  * per query (every trial): the per-query barrier (~2 x LDS round trips, 70), the argmin
#    (3 CREDUX, 66), the chooser's hit walk (table LDS + key LDS + ballot, 34+34+27) and its
#    accounting store chain (~2 LDS/STS, 68): 300 cycles;
#  * per RLT eviction (the fast segment's loop-carried chain): IMAD.HI 9 -> CREDUX 22 ->
#    SHFL 37 -> POPC 23 -> CREDUX 22 -> SHFL 37 = 150 cycles;
#  * per Leaf-LRU eviction: one 32-entry window of the recency log per ballot, i.e.
#    (LDS 34 + VOTE+POPC 44) / 32 ~= 3 cycles.
LAT_QUERY, LAT_EVICT_RLT, LAT_EVICT_LRU = 300.0, 150.0, 3.0


def latency_floor_cycles(res, evict):
    """Critical-path floor in cycles summed over the trials (one serial chain each)."""
    q = res["queries"].astype(np.float64)
    ev = res["evictions"].astype(np.float64)
    per_ev = np.where(np.asarray(evict) == 1, LAT_EVICT_RLT, LAT_EVICT_LRU)
    return q * LAT_QUERY + ev * per_ev


def peaks():
    p = {"hbm_gbs": 6452.8, "sm_max_mhz": 1965.0, "src": "fallback (B200_PROFILING.md)"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({"hbm_gbs": float(m["hbm_gbs"]), "sm_max_mhz": float(m["sm_max_mhz"]),
                  "src": "measured (MEASURED_PEAKS.json)"})
    except Exception:
        pass
    return p


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ------------------------------------------------------------------ CPU oracle
def oracle_sample(args, launches, n_trials, prefix=None):
    """A bounded sample of this workload's trials for the CPU oracle: n_trials spread
    over the launches / cells (full trials for config 5, the first `prefix` queries of
    each trial for config 2).  Returns [(W, trace, eviction, key)]."""
    out = []
    allt = [(L, i) for L in launches for i in range(len(L))]
    if not allt:
        return out
    step = max(1, len(allt) // max(1, n_trials))
    for L, i in allt[::step][:n_trials]:
        tr = L.traces[int(L.trial_trace[i])]
        if prefix:
            tr = tr.prefix(prefix)
        out.append((L.W, tr, int(L.evict[i]), int(L.keys[i]), L.ring))
    return out


def run_oracle_sample(sample, threads):
    """The CPU oracle (as it stands) on host cores, one trial per task.
    Returns (query-replays, seconds)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor

    def one(s):
        W, tr, ev, key, ring = s
        cfg = oracle.OracleConfig(W=W, capacity_blocks=B_BLOCKS, pending_ring=ring,
                                  batch_slots=BATCH_SLOTS[0])
        r = oracle.run(cfg, tr, oracle.OraclePolicy(eviction=ev), key)
        return r.result["queries"]

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:   # ctypes releases the GIL
        q = sum(ex.map(one, sample))
    return q, time.perf_counter() - t0


def sample_desc(args, n, prefix):
    if args.workload == "c5":
        return (f"{n} full config-5 trials spread over the 48 cells (W=4..32, B=512), one per "
                f"host thread")
    return f"{n} trials x first {prefix} queries of the config-2 traces (W=8, B=512)"


def reference_arm(args, rank, world):
    if rank != 0:
        return
    import oracle
    oracle.build_oracle()
    launches = make_plan(args, 0, 1)
    threads = max(1, min(os.cpu_count() or 1, 16))
    prefix = None if args.workload == "c5" else args.ref_queries
    sample = oracle_sample(args, launches, threads * args.ref_trials_per_thread, prefix)
    warm = oracle_sample(args, launches, threads, 50 if prefix else None)
    for _ in range(args.warmup):
        run_oracle_sample(warm[:threads], threads)
    tot_q, tot_s = 0, 0.0
    for _ in range(args.steps):
        q, s = run_oracle_sample(sample, threads)
        tot_q += q
        tot_s += s
    v = tot_q / tot_s
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_s / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.workload == "c5" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_json(args),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": sample_desc(args, len(sample), prefix) + " per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ main
NCU_CAPTURE = os.path.join(ROOT, "profiles", "r2_bench_replay_ncu.json")


def ncu_capture(args):
    """DRAM traffic per launch of the replay kernel from the committed `ncu --set full`
    capture of this workload (profiles/); None when absent or for other sizes."""
    if args.trials or args.queries or not os.path.exists(NCU_CAPTURE):
        return None
    with open(NCU_CAPTURE) as f:
        d = json.load(f)
    if d.get("workload") != args.workload:
        return None
    d["src"] = os.path.relpath(NCU_CAPTURE, ROOT) + " (ncu --set full)"
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kvr", choices=["kvr", "reference"])
    ap.add_argument("--workload", default="c5", choices=["c5", "c2"])
    ap.add_argument("--batch-slots", type=int, default=0,
                    help="continuous batching (beta concurrent queries per worker; config 2 only: "
                         "beta * L_max <= B)")
    ap.add_argument("--ref-queries", type=int, default=15000,
                    help="config 2 only: queries per oracle trial in the CPU sample")
    ap.add_argument("--ref-trials-per-thread", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--queries", type=int, default=0, help=argparse.SUPPRESS)   # c2: per trace
    ap.add_argument("--trials", type=int, default=0, help=argparse.SUPPRESS)    # list size
    ap.add_argument("--dump-results", default="", help=argparse.SUPPRESS)       # per-trial bytes
    ap.add_argument("--ncu", action="store_true",
                    help="profiling run: one step, no warm-up / e2e / cpu baseline")
    args = ap.parse_args()
    if args.batch_slots and args.workload != "c2":
        ap.error("--batch-slots needs --workload c2 (config 5's 292-block paths exceed B / beta)")
    BATCH_SLOTS[0] = args.batch_slots
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
    from paper_2601_18999_b200 import dist as kdist
    from paper_2601_18999_b200.kvr import POLICY_DTYPE, RESULT_DTYPE, DeviceTrace, Simulator

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

    launches = make_plan(args, rank, world)
    stream = torch.cuda.current_stream()
    state = []          # per launch: (sim, device traces, buffers)
    trace_hash = 0
    for L in launches:
        dts = [DeviceTrace(t, device=dev) for t in L.traces]
        sim = Simulator(L.W, B_BLOCKS, pending_ring=L.ring, batch_slots=args.batch_slots)
        n = len(L)
        buf = sim.alloc(dts, max(1, n), 0, dev)
        if n:
            buf["keys"][:n].copy_(torch.from_numpy(L.keys.view(np.int64)))
            buf["policies"][: n * POLICY_DTYPE.itemsize].copy_(torch.from_numpy(L.policies().view(np.uint8)))
            buf["trial_trace"][:n].copy_(torch.from_numpy(L.trial_trace.view(np.int32)))
        # every rank packs the same traces; their identity checksum rides in the reduce
        trace_hash += sum(d.identity_digest() for d in dts)
        state.append((sim, dts, buf))
    trace_hash &= 0xFFFFFFFFFFFFFFFF
    trace_hash = trace_hash - (1 << 64) if trace_hash >= (1 << 63) else trace_hash
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    summary = [None]
    kern_ms = []        # per step: the replay launches' own CUDA-event time

    def step(timed_ms):
        flush.fill_(1)                                     # L2 flush, outside the timed region
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * len(state) + 1)]
        ev[0].record(stream)
        for i, (L, (sim, dts, buf)) in enumerate(zip(launches, state)):
            ev[2 * i].record(stream) if i else None
            if len(L):
                sim.launch(dts, len(L), buf, with_policies=True, stream=stream)
            ev[2 * i + 1].record(stream)
        vec = torch.zeros(len(kdist.SUMMARY_FIELDS), dtype=torch.int64, device=dev)
        for L, (sim, dts, buf) in zip(launches, state):
            if len(L):
                vec += kdist.summary_tensor(buf["results"], len(L), 0)
        vec[12] = trace_hash
        if world > 1:   # the single NCCL reduce of summary counters
            coll(dist.reduce, vec, dst=0)
        summary[0] = vec
        ev[-1].record(stream)
        torch.cuda.synchronize()
        timed_ms.append(ev[0].elapsed_time(ev[-1]))
        kern_ms.append([ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(len(state))])

    warm = []
    for _ in range(args.warmup):
        step(warm)
    kern_ms.clear()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            step(times)
    outs = [sim.collect(buf, len(L)).results if len(L) else np.zeros(0, RESULT_DTYPE)
            for L, (sim, dts, buf) in zip(launches, state)]
    res = np.concatenate(outs)
    evict = np.concatenate([L.evict for L in launches])
    if args.dump_results:
        tids = np.concatenate([L.tids for L in launches])
        np.savez(f"{args.dump_results}.rank{rank}.npz", tids=tids, results=res.view(np.uint8))
    bad = int((res["status"] != 0).sum())
    t_local = float(np.sum(times))
    tmax = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        coll(dist.all_reduce, tmax, op=dist.ReduceOp.MAX)
    t_max = float(tmax.item())
    red = summary[0].cpu().tolist()
    q_per_step, bad_all = float(red[1]), int(red[11])
    total_q = q_per_step * args.steps
    value = total_q / (t_max / 1000.0)

    # roofline of the dominant kernel: the replay launch with the largest CUDA-event time
    # (config 5: one launch per W; the W = 32 launch dominates).  Algorithmic bytes of that
    # launch's trials (probe 10 B, insert 22 B, evict 14 B) over its mean
    # launch time, measured on the launch stream inside the timed steps.
    pk = peaks()
    prof = ncu_capture(args)
    clk_s = clk.summary()
    f_mhz = clk_s["sm_mhz"] or pk["sm_max_mhz"]
    smem_peak = 148 * 128 * pk["sm_max_mhz"] * 1e6 / 1e9        # GB/s at max clock
    per_launch_ms = np.mean(np.asarray(kern_ms, dtype=np.float64), axis=0)
    kern_s = float(per_launch_ms.sum()) / 1000.0
    launches_out = []
    for i, (L, out) in enumerate(zip(launches, outs)):
        if not len(L):
            continue
        t_s = float(per_launch_ms[i]) / 1000.0
        sim_i = state[i][0]
        slots_i = min(len(L), sim_i.plan(max(t.max_blocks for t in L.traces))[2] * 148)
        floor_i = float(latency_floor_cycles(out, L.evict).sum()) / (f_mhz * 1e6) / max(1, slots_i)
        launches_out.append({"W": L.W, "trials": len(L), "ms": t_s * 1000.0,
                             "query_replays": float(out["queries"].sum()),
                             "smem_alg_gbs": algorithmic_bytes(out) / t_s / 1e9,
                             "smem_frac": algorithmic_bytes(out) / t_s / 1e9 / smem_peak,
                             "hbm_trace_gbs": trace_bytes([L]) / t_s / 1e9,
                             "latency_floor_s": floor_i, "latency_frac": floor_i / t_s,
                             "resident_replays": slots_i})
    dom = max(launches_out, key=lambda d: d["ms"]) if launches_out else None
    achieved_smem = dom["smem_alg_gbs"] if dom else 0.0
    achieved_hbm = dom["hbm_trace_gbs"] if dom else 0.0
    probes = float(res["probes"].sum())

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.workload == "c5" else "weak", "vs_baseline": None,
            "dtype": "f64+u64", "data": "synthetic", "config": config_json(args),
            "roofline": {"bound": "smem", "achieved": achieved_smem, "peak": smem_peak,
                         "unit": "GB/s", "frac": achieved_smem / smem_peak,
                         "kernel": f"replay_kernel launch W={dom['W']}" if dom else None,
                         "traffic": prof.get("traffic_bytes_per_launch") if prof else None,
                         "traffic_src": prof.get("src") if prof else None,
                         "peak_src": "148 SM x 128 B/clk x sm_max_mhz (DESIGN.md §6)",
                         "kernel_ms_per_step": kern_s * 1000.0,
                         "dominant_launch_ms": dom["ms"] if dom else None,
                         "hbm_trace": {"achieved": achieved_hbm, "peak": pk["hbm_gbs"],
                                       "frac": achieved_hbm / pk["hbm_gbs"], "peak_src": pk["src"]},
                         "latency": {"bound": "dependent-latency chain per replay",
                                     "floor_s": dom["latency_floor_s"] if dom else None,
                                     "achieved_s": dom["ms"] / 1000.0 if dom else None,
                                     "frac": dom["latency_frac"] if dom else None,
                                     "resident_replays": dom["resident_replays"] if dom else None,
                                     "sm_mhz": f_mhz,
                                     "model": "DESIGN.md §6 (300 cyc/query + 150 cyc/RLT "
                                              "eviction + 3 cyc/L-LRU eviction)"},
                         "per_launch": launches_out},
            "prefix_probes_per_s": probes * world / kern_s,
            "hit_rate": float(res["hit_tokens"].sum() / max(1, res["input_tokens"].sum())),
            "trial_status_nonzero": bad_all,
            "gpu_launches": args.steps * sum(1 for L in launches if len(L)),
            "clocks": clk_s}

    if world > 1 and rank == 0:
        line["reduced_summary"] = dict(zip(kdist.SUMMARY_FIELDS, [int(x) for x in red]))
        # sum over ranks of identical checksums = world x rank 0's (mod 2^64)
        line["reduced_summary"]["trace_hash_consistent"] = (
            (line["reduced_summary"]["trace_hash"] - world * trace_hash) % (1 << 64) == 0)
    if not args.no_e2e:
        if world > 1:
            dist.barrier()
        e = e2e_measure(launches, dev, stream, args)
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
        import oracle
        oracle.build_oracle()
        threads = max(1, min(os.cpu_count() or 1, 16))
        prefix = None if args.workload == "c5" else args.ref_queries
        full = make_plan(args, 0, 1) if world > 1 else launches
        sample = oracle_sample(args, full, threads, prefix)
        q, s = run_oracle_sample(sample, threads)
        q1, s1 = run_oracle_sample(sample[:1], 1)    # one core
        line["cpu_baseline"] = {"value": q / s, "unit": UNIT, "cores": threads, "kind": "oracle",
                                "single_core_value": q1 / s1, "nproc": os.cpu_count(),
                                "cpu_model": cpu_model(),
                                "sample": sample_desc(args, len(sample), prefix) +
                                "; single core: the first of them"}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def e2e_measure(launches, dev, stream, args):  # noqa: C901
    """Same metric through the public API with HOST buffers: per step the pinned raw
    traces, keys, policies and trial->trace maps go host->device, kvr_trace_load packs
    (validates, chains) them, kvr_sim_run_multi replays, and the per-trial results come
    back device->host into pinned memory, all inside the timed region."""
    import torch
    from paper_2601_18999_b200.kvr import POLICY_DTYPE, RESULT_DTYPE, DeviceTrace, Simulator

    per = []
    h2d, d2h = 0, 0
    for L in launches:
        sim = Simulator(L.W, B_BLOCKS, pending_ring=L.ring, batch_slots=args.batch_slots)
        host = [DeviceTrace.pin(t) for t in L.traces]                 # pinned, outside timing
        n = len(L)
        hk = torch.from_numpy(L.keys.view(np.int64)).pin_memory()
        hp = torch.from_numpy(L.policies().view(np.uint8)).pin_memory()
        ht = torch.from_numpy(L.trial_trace.view(np.int32)).pin_memory()
        hr = torch.empty(max(1, n) * 144, dtype=torch.uint8).pin_memory()
        h2d += sum(int(v.numel() * v.element_size()) for hd in host for v in hd.values())
        h2d += int(hk.numel() * 8 + hp.numel() + ht.numel() * 4)
        d2h += n * 144
        per.append((L, sim, host, hk, hp, ht, hr))
    times = []
    q = 0.0
    n_e2e = 1 + max(1, args.steps // 4)
    for it in range(1 + n_e2e):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        opened = []
        for L, sim, host, hk, hp, ht, hr in per:
            n = len(L)
            if not n:
                continue
            dts = [DeviceTrace(t, device=dev, host=hd) for t, hd in zip(L.traces, host)]
            b = sim.alloc(dts, n, 0, dev)
            b["keys"].copy_(hk, non_blocking=True)
            b["policies"].copy_(hp, non_blocking=True)
            b["trial_trace"].copy_(ht, non_blocking=True)
            sim.launch(dts, n, b, with_policies=True, stream=stream)
            hr.copy_(b["results"][: n * 144], non_blocking=True)
            opened += dts
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= 1:
            times.append(e0.elapsed_time(e1))
        q = sum(float(hr.numpy().view(RESULT_DTYPE)[: len(L)]["queries"].sum())
                for L, sim, host, hk, hp, ht, hr in per if len(L))
        for d in opened:
            d.close()
    ms = float(np.mean(times))
    return {"value": q / (ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms, "queries_per_step": q,
            "steps": len(times)}


if __name__ == "__main__":
    main()
