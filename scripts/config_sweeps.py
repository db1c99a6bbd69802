"""Throughput of BASELINE.json configs 3, 4 and 5 on one B200, each at one GPU's
share of its replays (config c's trial list strided over 8 ranks, rank 0's
share; the full list is what `bench.py --gpus 8`-style sharding would spread).
bench.py times config 2; this script measures the other full-size sweeps with
the same clock (CUDA events on the launching stream around the replay launches
only; traces packed and resident beforehand).  SURVEY §8(d) recipes:

* config 3: DRIFT(8192, 1,000,000, s=1.1, N/64), W = 16, B = 512, RLT; LBGR
  (mu in {0.008,0.1,0.5,0.992} x dt in {10,20,40,80}), STATIC ((w_load, w_hit)
  in {0.25,1,4}^2), THRESHOLD (tau in {1.25,1.5,2,4}), cycled; 4,096 replays.
* config 4: ADV(B, 4, 8 cycles), W = 1, B = 2^6..2^16, {L-LRU, RLT} x 11;
  16,384 replays.
* config 5: {GSP(128,32,r), MT-ShareGPT(128,r), MT-UltraChat(128,r), LD(512,Qd)}
  x {low r=0.3/Qd=2, med 0.5/8, high 0.9/32} x W in {4,8,16,32}, B = 512, LBGR,
  RLT on even keys, L-LRU on odd; 65,536 replays (ranks 0 and 1: see below).

usage: python scripts/config_sweeps.py [configs=3,4,5] [ranks=8] [out.json]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_18999_b200 import workloads as wl  # noqa: E402
from paper_2601_18999_b200.kvr import DeviceTrace, Policy, Simulator, policies_array  # noqa: E402

which = [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "3,4,5").split(",")]
RANKS = int(sys.argv[2]) if len(sys.argv) > 2 else 8
out_path = sys.argv[3] if len(sys.argv) > 3 else None
RING = 16384


def timed_launch(sim, dts, keys, pols, trial_trace=None):
    """One warm-up launch, then one timed launch; returns (results, ms)."""
    n = len(keys)
    b = sim.alloc(dts, n)
    b["keys"].copy_(torch.from_numpy(np.asarray(keys, np.uint64).view(np.int64)))
    b["policies"].copy_(torch.from_numpy(np.ascontiguousarray(pols).view(np.uint8)))
    if trial_trace is not None:
        b["trial_trace"].copy_(torch.from_numpy(np.asarray(trial_trace, np.uint32).view(np.int32)))
    s = torch.cuda.current_stream()
    sim.launch(dts, n, b, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    sim.launch(dts, n, b, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    return sim.collect(b, n).results, e0.elapsed_time(e1)


def summarize(name, parts, extra):
    res = np.concatenate([r for r, _ in parts])
    ms = sum(m for _, m in parts)
    q = float(res["queries"].sum())
    pk = bench.peaks()
    smem_peak = 148 * 128 * pk["sm_max_mhz"] * 1e6 / 1e9      # GB/s
    alg = bench.algorithmic_bytes(res)
    row = dict(config=name, trials=int(len(res)), query_replays=int(q), gpu_ms=ms,
               query_replays_per_s=q / (ms / 1e3),
               prefix_probes_per_s=float(res["probes"].sum()) / (ms / 1e3),
               hit_rate=float(res["hit_tokens"].sum() / max(1, res["input_tokens"].sum())),
               status_nonzero=int((res["status"] != 0).sum()),
               smem_alg_gbs=alg / (ms / 1e3) / 1e9, smem_peak_gbs=smem_peak,
               smem_alg_frac=alg / (ms / 1e3) / 1e9 / smem_peak, **extra)
    print(json.dumps(row), flush=True)
    return row


rows = []
if 3 in which:
    t0 = time.time()
    tr = wl.drift(8192, 1_000_000, seed=0xC5, W=16)
    dt = DeviceTrace(tr)
    grid = ([dict(router=0, mu=mu, delta_t_ms=d) for mu in (0.008, 0.1, 0.5, 0.992)
             for d in (10.0, 20.0, 40.0, 80.0)] +
            [dict(router=1, w_load=a, w_hit=b) for a in (0.25, 1.0, 4.0) for b in (0.25, 1.0, 4.0)] +
            [dict(router=2, tau=tau) for tau in (1.25, 1.5, 2.0, 4.0)])
    # 1,366 / 1,365 / 1,365 trials per router, parameters cycled within a router
    by_router = {0: [g for g in grid if g["router"] == 0], 1: [g for g in grid if g["router"] == 1],
                 2: [g for g in grid if g["router"] == 2]}
    plan = []
    for t in range(4096):
        r = 0 if t < 1366 else (1 if t < 2731 else 2)
        k = t - (0 if r == 0 else (1366 if r == 1 else 2731))
        plan.append(by_router[r][k % len(by_router[r])])
    mine = list(range(0, 4096, RANKS))
    pols = policies_array([Policy(eviction=1, **plan[t]) for t in mine])
    # pending FIFO up to the trace length (pooled chunks, ABI v7): no trial stops at a ring
    # overflow, even the collapsing NLMS cells (mu = 0.992) whose queues grow without bound
    sim = Simulator(16, 512, pending_ring=tr.n_queries)
    res, ms = timed_launch(sim, [dt], np.array([t + 1 for t in mine], np.uint64), pols)
    rows.append(summarize("config3: DRIFT 1M queries, W=16, B=512, RLT, LBGR/STATIC/THRESHOLD grid",
                          [(res, ms)], dict(share=f"trials t = 0 mod {RANKS} of 4,096",
                                            build_s=time.time() - t0)))
    sim.close()

if 4 in which:
    parts = []
    trials = 0
    for bi, B in enumerate(2 ** np.arange(6, 17)):
        B = int(B)
        tr = wl.adv(B, 4, 8, seed=0xC6)
        dt = DeviceTrace(tr)
        # cells (B, LRU) and (B, RLT) of 744/745 trials; this rank's share of both
        cell_trials = [t for t in range(16384) if t // 745 in (2 * bi, 2 * bi + 1)]
        mine = [t for t in cell_trials if t % RANKS == 0]
        pols = policies_array([Policy(eviction=1 if (t // 745) % 2 else 0, router=3) for t in mine])
        sim = Simulator(1, B, pending_ring=RING)
        res, ms = timed_launch(sim, [dt], np.array([t + 1 for t in mine], np.uint64), pols)
        parts.append((res, ms))
        trials += len(mine)
        sim.close()
    rows.append(summarize("config4: ADV(B,4,8), W=1, B=64..65536, {L-LRU, RLT}", parts,
                          dict(share=f"trials t = 0 mod {RANKS} of 16,384 (one launch per B)")))

if 5 in which:
    # the bench's fixed 65,536-trial list, this script's share = rank 0 of RANKS under the
    # bench's (t div 2) mod N sharding (RLT and Leaf-LRU mixed), one launch per W
    parts = []
    for L in bench.c5_plan(0, RANKS):
        dts = [DeviceTrace(t) for t in L.traces]
        sim = Simulator(L.W, bench.B_BLOCKS, pending_ring=L.ring)
        res, ms = timed_launch(sim, dts, L.keys, L.policies(), trial_trace=L.trial_trace)
        parts.append((res, ms))
        rows.append(summarize(f"config5 W={L.W}: 4 benchmarks x 3 settings, B=512, LBGR, RLT/L-LRU mixed",
                              [(res, ms)], dict(share=f"(t div 2) mod {RANKS} == 0 of 65,536",
                                                tier=sim.plan(max(t.max_blocks for t in L.traces))[0])))
        sim.close()
    rows.append(summarize("config5 all W (sum of the four launches)", parts,
                          dict(share=f"(t div 2) mod {RANKS} == 0 of 65,536")))

if out_path:
    with open(out_path, "w") as f:
        json.dump(dict(gpu=torch.cuda.get_device_name(0), ranks=RANKS, rows=rows), f, indent=1)
