"""Per-phase cycle breakdown of the continuous-batching kernel (profiling build libkvr_prof.so).

usage: python scripts/batch_phase_profile.py [queries] [trials] [W] [beta]
Phases 0-3 are summed over all warps (printed per warp); 4-16 over the warps that ran them.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_18999_b200 import build  # noqa: E402

os.environ["KVR_LIB"] = os.environ.get("KVR_PROF_LIB") or build.build(profile=True)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_18999_b200 import kvr  # noqa: E402

NAMES = {0: "header + catch-up (per warp)", 1: "match + score (per warp)", 2: "barrier (per warp)",
         3: "argmin (per warp)", 4: "assignment (chosen)", 8: "update: hit run", 9: "L-LRU take",
         10: "L-LRU erase", 11: "L-LRU miss run total", 12: "serial loop (RLT misses)",
         13: "log append", 17: "deferred inserts", 18: "rebuilds", 14: "dequeue: staging", 15: "dequeue: accounting",
         16: "completion: release path"}

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 296
Wk = int(sys.argv[3]) if len(sys.argv) > 3 else 8
beta = int(sys.argv[4]) if len(sys.argv) > 4 else 3
trs = bench.build_traces(nq)
dts = [kvr.DeviceTrace(t) for t in trs]
L = kvr.lib()
L.kvr_debug_phase_cycles.argtypes = [C.c_void_p, C.c_int]
L.kvr_debug_phase_cycles.restype = C.c_int32
buf = np.zeros(32, dtype=np.uint64)
for label, ev in (("RLT", 1), ("LRU", 0)):
    t_of, _, keys = bench.trial_plan(0, nt)
    sim = kvr.Simulator(Wk, 512, pending_ring=bench.RING, batch_slots=beta)
    pols = kvr.policies_array([kvr.Policy(eviction=ev) for _ in keys])
    sim.run(dts, keys[:8], pols[:8], trial_trace=t_of[:8])     # warm-up
    L.kvr_debug_phase_cycles(buf.ctypes.data, 4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = sim.run(dts, keys, pols, trial_trace=t_of)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    L.kvr_debug_phase_cycles(buf.ctypes.data, 4)
    q = float(out.results["queries"].sum())
    print(f"== {label} W={Wk} beta={beta}: {nt} trials x {nq} queries, {ms:.1f} ms, "
          f"{q / ms / 1e3:.2f} M q-r/s, evict/q {out.results['evictions'].sum() / q:.1f}, "
          f"wall {ms * 1.965e6 / nq:.0f} cycles/query/trial")
    for i, n in NAMES.items():
        per = buf[i] / q / (Wk if i <= 3 else 1)
        print(f"  {i:2d} {n:32s} {per:10.0f} cycles/query")
    print(f"  dequeues/query {buf[20] / q:.2f}, completions/query {buf[21] / q:.2f}, "
          f"assignments/query {buf[22] / q:.2f}, rebuilds/query {buf[23] / q:.3f}")
