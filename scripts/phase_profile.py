"""Per-phase cycle breakdown of the replay kernel (profiling build libkvr_prof.so).

usage: python scripts/phase_profile.py [queries] [trials]
Phases 0-4 are summed over all warps; 5-12 only over the chosen warp i*.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_18999_b200 import build  # noqa: E402

_defs = [d for d in os.environ.get("KVR_DEFS", "").split(",") if d]
os.environ["KVR_LIB"] = (build.build_variant("prof_x", ["KVR_PHASE_PROFILE"] + _defs) if _defs
                         else build.build(profile=True))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_18999_b200 import kvr  # noqa: E402

NAMES = ["stage wait", "catch-up", "match", "score", "barrier", "argmin",
         "deferred apply", "prologue+hits", "miss decisions", "accounting"]

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 444
Wk = int(sys.argv[3]) if len(sys.argv) > 3 else 8
trs = bench.build_traces(nq)
dts = [kvr.DeviceTrace(t) for t in trs]
L = kvr.lib()
L.kvr_debug_phase_cycles.argtypes = [C.c_void_p, C.c_int]
L.kvr_debug_phase_cycles.restype = C.c_int32
buf = np.zeros(32, dtype=np.uint64)
for label, ev in (("RLT", 1), ("LRU", 0)):
    t_of, _, keys = bench.trial_plan(0, nt)
    sim = kvr.Simulator(Wk, 512, pending_ring=bench.RING)
    pols = kvr.policies_array([kvr.Policy(eviction=ev) for _ in keys])
    sim.run(dts, keys[:8], pols[:8], trial_trace=t_of[:8])     # warm-up
    L.kvr_debug_phase_cycles(buf.ctypes.data, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = sim.run(dts, keys, pols, trial_trace=t_of)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    L.kvr_debug_phase_cycles(buf.ctypes.data, 1)
    q = float(out.results["queries"].sum())
    print(f"== {label} W={Wk}: {nt} trials x {nq} queries, {ms:.1f} ms, {q / ms / 1e3:.2f} M q-r/s, "
          f"hit {out.results['hit_tokens'].sum() / out.results['input_tokens'].sum():.3f}, "
          f"evict/q {out.results['evictions'].sum() / q:.1f}, probes/q {out.results['probes'].sum() / q:.1f}")
    tot = 0
    for i, n in enumerate(NAMES):
        per = buf[i] / q / (Wk if i <= 5 else 1)
        if i > 6:
            tot += per
        print(f"  {i:2d} {n:14s} {per:10.0f} cycles/query{' (per warp)' if i <= 6 else ' (i*)'}")
    print(f"  i* update total {tot:.0f} cycles/query")
    nc = max(int(buf[15]), 1)
    print(f"  LRU log: compactions {int(buf[15])} ({buf[10] / q:.0f} cycles/query, "
          f"{buf[10] / nc:.0f} cycles each, len {buf[13] / nc:.0f} -> {buf[14] / nc:.0f}); "
          f"take {buf[11] / q:.0f} cycles/query, {buf[12] / q:.1f} entries scanned/query")
    print(f"  critical-path applies: {int(buf[17])} of {int(q)} queries, {buf[16] / max(int(buf[17]), 1):.0f} cycles each; "
          f"kf {buf[18] / q:.0f}, hits loop {buf[19] / q:.0f} cycles/query")
    if buf[25]:
        print(f"  RLT fast segment: {buf[25] / q:.0f} cycles/query, {int(buf[26]) % (1 << 32)} iterations "
              f"(mod 2^32), {buf[25] / max(1, int(buf[26]) % (1 << 32)):.0f} cycles/iteration")
    print(f"  accounting split: fifo push + Pt {buf[27] / q:.0f}, trial sums (lane 0) {buf[28] / q:.0f} cycles/query")
    print(f"  apply split (per query): erase {buf[29] / q:.0f}, arrays/log {buf[30] / q:.0f}, "
          f"inserts {buf[31] / q:.0f}, rebuilds {buf[24] / q:.0f}, digest/record {buf[23] / q:.0f}")
    tc = np.zeros(4096, dtype=np.uint64)
    L.kvr_debug_phase_cycles(tc.ctypes.data, 2)
    tq = tc[:nt].astype(np.float64) / nq
    print(f"  per-trial cycles/query: min {tq.min():.0f} median {np.median(tq):.0f} "
          f"p90 {np.percentile(tq, 90):.0f} max {tq.max():.0f}; wall {ms * 1.965e6 / nq:.0f}")
    for ti in range(3):
        sel = tq[t_of == ti]
        print(f"    trace {ti}: median {np.median(sel):.0f} max {sel.max():.0f}")
