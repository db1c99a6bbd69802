"""Experiment build (KVR_WHO_LAST): per config-5 launch (one eighth of the fixed list),
which warp arrives last at the per-query barrier -- the warp that updated the previous
query's chosen worker, one that ran a deferred apply, or a scoring-only warp -- and by
how much.  usage: KVR_LIB=.../libkvr_who.so python scripts/who_last.py [W,...]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_18999_b200 import kvr  # noqa: E402

Ws = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else list(bench.C5_WS)
L_ = kvr.lib()
L_.kvr_debug_phase_cycles.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(16, dtype=np.uint64)
for L in bench.c5_plan(0, 8):
    if L.W not in Ws:
        continue
    dts = [kvr.DeviceTrace(t) for t in L.traces]
    sim = kvr.Simulator(L.W, bench.B_BLOCKS, pending_ring=L.ring)
    L_.kvr_debug_phase_cycles(buf.ctypes.data, 6)
    sim.run(dts, L.keys, L.policies(), trial_trace=L.trial_trace)
    torch.cuda.synchronize()
    L_.kvr_debug_phase_cycles(buf.ctypes.data, 6)
    n = buf[:3].sum()
    names = ["updated prev chosen", "deferred apply", "scoring only"]
    print(f"W={L.W}: " + ", ".join(f"{names[i]} {100 * buf[i] / n:.1f} % (lead {buf[4 + i] / max(1, buf[i]):.0f} cyc)"
                                  for i in range(3)) +
          f"; deferred apply {buf[3] / max(1, buf[7]):.0f} cycles on average ({int(buf[7])} applies): " +
          ", ".join(f"{nm} {buf[8 + i] / max(1, buf[7]):.0f}" for i, nm in
                    enumerate(["erase", "arrays/log", "inserts", "rebuild", "digest/record"])))
