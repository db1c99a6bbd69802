"""SASS with per-instruction stall samples / executions in an address range (hex suffixes).

usage: python scripts/ncu_sass_range.py report.ncu-rep lo_hex hi_hex
"""
import csv
import subprocess
import sys

rep, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
hdr = None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "Address":
        hdr = r
        si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        st = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr and len(r) == len(hdr):
        a = int(r[0], 16) & 0xfffff
        if lo <= a <= hi:
            top = sorted(((int(r[i]), h[6:]) for i, h in st), reverse=True)[:2]
            print(f"{a:05x} {int(r[si]):6d} {int(r[ii]):>9}  {r[1].strip()[:60]:60s} "
                  + " ".join(f"{h}:{v}" for v, h in top if v))
