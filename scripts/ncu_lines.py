"""Top CUDA source lines by warp-stall samples (ncu source page), optionally excluding lines.

usage: python scripts/ncu_lines.py report.ncu-rep [topn] [exclude_line ...]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
excl = {int(a) for a in sys.argv[3:]}
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, agg = None, {}
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[2] == "-" and r[0].isdigit():
        k = (cur, int(r[0]))
        s, i, src = agg.get(k, (0, 0, r[1]))
        agg[k] = (s + int(r[4]), i + int(r[7]), src)
tot = sum(v[0] for v in agg.values())
keep = {k: v for k, v in agg.items() if k[1] not in excl}
sub = sum(v[0] for v in keep.values())
print(f"total samples {tot}, after exclusions {sub}")
for (f, ln), (s, i, src) in sorted(keep.items(), key=lambda x: -x[1][0])[:topn]:
    print(f"{f}:{ln:<5} {100 * s / sub:5.2f}% exec {i:>10}  {src.strip()[:80]}")
