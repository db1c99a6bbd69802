"""Map SASS addresses (hex suffixes) of an ncu report to CUDA source lines.

usage: python scripts/ncu_addr2line.py report.ncu-rep addr_hex [...]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
want = {int(a, 16) for a in sys.argv[2:]}
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, cur_line, cur_src = None, None, None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[2] == "-" and r[0].isdigit():
        cur_line, cur_src = int(r[0]), r[1]
        continue
    if len(r) > 3 and r[2].startswith("0x"):
        a = int(r[2], 16) & 0xfffff
        if a in want:
            print(f"{a:05x} {cur_file}:{cur_line}  {cur_src.strip()[:70]}  ||  {r[3].strip()}")
