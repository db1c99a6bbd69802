"""Stall-reason totals from an ncu source page, optionally restricted to source line ranges."""
import csv, subprocess, sys
rep = sys.argv[1]
rng = None
if len(sys.argv) > 3:
    rng = (sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))   # file, lo, hi
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; cur = None; tot = {}; line = None
for r in rows:
    if r and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if not hdr or len(r) < len(hdr): continue
    if r[2] == "-":           # source line row
        try: line = int(r[0])
        except ValueError: line = None
        continue
    if rng and not (cur == rng[0] and line is not None and rng[1] <= line <= rng[2]): continue
    if "abortf" in (r[1] or ""): pass
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try: tot[h] = tot.get(h, 0) + int(r[i])
            except ValueError: pass
s = sum(tot.values()) or 1
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:14]:
    print(f"{k:28s} {v:10d} {100*v/s:5.1f}%")
