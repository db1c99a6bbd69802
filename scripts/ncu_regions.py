"""Sum ncu per-line samples / instructions over named source-line regions."""
import csv, subprocess, sys
rep = sys.argv[1]; src = sys.argv[2]
regions = [tuple(a.split(":")) for a in sys.argv[3:]]   # name:lo:hi
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; agg = {}
for r in rows:
    if r and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": continue
    if len(r) > 8 and r[2] == "-":
        try: ln = int(r[0]); s = int(r[4]); i = int(r[7])
        except ValueError: continue
        agg[(cur, ln)] = (s, i)
ts = sum(v[0] for v in agg.values()); ti = sum(v[1] for v in agg.values())
rest_s, rest_i = ts, ti
for name, lo, hi in regions:
    s = sum(v[0] for (f, l), v in agg.items() if f == src and int(lo) <= l <= int(hi))
    i = sum(v[1] for (f, l), v in agg.items() if f == src and int(lo) <= l <= int(hi))
    rest_s -= s; rest_i -= i
    print(f"{name:16s} samples {100*s/ts:5.1f}%  instructions {100*i/ti:5.1f}%")
print(f"{'other':16s} samples {100*rest_s/ts:5.1f}%  instructions {100*rest_i/ti:5.1f}%")
