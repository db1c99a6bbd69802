"""Aggregate an ncu source page (cuda,sass) to per-source-line samples / instructions."""
import csv, subprocess, sys
rep = sys.argv[1]; topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; agg = {}
for r in rows:
    if r and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": continue
    if cur and len(r) > 8 and r[2] == "-":
        try: samp = int(r[4]); inst = int(r[7])
        except ValueError: continue
        agg[(cur, int(r[0]))] = (samp, inst, r[1][:100])
ts = sum(v[0] for v in agg.values()) or 1; ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts} warp-instructions {ti}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:topn]:
    print(f"{k[0]}:{k[1]:4d} samp {100*v[0]/ts:5.1f}% inst {100*v[1]/ti:5.1f}%  {v[2]}")
print("--- by instructions")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:topn]:
    print(f"{k[0]}:{k[1]:4d} samp {100*v[0]/ts:5.1f}% inst {100*v[1]/ti:5.1f}%  {v[2]}")
