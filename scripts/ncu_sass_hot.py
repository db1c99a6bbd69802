"""Top SASS instructions by warp-stall samples with their dominant stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]; topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
skip = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; data = []
for r in rows:
    if r and r[0] == "Address": hdr = r; continue
    if hdr and len(r) == len(hdr):
        data.append(r)
si = hdr.index("Warp Stall Sampling (All Samples)"); ii = hdr.index("Instructions Executed")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[si]) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -int(r[si]))[:topn]:
    if skip and skip in r[1]: continue
    st = sorted(((int(r[i]), h[6:]) for i, h in stall_cols), reverse=True)[:3]
    print(f"{r[0][-5:]} {100*int(r[si])/tot:5.2f}% exec {int(r[ii]):>10}  {r[1].strip()[:48]:48s} " +
          " ".join(f"{h}:{v}" for v, h in st if v))
