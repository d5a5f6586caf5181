"""Summarise an ncu report's SASS source page: top instructions by warp-stall samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
data = [dict(zip(hdr, r)) for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", tot)
data.sort(key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))
for d in data[:top]:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    st = sorted(((int(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{s:7d} {100.0 * s / tot:5.1f}%  {d['Address'][-5:]}  {d['Source'].strip()[:60]:60s} "
          + " ".join(f"{n}:{v}" for v, n in st if v))
