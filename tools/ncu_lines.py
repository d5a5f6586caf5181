"""Per-CUDA-source-line warp-stall samples from an ncu report (cuda,sass source view)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = next(r for r in rows if r and r[0] == "Line No")
col = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lines = []
for r in rows:
    if len(r) == len(hdr) and r[0] not in ("", "Line No") and r[2] == "-":
        s = int(r[col] or 0)
        st = sorted(((int(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        lines.append((s, r[0], r[1], st))
tot = sum(l[0] for l in lines)
print("total", tot)
for s, ln, src, st in sorted(lines, reverse=True)[:top]:
    print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}%  L{ln:>4} {src.strip()[:70]:70s} " + " ".join(f"{n}:{v}" for v, n in st if v))
