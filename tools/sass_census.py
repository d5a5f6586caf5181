"""Per-kernel SASS census of the built extension (cuobjdump -sass): how many DMMA (FP64 tensor
core), UTMALDG (TMA tensor load), UBLKCP (bulk copy), UCGABAR (cluster barrier), SYNCS (mbarrier),
LDGSTS (cp.async), DFMA and spill (LDL/STL) instructions each kernel contains.

    python tools/sass_census.py [path/to/_hps_b200.so] > profiles/round2_sass_census.txt
"""
import os
import re
import subprocess
import sys

SO = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "paper_1612_02736_b200",
                                                        "_hps_b200.so")
KEYS = [("DMMA", r"\bDMMA\."), ("UTMALDG", r"\bUTMALDG"), ("UBLKCP", r"\bUBLKCP"), ("UCGABAR", r"\bUCGABAR"),
        ("SYNCS", r"\bSYNCS\."), ("LDGSTS", r"\bLDGSTS"), ("DFMA", r"\bDFMA\b"), ("LDL/STL", r"\b(LDL|STL)\b")]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
        return out.splitlines()
    except Exception:
        return names


def main():
    sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
    kernels, cur = {}, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = {k: 0 for k, _ in KEYS}
            continue
        if cur is None:
            continue
        for k, pat in KEYS:
            if re.search(pat, line):
                kernels[cur][k] += 1
    names = list(kernels)
    pretty = demangle(names)
    print(f"{'kernel':<90}" + "".join(f"{k:>9}" for k, _ in KEYS))
    tot = {k: 0 for k, _ in KEYS}
    for n, pn in sorted(zip(names, pretty), key=lambda x: x[1]):
        row = kernels[n]
        for k in tot:
            tot[k] += row[k]
        print(f"{pn[:89]:<90}" + "".join(f"{row[k]:>9}" for k, _ in KEYS))
    print(f"{'TOTAL (%d kernels)' % len(names):<90}" + "".join(f"{tot[k]:>9}" for k, _ in KEYS))
    with_dmma = sum(1 for r in kernels.values() if r["DMMA"])
    print(f"kernels with DMMA: {with_dmma}/{len(names)}; no UTC*MMA/TMEM by design (tcgen05 has no f64 kind)")


if __name__ == "__main__":
    main()
