"""Build an alternate library for A/B runs: python tools/build_alt.py NAME [file.cu=replacement.cu ...] [-DFLAG ...]
-> abtest/NAME/_hps_b200.so (load with HPS_B200_LIB=abtest/NAME/_hps_b200.so)."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1612_02736_b200 import build_ext as B

name = sys.argv[1]
subs = dict(a.split("=") for a in sys.argv[2:] if "=" in a and not a.startswith("-"))
flags = [a for a in sys.argv[2:] if a.startswith("-")]
out = os.path.join(ROOT, "abtest", name)
os.makedirs(out, exist_ok=True)


def one(src):
    cu = subs.get(src, os.path.join(B.CSRC, src))
    obj = os.path.join(out, src.replace(".cu", ".o"))
    subprocess.run([B.nvcc(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *flags,
                    "-I", os.path.join(ROOT, "include"), "-I", B.CSRC, "-c", cu, "-o", obj], check=True,
                   capture_output=True)
    return obj


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, B.SOURCES))
lib = os.path.join(out, "_hps_b200.so")
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs], check=True)
print(lib)
