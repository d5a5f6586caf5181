"""Compile the sm_100a C-ABI extension in-tree: paper_1612_02736_b200/_hps_b200.so.

Plain nvcc (no torch extension machinery): the library exports only the C symbols of
include/hps_b200.h and is loaded with ctypes (_ext.py).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "_hps_b200.so")
SOURCES = ("hps_abi.cu", "gemm_dmma.cu", "gj.cu", "gj_fused.cu", "gj_cluster.cu", "gj_pair.cu", "gj_la.cu", "leaf_merge.cu", "sweep.cu", "sweep_tma.cu", "leaf_apply.cu")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the HPS extension needs the CUDA 12.9 toolkit")


HOST_LIB = os.path.join(PKG, "_hps_host.so")
HOST_SRC = os.path.join(CSRC, "host_gather.cpp")


def build_host(force: bool = False) -> str | None:
    """Compile the CPython helper module `_hps_host` (host-side gather of body-load mappings; not
    on the device path). Returns its path, or None when no host compiler / headers are available
    (solver.py then uses its numpy path)."""
    if not force and os.path.exists(HOST_LIB) and os.path.getmtime(HOST_LIB) >= os.path.getmtime(HOST_SRC):
        return HOST_LIB
    import sysconfig
    try:
        import numpy
        cxx = shutil.which("g++") or shutil.which("c++")
        if not cxx:
            return None
        cmd = [cxx, "-O3", "-std=c++17", "-shared", "-fPIC", "-pthread", "-I", sysconfig.get_paths()["include"],
               "-I", numpy.get_include(), HOST_SRC, "-o", HOST_LIB + ".tmp"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            return None
        os.replace(HOST_LIB + ".tmp", HOST_LIB)
        return HOST_LIB
    except Exception as exc:  # host helper is optional
        sys.stderr.write(f"_hps_host not built: {exc}\n")
        return None


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if not f.endswith(".cpp")]
    deps.append(os.path.join(ROOT, "include", "hps_b200.h"))
    return all(os.path.getmtime(d) <= t for d in deps if os.path.exists(d))


OBJ = os.path.join(PKG, "_build")


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "hps_b200.h")]


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile each source to an object (in parallel; a source is recompiled when it or any
    header is newer than its object), then link the shared library."""
    build_host(force)
    if not force and up_to_date():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max(os.path.getmtime(h) for h in _headers() if os.path.exists(h))
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include")]

    def compile_one(src):
        cu, obj = os.path.join(CSRC, src), os.path.join(OBJ, src.replace(".cu", ".o"))
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(cu), hdr_t):
            return obj, None
        res = subprocess.run([nvcc(), *flags, "-c", cu, "-o", obj + ".tmp"], capture_output=True, text=True)
        if res.returncode != 0:
            return obj, res.stdout + res.stderr
        os.replace(obj + ".tmp", obj)
        if verbose:
            sys.stderr.write(res.stderr)
        return obj, None

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    errs = [e for _, e in results if e]
    if errs:
        sys.stderr.write("\n".join(errs))
        raise RuntimeError("nvcc failed building the HPS extension")
    res = subprocess.run([nvcc(), *ARCH, "-shared", "-o", LIB + ".tmp", *[o for o, _ in results]],
                         capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking the HPS extension")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
