"""Phase profile of the fused Gauss-Jordan kernel (clock64 counters of CTA 0, -DFU_PROFILE build).

  python tools/fu_prof.py build            # here (no GPU): abtest/fuprof/_hps_b200.so
  python tools/fu_prof.py run n ncols batch  # on the GPU box

Phases: 0 panel rows -> registers, 1 pivot-column loop, 2 panel -> smem/global + interchange
composition, 3 W rows + displaced rows, 4 DMMA update tiles, 5 end of matrix."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "abtest", "fuprof")
LIB = os.path.join(OUT, "_hps_b200.so")


def build():
    from paper_1612_02736_b200 import build_ext as B
    os.makedirs(OUT, exist_ok=True)
    objs = []
    for src in B.SOURCES:
        obj = os.path.join(OUT, src.replace(".cu", ".o"))
        cmd = [B.nvcc(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-DFU_PROFILE",
               "-I", os.path.join(ROOT, "include"), "-c", os.path.join(B.CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", LIB, *objs], check=True)
    print(LIB)


def run(n, ncols, batch):
    os.environ["HPS_B200_LIB"] = LIB
    import torch
    from paper_1612_02736_b200 import _ext
    lib = _ext.load()
    prof = ctypes.CDLL(LIB).hps_fu_prof
    g = torch.Generator(device="cuda").manual_seed(0)
    A0 = torch.randn(batch, n, ncols, dtype=torch.float64, device="cuda", generator=g)
    A0[:, :, :n] += n ** 0.5 * torch.eye(n, dtype=torch.float64, device="cuda")
    M = A0.clone()
    piv = torch.empty(batch, n, dtype=torch.int32, device="cuda")
    ws = torch.empty(int(lib.hps_gj_workspace_bytes(batch, n, ncols)), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    h = (ctypes.c_longlong * 8)()
    for rep in range(2):
        M.copy_(A0)
        torch.cuda.synchronize()
        prof(h, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.hps_gj_invert_batched(batch, n, ncols, _ext.mat(M, n * ncols, ncols), piv.data_ptr(), ws.data_ptr(),
                                  None, None, None, None, s)
        e1.record()
        torch.cuda.synchronize()
        prof(h, 0)
    tot = sum(h[:6])
    print(f"GJ n={n} ncols={ncols} batch={batch}: {e0.elapsed_time(e1):.3f} ms; CTA-0 cycles by phase (total {tot}):")
    for i, name in enumerate(("load panel", "column loop", "store panel", "W + moves", "DMMA tiles", "tail")):
        print(f"  {name:12s} {h[i]:12d}  {100.0 * h[i] / max(tot, 1):5.1f} %")


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(*(int(x) for x in sys.argv[2:5]))
