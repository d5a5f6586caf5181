"""Microbenchmark of hps_gemm_batched (DMMA GEMM) vs shapes; prints TFLOP/s."""
import sys

sys.path.insert(0, ".")
import torch

from paper_1612_02736_b200 import _ext

lib = _ext.load()
s = torch.cuda.current_stream().cuda_stream
shapes = [(4096, 4096, 4096, 1, 0), (7680, 7680, 1920, 1, 1), (900, 1024, 64, 256, 0), (900, 1024, 64, 1024, 1), (960, 960, 240, 16, 1), (196, 256, 64, 1024, 0)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
shapes = [sh if len(sh) == 5 else sh + (0,) for sh in shapes]
for M, N, K, b, beta in shapes:
    A = torch.randn(b, M, K, dtype=torch.float64, device="cuda")
    B = torch.randn(b, K, N, dtype=torch.float64, device="cuda")
    C = torch.zeros(b, M, N, dtype=torch.float64, device="cuda")
    args = (b, M, N, K, 1.0, _ext.mat(A, M * K, K), _ext.mat(B, K * N, N), float(beta), _ext.mat(C, M * N, N), None, 0, s)
    for _ in range(2):
        lib.hps_gemm_batched(*args)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        lib.hps_gemm_batched(*args)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{M}x{N}x{K} x{b} beta={beta}: {ms:.3f} ms  {2.0 * M * N * K * b / ms / 1e9:.2f} TFLOP/s", flush=True)
    if not beta:
        ref = torch.bmm(A[:1], B[:1])
        print("   err", (ref - C[:1]).abs().max().item())
