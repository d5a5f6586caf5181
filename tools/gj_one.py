"""Batched GJ inversion microbenchmark / ncu target: python tools/gj_one.py n ncols batch [reps]."""
import sys

sys.path.insert(0, ".")
import torch

from paper_1612_02736_b200 import _ext

n, ncols, batch = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
lib = _ext.load()
s = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda").manual_seed(0)
A0 = torch.randn(batch, n, ncols, dtype=torch.float64, device="cuda", generator=g)
A0[:, :, :n] += n ** 0.5 * torch.eye(n, dtype=torch.float64, device="cuda")
M = A0.clone()
piv = torch.empty(batch, n, dtype=torch.int32, device="cuda")
ws = torch.empty(int(lib.hps_gj_workspace_bytes(batch, n, ncols)), dtype=torch.uint8, device="cuda")
times = []
for r in range(reps):
    M.copy_(A0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lib.hps_gj_invert_batched(batch, n, ncols, _ext.mat(M, n * ncols, ncols), piv.data_ptr(), ws.data_ptr(),
                              None, None, None, None, s)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
ms = min(times)
fl = 2.0 * n * n * ncols * batch
print(f"GJ n={n} ncols={ncols} batch={batch}: {ms:.3f} ms  {fl / ms / 1e9:.2f} TFLOP/s (2n^2 ncols)")
