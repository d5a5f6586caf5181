O=gpurun_out
cd abtest/gptrace && timeout 300 python - > /root/repo/$O/gptrace.log 2>&1 <<'PY'
import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1612_02736_b200 import _ext
lib = _ext.load()
n, nrhs, batch = 196, 60, 148
rng = np.random.default_rng(1)
A = rng.standard_normal((batch, n, n)) + 14 * np.eye(n)
M = torch.tensor(np.concatenate([A, rng.standard_normal((batch, n, nrhs))], axis=2), device="cuda")
ncols = n + nrhs
piv = torch.empty(batch, n, dtype=torch.int32, device="cuda")
ws = torch.empty(int(lib.hps_gj_workspace_bytes(batch, n, ncols)), dtype=torch.uint8, device="cuda")
an = torch.empty(batch, dtype=torch.float64, device="cuda"); ai = torch.empty(batch, dtype=torch.float64, device="cuda")
st = torch.zeros(batch, dtype=torch.int32, device="cuda")
lib.hps_gj_invert_batched(batch, n, ncols, _ext.mat(M, n * ncols, ncols), piv.data_ptr(), ws.data_ptr(), an.data_ptr(), ai.data_ptr(), st.data_ptr(), None, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("done")
PY
