"""Debug harness for the gj_pair kernel: batches of n=196 x (196+60) matrices through
hps_gj_invert_batched, compared with numpy; reports bad matrices, first bad column, pivots."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
from scipy.linalg import lu_factor

from paper_1612_02736_b200 import _ext

lib = _ext.load()
n, nrhs = 196, 60
for batch in (3, 74, 75, 148, 300):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((batch, n, n)) + n ** 0.5 * np.eye(n) * rng.choice([-1, 1], size=(batch, 1, 1))
    R = rng.standard_normal((batch, n, nrhs))
    M = torch.tensor(np.concatenate([A, R], axis=2), device="cuda")
    ncols = n + nrhs
    piv = torch.empty(batch, n, dtype=torch.int32, device="cuda")
    ws = torch.empty(int(lib.hps_gj_workspace_bytes(batch, n, ncols)), dtype=torch.uint8, device="cuda")
    an = torch.empty(batch, dtype=torch.float64, device="cuda")
    ai = torch.empty(batch, dtype=torch.float64, device="cuda")
    st = torch.zeros(batch, dtype=torch.int32, device="cuda")
    rc = lib.hps_gj_invert_batched(batch, n, ncols, _ext.mat(M, n * ncols, ncols), piv.data_ptr(), ws.data_ptr(),
                                   an.data_ptr(), ai.data_ptr(), st.data_ptr(), None,
                                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    out = M.cpu().numpy()
    pv = piv.cpu().numpy()
    bad = []
    for i in range(batch):
        inv = np.linalg.inv(A[i])
        err = np.abs(out[i, :, :n] - inv).max() / np.abs(inv).max()
        _, lp = lu_factor(A[i])
        pbad = int(np.argmax(pv[i] != lp)) if (pv[i] != lp).any() else -1
        x = np.linalg.solve(A[i], R[i])
        xerr = np.abs(out[i, :, n:] - x).max() / max(np.abs(x).max(), 1.0)
        aerr = abs(ai[i].item() - np.linalg.norm(inv, 1)) / np.linalg.norm(inv, 1)
        if err > 1e-11 or pbad >= 0 or xerr > 1e-11 or aerr > 1e-10:
            colerr = np.abs(out[i, :, :n] - inv).max(axis=0)
            bad.append((i, err, xerr, aerr, pbad, int(np.argmax(colerr > 1e-9 * np.abs(inv).max()))))
    print("batch", batch, "rc", rc, "bad", len(bad), bad[:8], "status", int(st.sum()))

# what do the wrong right-hand-side columns hold?
batch = 148
rng = np.random.default_rng(n)
A = rng.standard_normal((batch, n, n)) + n ** 0.5 * np.eye(n) * rng.choice([-1, 1], size=(batch, 1, 1))
R = rng.standard_normal((batch, n, nrhs))
M = torch.tensor(np.concatenate([A, R], axis=2), device="cuda")
ncols = n + nrhs
piv = torch.empty(batch, n, dtype=torch.int32, device="cuda")
ws = torch.empty(int(lib.hps_gj_workspace_bytes(batch, n, ncols)), dtype=torch.uint8, device="cuda")
an = torch.empty(batch, dtype=torch.float64, device="cuda")
ai = torch.empty(batch, dtype=torch.float64, device="cuda")
st = torch.zeros(batch, dtype=torch.int32, device="cuda")
lib.hps_gj_invert_batched(batch, n, ncols, _ext.mat(M, n * ncols, ncols), piv.data_ptr(), ws.data_ptr(),
                          an.data_ptr(), ai.data_ptr(), st.data_ptr(), None, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
out = M.cpu().numpy()
for i in (0, 1, 74, 75):
    x = np.linalg.solve(A[i], R[i])
    got = out[i, :, n:]
    print("item", i, "err", np.abs(got - x).max(), "== R", np.abs(got - R[i]).max(),
          "rows bad", int((np.abs(got - x).max(axis=1) > 1e-8).sum()), "cols bad", int((np.abs(got - x).max(axis=0) > 1e-8).sum()))
    for j in (i + 74, i - 74):
        if 0 <= j < batch:
            xj = np.linalg.solve(A[j], R[j])
            print("   vs x of", j, np.abs(got - xj).max(), " inv(A_i) R_j", np.abs(got - np.linalg.solve(A[i], R[j])).max())
