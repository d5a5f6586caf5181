"""Kernel-level parity of the sm_100a primitives (through the C ABI) against float64 references."""
import ctypes

import numpy as np
import pytest
import torch

from paper_1612_02736_b200 import _ext

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    return _ext.load()


def _stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("M,N,K,batch", [(1, 1, 1, 1), (64, 64, 16, 3), (65, 70, 33, 5), (196, 60, 60, 7),
                                         (60, 196, 196, 2), (300, 129, 77, 1), (256, 256, 64, 3),
                                         (257, 131, 33, 2), (130, 250, 48, 1), (1000, 700, 200, 1)])
def test_gemm_batched(lib, M, N, K, batch):
    g = torch.Generator(device="cuda").manual_seed(M * 1000 + N)
    A = torch.randn(batch, M, K, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(batch, K, N, dtype=torch.float64, device="cuda", generator=g)
    C = torch.randn(batch, M, N, dtype=torch.float64, device="cuda", generator=g)
    bias = torch.randn(M, N, dtype=torch.float64, device="cuda", generator=g)
    ref = 0.5 * torch.bmm(A, B) - 2.0 * C + bias
    rc = lib.hps_gemm_batched(batch, M, N, K, 0.5, _ext.mat(A, M * K, K), _ext.mat(B, K * N, N), -2.0,
                              _ext.mat(C, M * N, N), bias.data_ptr(), N, _stream())
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.allclose(C, ref, rtol=1e-13, atol=1e-12 * ref.abs().max().item())


def test_gemm_pointer_array_and_offsets(lib):
    # operands addressed through device pointer arrays with a column offset, shared B (stride 0)
    A = [torch.randn(40, 30, dtype=torch.float64, device="cuda") for _ in range(3)]
    B = torch.randn(30, 25, dtype=torch.float64, device="cuda")
    C = torch.zeros(3, 40, 50, dtype=torch.float64, device="cuda")
    aptr = torch.tensor([a.data_ptr() for a in A], dtype=torch.int64, device="cuda")
    rc = lib.hps_gemm_batched(3, 40, 25, 30, 1.0, _ext.mat(0, 0, 30, ptrs=aptr), _ext.mat(B, 0, 25), 0.0,
                              _ext.mat(C, 40 * 50, 50, off=25), None, 0, _stream())
    assert rc == 0
    torch.cuda.synchronize()
    for i in range(3):
        assert torch.allclose(C[i, :, 25:], A[i] @ B, rtol=1e-13, atol=1e-12)
        assert torch.count_nonzero(C[i, :, :25]) == 0


def _gj(lib, M, n, ncols):
    batch = M.shape[0]
    piv = torch.empty(batch, n, dtype=torch.int32, device="cuda")
    ws = torch.empty(int(lib.hps_gj_workspace_bytes(batch, n, ncols)), dtype=torch.uint8, device="cuda")
    an = torch.empty(batch, dtype=torch.float64, device="cuda")
    ai = torch.empty(batch, dtype=torch.float64, device="cuda")
    st = torch.zeros(batch, dtype=torch.int32, device="cuda")
    rc = lib.hps_gj_invert_batched(batch, n, ncols, _ext.mat(M, n * ncols, ncols), piv.data_ptr(), ws.data_ptr(),
                                   an.data_ptr(), ai.data_ptr(), st.data_ptr(), None, _stream())
    assert rc == 0
    torch.cuda.synchronize()
    return piv, an, ai, st


@pytest.mark.parametrize("n,nrhs,batch", [(1, 0, 2), (5, 3, 4), (15, 90, 3), (33, 7, 2), (60, 240, 5),
                                          (196, 60, 3), (196, 60, 300), (100, 40, 50), (196, 0, 20), (130, 500, 150), (300, 10, 2),
                                          (900, 124, 1), (1000, 3000, 1), (1003, 37, 2), (1920, 200, 1)])
def test_gj_inverse_matches_numpy(lib, n, nrhs, batch):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((batch, n, n)) + n ** 0.5 * np.eye(n) * rng.choice([-1, 1], size=(batch, 1, 1))
    R = rng.standard_normal((batch, n, nrhs))
    M = torch.tensor(np.concatenate([A, R], axis=2), device="cuda")
    piv, an, ai, st = _gj(lib, M, n, n + nrhs)
    out = M.cpu().numpy()
    for i in range(batch):
        inv = np.linalg.inv(A[i])
        assert np.abs(out[i, :, :n] - inv).max() <= 1e-11 * np.abs(inv).max()
        if nrhs:
            x = np.linalg.solve(A[i], R[i])
            assert np.abs(out[i, :, n:] - x).max() <= 1e-11 * max(np.abs(x).max(), 1.0)
        assert abs(an[i].item() - np.linalg.norm(A[i], 1)) <= 1e-12 * np.linalg.norm(A[i], 1)
        assert abs(ai[i].item() - np.linalg.norm(inv, 1)) <= 1e-10 * np.linalg.norm(inv, 1)
    assert int(st.abs().sum()) == 0


@pytest.mark.parametrize("n", [70, 1000])
def test_gj_pivot_sequence_matches_lapack(lib, n):
    from scipy.linalg import lu_factor
    rng = np.random.default_rng(3)
    A = rng.standard_normal((1, n, n))
    M = torch.tensor(A.copy(), device="cuda")
    piv, *_ = _gj(lib, M, n, n)
    _, lp = lu_factor(A[0])
    np.testing.assert_array_equal(piv.cpu().numpy()[0], lp)


def test_gj_flags_singular(lib):
    n = 12
    A = np.zeros((2, n, n))
    A[1] = np.eye(n)
    A[0, :, 3] = 0.0  # column of zeros -> zero pivot
    A[0] += np.eye(n)
    A[0, 3, 3] = 0.0
    M = torch.tensor(A, device="cuda")
    _, an, ai, st = _gj(lib, M, n, n)
    s = st.cpu().numpy()
    assert s[0] != 0 and s[1] == 0


@pytest.mark.parametrize("n,batch", [(60, 3), (196, 200), (300, 2)])
def test_gj_permuted_columns_output(lib, n, batch):
    rng = np.random.default_rng(n + 1)
    A = rng.standard_normal((batch, n, n)) + 2 * n ** 0.5 * np.eye(n)
    M = torch.tensor(A.copy(), device="cuda")
    piv = torch.empty(batch, n, dtype=torch.int32, device="cuda")
    perm = torch.empty(batch, n, dtype=torch.int32, device="cuda")
    ws = torch.empty(int(lib.hps_gj_workspace_bytes(batch, n, n)), dtype=torch.uint8, device="cuda")
    rc = lib.hps_gj_invert_batched(batch, n, n, _ext.mat(M, n * n, n), piv.data_ptr(), ws.data_ptr(), None, None,
                                   None, perm.data_ptr(), _stream())
    assert rc == 0
    torch.cuda.synchronize()
    out, pm = M.cpu().numpy(), perm.cpu().numpy()
    for i in range(batch):
        inv = np.linalg.inv(A[i])
        assert np.abs(out[i] - inv[:, pm[i]]).max() <= 1e-11 * np.abs(inv).max()


def test_gj_pair_kernel_opt_in():
    """The 2-CTA cluster Gauss-Jordan kernel (csrc/gj_pair.cu, opt-in with HPS_GJ_PAIR=1, read once
    per process) passes the same inverse / pivot / permuted-output checks."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, HPS_GJ_PAIR="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", __file__,
                        "-k", "gj_inverse or gj_pivot or gj_permuted or gj_flags"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_gj_lookahead_kernel_opt_in():
    """The warp-specialised look-ahead Gauss-Jordan kernel (csrc/gj_la.cu, opt-in with HPS_GJ_LA=1,
    read once per process; taken for 56 < n <= 224 with >= 148 matrices) passes the same inverse /
    permuted-output checks, several matrices per persistent CTA included."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, HPS_GJ_LA="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", __file__,
                        "-k", "(gj_inverse and (196 or 130)) or gj_permuted"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]

