"""Config 5 at its real shape on the GPU: 128x128 leaves, p=16, backward Euler with dt=1e-3, all
16 seeded right-hand sides stepped TOGETHER through DeviceStepper / be_run (multi-RHS leaf
kernels: hps_leaf_apply g = u/dt, the 16-RHS TMA leaf-down kernel gemv_tma_kernel<16>, the DMMA
multi-RHS parent steps), checked after every one of the first 3 steps against the reference's own
trajectory (tests/golden/full_cfg5_traj.npz, made by make_golden.py --only-traj through
specdtn's FactorizedSolver.solve loop, solver.py:337-354).

Fingerprint coverage: every leaf of every RHS enters an RHS-mixed random projection per step;
per RHS, u on 500 seeded Gauss nodes and the max-norms; at step 3 the RHS-mixed projection of
every Gauss edge segment and 4 complete leaf tabulations per RHS. A wrong value anywhere moves
a projection. Tolerance: the north star's relative max-norm 1e-10, turned into bounds for the
projections via |sum_i w_i d_i| <= ||w||_1 max|d|.

A second test runs the reference's 50-step single-RHS trajectory at 16x16 leaves for drift
(tests/golden/cfg5_drift_n16.npz), with nrhs = 1 and with the seed replicated over 3 RHS."""
import numpy as np
import pytest
import torch

from hps_testutil import golden
from paper_1612_02736_b200 import build_stage, build_uniform_tree, problems
from paper_1612_02736_b200.timestepping import DeviceStepper, _leaf_points, be_run

pytestmark = pytest.mark.gpu
UNIT = (0.0, 1.0, 0.0, 1.0)
PROJ_SEED = 99  # tests/golden/make_golden.py


def proj_weights(n):
    return np.random.default_rng([PROJ_SEED, n]).standard_normal(n)


def _initial(solver, seeds):
    pts = _leaf_points(solver).reshape(-1, 2)
    cols = [problems.config5_initial(s)(pts).reshape(solver._n_leaves, -1) for s in seeds]
    return torch.as_tensor(np.stack(cols, axis=-1), device="cuda").contiguous()


def _dirichlet(solver, nrhs):
    bpts = solver.plan.coords[solver.plan.node[solver.tree.root].ext]

    def f(t):
        v = problems.config5_dirichlet(bpts, t)
        return torch.as_tensor(np.repeat(v[:, None], nrhs, axis=1), device="cuda").contiguous()
    return f


def _sorted_rows(solver, leaf_ids):
    row = {int(n): r for r, n in enumerate(solver._leaf_ids)}
    return np.array([row[int(n)] for n in leaf_ids])


def test_config5_16rhs_three_steps_vs_reference():
    fx = golden("full_cfg5_traj.npz")
    dt, tol = 1e-3, 1e-10
    nrhs, steps = int(fx["nrhs"][0]), int(fx["steps"][0])
    solver = build_stage(build_uniform_tree(UNIT, 128), problems.config5_spec(dt), 16, 15)
    u0 = _initial(solver, range(nrhs))
    fdir = _dirichlet(solver, nrhs)
    stp = DeviceStepper(solver, nrhs, 1.0 / dt, 0.0)
    stp.set_state(u0)
    rows = _sorted_rows(solver, fx["leaf_ids"])
    cmix = np.random.default_rng([PROJ_SEED, 16, 1]).standard_normal(nrhs)
    wP, wq = proj_weights(solver.p ** 2), proj_weights(solver.q)
    N = solver.plan.n_gauss
    for k in range(1, steps + 1):
        stp.step(fdir(k * dt))
        T = stp.leaf_tabulations().cpu().numpy()[rows]            # (n_leaves, P, nrhs), sorted ids
        U = stp.pool[stp.lay["U"]:stp.lay["U"] + N].cpu().numpy()  # (N_gauss, nrhs)
        umax, lmax = fx["u_max"][k - 1], fx["leaf_max"][k - 1]
        scale = max(umax.max(), lmax.max())
        np.testing.assert_allclose(np.abs(U).max(axis=0), umax, rtol=0, atol=tol * scale)
        np.testing.assert_allclose(np.abs(T).max(axis=(0, 1)), lmax, rtol=0, atol=tol * scale)
        du = np.abs(U[fx["u_idx"]].T - fx["u_vals"][k - 1])
        assert du.max() <= tol * scale, (k, du.max() / scale)
        mix = np.einsum("lpr,p,r->l", T, wP, cmix)
        bound = tol * scale * np.abs(wP).sum() * np.abs(cmix).sum()
        assert np.abs(mix - fx["mix_proj"][k - 1]).max() <= bound, k
    seg = np.einsum("sqr,q,r->s", U.reshape(-1, solver.q, nrhs), wq, cmix)
    assert np.abs(seg - fx["mix_seg"]).max() <= tol * scale * np.abs(wq).sum() * np.abs(cmix).sum()
    pick = _sorted_rows(solver, fx["leaf_pick"])
    T = stp.leaf_tabulations().cpu().numpy()[pick]                # (4, P, nrhs)
    assert np.abs(T.transpose(2, 0, 1) - fx["leaf_sol"]).max() <= tol * scale
    # the public be_run driver reproduces the stepper's trajectory bit for bit
    st2 = be_run(solver, u0, fdir, dt, steps)
    final = st2.leaf_tabulations().cpu().numpy()[pick]
    assert np.array_equal(final, T)


@pytest.mark.parametrize("nrhs", [1, 3])
def test_config5_drift_50_steps_vs_reference(nrhs):
    fx = golden("cfg5_drift_n16.npz")
    dt, tol = 1e-3, 1e-10
    n = int(fx["n"][0])
    solver = build_stage(build_uniform_tree(UNIT, n), problems.config5_spec(dt), 16, 15)
    stp = DeviceStepper(solver, nrhs, 1.0 / dt, 0.0)
    stp.set_state(_initial(solver, [0] * nrhs))
    fdir = _dirichlet(solver, nrhs)
    rows = _sorted_rows(solver, fx["leaf_ids"])
    wP, wq = proj_weights(solver.p ** 2), proj_weights(solver.q)
    keep = [int(k) for k in fx["keep"]]
    N = solver.plan.n_gauss
    for k in range(1, keep[-1] + 1):
        stp.step(fdir(k * dt))
        if k not in keep:
            continue
        T = stp.leaf_tabulations().cpu().numpy()[rows]
        U = stp.pool[stp.lay["U"]:stp.lay["U"] + N].cpu().numpy()
        scale = fx[f"s{k}_all_leaf_absmax"].max()
        for r in range(nrhs):
            np.testing.assert_allclose(np.abs(T[:, :, r]).max(axis=1), fx[f"s{k}_all_leaf_absmax"],
                                       rtol=0, atol=tol * scale)
            assert np.abs(T[:, :, r] @ wP - fx[f"s{k}_all_leaf_proj"]).max() <= tol * scale * np.abs(wP).sum()
            assert np.abs(U[:, r].reshape(-1, solver.q) @ wq - fx[f"s{k}_seg_proj"]).max() \
                <= tol * scale * np.abs(wq).sum()
    for r in range(nrhs):
        assert np.abs(U[:, r] - fx["u_final"]).max() <= tol * scale
        assert np.abs(T[:, :, r] - fx["leaf_sol_final"]).max() <= tol * scale
