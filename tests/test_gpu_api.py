"""The reference's error contract and solve-API semantics, exercised on the GPU path
(SURVEY.md 8b "errors", "ownership" and "threading" rows):

* MergeSingularError for an interface resonance through build_stage (solver.py:108-119; the
  reference tests it on merge_siblings, test_solver.py:85-91). The resonant wavenumber is found
  and the raising box recorded by the reference itself (tests/golden/resonance.npz).
* invalid order, non-finite coefficients (host callable and on-device sympy evaluation),
  MeshConformityError, through the GPU build_stage (test_solver.py:219-224, test_model.py:60,
  test_geometry.py:200,235).
* downward_pass completes the state it is given, in place, from that state's w and g_tab
  (solver.py:428-432, 293-335) - no upward sweep is re-run.
* concurrent solves on one built solver from several threads give the serial results
  (SPEC.md:421-422); host result arrays of earlier states survive later solves.
* economy mode with a split-size leaf upward step (p = 26, K = 576 >= 512).
"""
import threading

import numpy as np
import pytest

from hps_testutil import golden
from paper_1612_02736_b200 import (CoefficientField, MergeSingularError, MeshConformityError, ProblemSpec,
                                   RefinementSpec, build_forest, build_stage, build_uniform_tree, catalog,
                                   refine_near_point)
from paper_1612_02736_b200.solver import downward_pass, upward_pass

pytestmark = pytest.mark.gpu
UNIT = (0.0, 1.0, 0.0, 1.0)


def test_merge_singular_error_at_interface_resonance():  # solver.py:108-119, test_solver.py:85-91
    fx = golden("resonance.npz")
    n, p, q = int(fx["n"][0]), int(fx["p"][0]), int(fx["q"][0])
    kappa, box = float(fx["kappa"][0]), int(fx["box"][0])
    with pytest.raises(MergeSingularError, match=f"interface operator of box {box} is numerically singular"):
        build_stage(build_uniform_tree(UNIT, n), catalog("helmholtz", kappa=kappa), p, q)
    # away from the resonance the same mesh builds and solves
    solver = build_stage(build_uniform_tree(UNIT, n), catalog("helmholtz", kappa=kappa * 0.9), p, q)
    assert np.isfinite(solver.solve(f=lambda pts: pts[:, 0]).u).all()


def test_invalid_order_rejected_gpu():  # test_solver.py:219-224
    tree = build_uniform_tree(UNIT, 2)
    with pytest.raises(ValueError, match="before its children"):
        build_stage(tree, catalog("laplace"), 9, 8, order=range(len(tree.nodes)))


def test_nonfinite_coefficient_host_callable():  # model.py:174-176, test_model.py:53-60
    spec = ProblemSpec("nan", CoefficientField(c11=lambda pts: np.full(len(pts), np.nan), c22=1))
    with pytest.raises(ValueError, match="non-finite coefficient evaluation on leaf"):
        build_stage(build_uniform_tree(UNIT, 2), spec, 9, 8)


def test_nonfinite_coefficient_device_expression():
    # c = 1/(x1 - 1/2) is evaluated on the device (sympy -> torch) and is infinite on the leaf
    # edges at x1 = 1/2: the device-side finiteness check must name a leaf touching that line
    spec = ProblemSpec("inf", CoefficientField(1, 0, 1, c="1/(x1 - 1/2)"))
    with pytest.raises(ValueError, match="non-finite coefficient evaluation on leaf") as ei:
        build_stage(build_uniform_tree(UNIT, 2), spec, 9, 8)
    assert "0.5" in str(ei.value)


def test_mesh_conformity_errors_gpu():  # test_geometry.py:192-199, 231-235
    tree = build_uniform_tree(UNIT, 2)
    refine_near_point(tree, RefinementSpec((0.45, 0.25), 2, threshold=1e-6))
    with pytest.raises(MeshConformityError, match="2:1"):
        build_stage(tree, catalog("laplace"), 9, 8)
    with pytest.raises(MeshConformityError, match="share no interface"):
        build_stage(build_forest([(0.0, 1.0, 0.0, 1.0), (2.0, 3.0, 0.0, 1.0)], 2), catalog("laplace"), 9, 8)


def _problem():
    spec = catalog("varcoef_helmholtz", kappa=10.0)
    f = lambda pts: np.sin(2 * pts[:, 0]) + pts[:, 1]  # noqa: E731
    return spec, f


@pytest.mark.parametrize("mode", ["stored", "econ"])
@pytest.mark.parametrize("refined", [False, True])
def test_downward_pass_in_place(mode, refined):  # solver.py:418-432
    spec, f = _problem()
    tree = build_uniform_tree(UNIT, 4)
    if refined:
        refine_near_point(tree, RefinementSpec((0.5, 0.5), 1))
    solver = build_stage(tree, spec, 9, 8, mode)
    full = solver.solve(f=f)
    st = upward_pass(solver)
    out = downward_pass(solver, f, st)
    assert out is st and st.scratch is None
    scale = np.abs(full.u).max()
    assert np.abs(st.u - full.u).max() <= 1e-13 * scale
    for nid in full.leaf_solutions:
        assert np.abs(st.leaf_solutions[nid] - full.leaf_solutions[nid]).max() <= 1e-13 * scale
    # the downward pass reads the STATE: with w and g_tab zeroed it gives the f-only solution
    st2 = upward_pass(solver)
    st2.w[:] = 0.0
    st2.g_tab = {nid: np.zeros_like(np.asarray(v)) for nid, v in st2.g_tab.items()}
    downward_pass(solver, f, st2)
    harmonic = solver.solve(f=f, g=lambda pts: np.zeros(len(pts)))
    assert np.abs(st2.u - harmonic.u).max() <= 1e-13 * scale


def test_concurrent_solves_match_serial():
    spec, _ = _problem()
    solver = build_stage(build_uniform_tree(UNIT, 8), spec, 12, 11)
    fs = [lambda pts, a=a: np.cos(a * pts[:, 0]) + a * pts[:, 1] for a in range(8)]
    serial = [solver.solve(f=fn) for fn in fs]
    results = [None] * len(fs)

    def worker(i):
        for _ in range(3):
            results[i] = solver.solve(f=fs[i])

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(fs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for ref, got in zip(serial, results):
        assert np.array_equal(ref.u, got.u)
        for nid in ref.leaf_solutions:
            assert np.array_equal(ref.leaf_solutions[nid], got.leaf_solutions[nid])
    # the serial states kept their own values while 24 more solves ran
    again = solver.solve(f=fs[0])
    assert np.array_equal(serial[0].u, again.u)
    assert not np.array_equal(serial[0].u, serial[1].u)


def test_host_results_survive_later_solves():
    spec, _ = _problem()
    solver = build_stage(build_uniform_tree(UNIT, 4), spec, 9, 8)
    states = [solver.solve(f=lambda pts, a=a: a + pts[:, 0]) for a in range(5)]
    leaf = next(iter(states[0].leaf_solutions))
    for a, st in enumerate(states):
        fresh = solver.solve(f=lambda pts, a=a: a + pts[:, 0])
        assert np.array_equal(st.u, fresh.u)
        assert np.array_equal(st.leaf_solutions[leaf], fresh.leaf_solutions[leaf])


def test_solve_device_out_buffers():
    import torch
    spec, f = _problem()
    solver = build_stage(build_uniform_tree(UNIT, 4), spec, 9, 8)
    root_ext = solver.plan.node[solver.tree.root].ext
    fv = torch.as_tensor(f(solver.plan.coords[root_ext]), device="cuda").reshape(-1, 1)
    g = torch.as_tensor(solver._leaf_table(None), device="cuda").reshape(-1, 1)
    u_keep = torch.empty((solver.plan.n_gauss, 1), dtype=torch.float64, device="cuda")
    r1 = solver.solve_device(fv, g, out={"u": u_keep})
    assert r1["u"] is u_keep
    solver.solve_device(2 * fv, g)
    ref = solver.solve(f=f)
    assert np.abs(u_keep[:, 0].cpu().numpy() - ref.u).max() <= 1e-13 * np.abs(ref.u).max()


@pytest.mark.parametrize("nrhs", [1, 4])
def test_econ_split_size_leaf_step(nrhs):  # econ, 4x4 leaves, p = 26
    import torch
    spec, f = _problem()
    tree = build_uniform_tree(UNIT, 4)
    stored = build_stage(tree, spec, 26, 25)
    econ = build_stage(tree, spec, 26, 25, "econ")
    a, b = stored.solve(f=f), econ.solve(f=f)
    assert np.abs(a.u - b.u).max() <= 1e-12 * np.abs(a.u).max()
    root_ext = stored.plan.node[tree.root].ext
    fv = torch.as_tensor(f(stored.plan.coords[root_ext]), device="cuda")[:, None].repeat(1, nrhs).contiguous()
    g = torch.as_tensor(stored._leaf_table(None), device="cuda").reshape(-1, 1).repeat(1, nrhs).contiguous()
    ua = stored.solve_device(fv, g)["uc"].clone()
    ub = econ.solve_device(fv, g)["uc"].clone()
    assert (ua - ub).abs().max().item() <= 1e-12 * ua.abs().max().item()


def test_load_conventions_agree_on_a_large_mesh():
    """g as a callable, as the reference's {leaf id: (m,)} mapping (solver.py:241-253; the C
    gather helper with range-by-range uploads handles >= 2048 leaves), as a mapping whose values
    the fast path does not take (float32, lists, strided views: generic numpy path) and as the
    (n_leaves, m) table give the same solution; a wrong-length value raises like the reference."""
    n, p, q = 64, 8, 7  # 4096 leaves, small order: exercises the chunked gather cheaply
    tree = build_uniform_tree(UNIT, n)
    solver = build_stage(tree, catalog("laplace"), p, q)
    gfn = lambda pts: np.sin(3 * pts[:, 0]) * np.cos(2 * pts[:, 1])
    ref = solver.solve(g=gfn)
    tab = np.asarray(solver._leaf_table(gfn))
    ids = [int(i) for i in solver._leaf_ids]
    gmap = {nid: tab[r].copy() for r, nid in enumerate(ids)}
    st = solver.solve(g=gmap)
    assert np.array_equal(st.u, ref.u)
    assert st.g_tab is gmap  # the state keeps the caller's mapping, as the reference does
    odd = dict(gmap)
    odd[ids[5]] = tab[5].astype(np.float32).astype(np.float64).tolist()          # a list
    odd[ids[77]] = np.repeat(tab[77], 2)[::2]                                      # a strided view
    st2 = solver.solve(g=odd)
    exact = dict(gmap)
    exact[ids[5]] = np.asarray(odd[ids[5]])
    assert np.array_equal(st2.u, solver.solve(g=exact).u)
    assert np.array_equal(solver.solve(g=tab).u, ref.u)
    bad = dict(gmap)
    bad[ids[9]] = np.zeros(tab.shape[1] + 1)
    with pytest.raises(ValueError, match=f"leaf {ids[9]} load has shape"):
        solver.solve(g=bad)
    missing = dict(gmap)
    del missing[ids[3]]
    with pytest.raises(KeyError):
        solver.solve(g=missing)
