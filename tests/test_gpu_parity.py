"""GPU build/solve (through build_stage -> C ABI) vs the pinned CPU oracle and the golden
vectors produced by the reference. Tolerances: relative max-norm <= 1e-10 (<= 1e-9 at
p >= 32), as BASELINE.json's north star states."""
import numpy as np
import pytest

from hps_testutil import golden, rel_maxdiff
from oracle import hps_oracle as orc
from paper_1612_02736_b200 import (LeafSingularError, build_balanced_refined_tree, build_stage, build_uniform_tree,
                                   catalog, enumerate_gauss_nodes, problems, refine_near_point)

pytestmark = pytest.mark.gpu
UNIT = (0.0, 1.0, 0.0, 1.0)


def _compare_fixture(fx, st, tol, prefix=""):
    ids = fx[prefix + "leaf_ids"]
    sol = np.stack([st.leaf_solutions[int(i)] for i in ids])
    assert rel_maxdiff(sol, fx[prefix + "leaf_sol"]) <= tol
    assert rel_maxdiff(st.u, fx[prefix + "u"]) <= tol


def test_config1_vs_golden_and_oracle():
    fx = golden("cfg1.npz")
    tree = build_uniform_tree(UNIT, 4)
    spec = problems.config1_spec()
    solver = build_stage(tree, spec, 16, 15)
    st = solver.solve()
    _compare_fixture(fx, st, 1e-10)
    assert rel_maxdiff(st.h_root, fx["h_root"]) <= 1e-10 or np.abs(fx["h_root"]).max() == 0
    # random-RHS variant (8 Gaussians, f = 0)
    st2 = solver.solve(f=lambda pts: np.zeros(len(pts)), g=problems.config1_random_load(0))
    _compare_fixture(fx, st2, 1e-10, prefix="rand_")
    # error vs the exact solution within 2x of the reference's
    exact = spec.u_exact
    err = 0.0
    for lf in tree.leaves():
        pts = orc.leaf_points(lf.bounds, 16, 15)
        geo = orc.leaf_geometry(16, 15, lf.bounds.width, lf.bounds.height)
        err = max(err, np.abs(st.leaf_solutions[lf.id][geo["i_ce"]] - exact(pts[geo["i_ce"]])).max())
    assert err <= 2.0 * fx["linf_error"][0] + 1e-15


def test_config2_small_vs_golden():
    fx = golden("cfg2_n4.npz")
    spec = problems.config2_spec()
    st = build_stage(build_uniform_tree(UNIT, 4), spec, 16, 15).solve()
    _compare_fixture(fx, st, 1e-10)


def test_config3_small_vs_golden():
    fx = golden("cfg3_n4.npz")
    st = build_stage(build_uniform_tree(UNIT, 4), problems.config3_spec(), 32, 31).solve()
    _compare_fixture(fx, st, 1e-9)


def test_config4_small_vs_golden():
    fx = golden("cfg4_small.npz")
    tree = build_balanced_refined_tree(4, (0.3, 0.7), 3)
    st = build_stage(tree, problems.config4_spec(), 16, 14).solve()
    _compare_fixture(fx, st, 1e-10)


def test_refined_reference_native_vs_golden():
    fx = golden("refined_r4.npz")
    tree = build_uniform_tree(UNIT, 4)
    refine_near_point(tree, (0.5, 0.5), 1)
    st = build_stage(tree, catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)"), 9, 8).solve()
    _compare_fixture(fx, st, 1e-10)


def test_config5_small_backward_euler_vs_golden():
    fx = golden("cfg5_n4.npz")
    dt = 1e-3
    tree = build_uniform_tree(UNIT, 4)
    solver = build_stage(tree, problems.config5_spec(dt), 16, 15)
    for r in range(2):
        u0 = problems.config5_initial(r)
        tabs = {lf.id: u0(orc.leaf_points(lf.bounds, 16, 15)) for lf in tree.leaves()}
        for step in (1, 2):
            t = step * dt
            st = solver.solve(f=lambda pts, _t=t: problems.config5_dirichlet(pts, _t),
                              g=orc.be_loads(tabs, tree, 16, 15, dt))
            tabs = st.leaf_solutions
        sol = np.stack([tabs[i] for i in sorted(tabs)])
        assert rel_maxdiff(sol, fx[f"rhs{r}_leaf_sol"]) <= 1e-10


@pytest.mark.parametrize("n,p,q", [(2, 9, 8), (4, 12, 11), (8, 16, 15), (16, 16, 15)])
def test_varcoef_vs_oracle(n, p, q):
    spec = catalog("varcoef_helmholtz", kappa=10.0)
    tree = build_uniform_tree(UNIT, n)
    solver = build_stage(tree, spec, p, q)
    f = lambda pts: np.sin(2 * pts[:, 0] + pts[:, 1])
    st = solver.solve(f=f)
    ref = orc.solve(orc.build(tree, spec, p, q, enumerate_gauss_nodes(tree, q)), f)
    sol = np.stack([st.leaf_solutions[i] for i in sorted(ref["leaf_solutions"])])
    rsol = np.stack([ref["leaf_solutions"][i] for i in sorted(ref["leaf_solutions"])])
    assert rel_maxdiff(sol, rsol) <= 1e-10
    assert rel_maxdiff(st.u, ref["u"]) <= 1e-10
    assert rel_maxdiff(st.w, ref["w"]) <= 1e-10


def test_harmonic_reproduction_and_boundary_exact():
    tree = build_uniform_tree(UNIT, 4)
    solver = build_stage(tree, catalog("laplace"), 9, 8)
    f = lambda pts: np.cos(3 * pts[:, 0]) + pts[:, 1]
    st = solver.solve(f=f)
    ext = solver.plan.root_exterior()
    np.testing.assert_array_equal(st.u[ext], f(solver.plan.coords[ext]))
    st = solver.solve(f=lambda pts: pts[:, 0])
    for lf in tree.leaves():
        pts = orc.leaf_points(lf.bounds, 9, 8)
        assert np.abs(st.leaf_solutions[lf.id] - pts[:, 0]).max() <= 1e-11


def test_zero_data_zero_solution():
    solver = build_stage(build_uniform_tree(UNIT, 2), catalog("laplace"), 9, 8)
    assert np.abs(solver.solve().u).max() == 0.0


def test_resonant_leaf_raises():
    tree = build_uniform_tree(UNIT, 1)
    with pytest.raises(LeafSingularError, match="singular"):
        build_stage(tree, catalog("helmholtz", kappa=np.sqrt(2.0) * np.pi), 20, 19)


@pytest.mark.parametrize("nrhs,n,p", [(1, 4, 10), (2, 4, 10), (3, 4, 10), (8, 4, 10), (16, 4, 10), (16, 16, 12),
                                       (5, 16, 16), (16, 16, 16), (11, 32, 10)])
def test_multi_rhs_device_solve_matches_single(nrhs, n, p):
    import torch
    tree = build_uniform_tree(UNIT, n)
    refine_near_point(tree, (0.5, 0.5), 1)
    spec = catalog("varcoef_helmholtz", kappa=10.0)
    solver = build_stage(tree, spec, p, p - 2)
    m = (p - 2) ** 2
    nl = solver._n_leaves
    rng = np.random.default_rng(nrhs)
    root_ext = solver.plan.node[tree.root].ext
    F = rng.standard_normal((root_ext.size, nrhs))
    G = rng.standard_normal((nl * m, nrhs))
    out = solver.solve_device(torch.tensor(F, device="cuda"), torch.tensor(G, device="cuda"))
    u = out["u"].cpu().numpy()
    uc = out["uc"].cpu().numpy()
    for j in range(nrhs):
        st = solver.solve(f=F[:, j], g=G[:, j].reshape(nl, m))
        assert rel_maxdiff(u[:, j], st.u) <= 1e-12
        ref = np.stack([st.leaf_solutions[i] for i in solver._leaf_ids])
        assert rel_maxdiff(uc[:, :, j], ref) <= 1e-12


def test_upward_downward_split_matches_solve():
    from paper_1612_02736_b200 import downward_pass, upward_pass
    spec = catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)")
    tree = build_uniform_tree(UNIT, 2)
    solver = build_stage(tree, spec, 17, 16)
    st = upward_pass(solver)
    assert np.abs(st.u).max() == 0.0
    j3 = solver.plan.node[tree.root].j3
    pts = solver.plan.coords[j3]
    np.testing.assert_allclose(st.w[j3], np.sin(np.pi * pts[:, 0]) * np.sin(np.pi * pts[:, 1]), atol=1e-9)
    full = downward_pass(solver, None, st)
    ref = solver.solve()
    assert rel_maxdiff(full.u, ref.u) <= 1e-14


class TestEconomyMode:
    """Reference test_solver.py:226-247,284-292 (econ == stored, memory strictly smaller)."""

    def test_solutions_match_stored(self):
        spec = catalog("varcoef_helmholtz", kappa=8.0)
        tree = build_uniform_tree(UNIT, 4)
        stored = build_stage(tree, spec, 9, 8, "stored")
        econ = build_stage(tree, spec, 9, 8, "econ")
        s, e = stored.solve(), econ.solve()
        assert np.abs(s.u - e.u).max() <= 1e-12
        for nid in s.leaf_solutions:
            np.testing.assert_allclose(s.leaf_solutions[nid], e.leaf_solutions[nid], atol=1e-12)

    def test_memory_strictly_smaller(self):
        tree = build_uniform_tree(UNIT, 4)
        stored = build_stage(tree, catalog("laplace"), 9, 8, "stored")
        econ = build_stage(tree, catalog("laplace"), 9, 8, "econ")
        assert econ.memory_floats() < stored.memory_floats()
        assert econ.leaf_memory_floats() == 0 and stored.leaf_memory_floats() > 0
        assert econ.device_bytes() < stored.device_bytes()

    def test_econ_on_refined_mesh_and_repeat(self):
        spec = catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)")
        tree = build_uniform_tree(UNIT, 4)
        refine_near_point(tree, (0.5, 0.5), 1)
        us = build_stage(tree, spec, 9, 8, "stored").solve().u
        econ = build_stage(tree, spec, 9, 8, "econ")
        ue1, ue2 = econ.solve().u, econ.solve().u
        assert np.abs(us - ue1).max() <= 1e-12
        np.testing.assert_array_equal(ue1, ue2)

    def test_unknown_mode(self):
        with pytest.raises(ValueError, match="unknown mode"):
            build_stage(build_uniform_tree(UNIT, 1), catalog("laplace"), 9, 8, mode="compressed")


@pytest.mark.parametrize("n", [8, 32])
def test_overlapped_host_path_matches_eager_program(n):
    """The host-API path (graph up to the leaf step, leaf-range launches, reads overlapped on a
    side stream) gives bit-identical results to the eager one-launch-per-step program; n = 32
    gives 1024 leaves, i.e. 4 leaf ranges."""
    spec = catalog("varcoef_helmholtz", kappa=10.0)
    tree = build_uniform_tree(UNIT, n)
    a = build_stage(tree, spec, 12, 11)
    f = lambda pts: np.sin(2 * pts[:, 0] + pts[:, 1])
    g = lambda pts: np.cos(3 * pts[:, 0]) * pts[:, 1]
    sa = a.solve(f=f, g=g)
    assert len(a._program(1)["leaf_chunks"]) == (4 if n * n >= 4 * 148 else 1)
    a.use_graphs = False
    sb = a.solve(f=f, g=g)
    np.testing.assert_array_equal(sa.u, sb.u)
    np.testing.assert_array_equal(sa.w, sb.w)
    np.testing.assert_array_equal(sa.h_root, sb.h_root)
    for nid in sb.leaf_solutions:
        np.testing.assert_array_equal(sa.leaf_solutions[nid], sb.leaf_solutions[nid])
        np.testing.assert_array_equal(sa.g_tab[nid], sb.g_tab[nid])
    # result buffers: states that are kept alive are never overwritten by later solves
    a.use_graphs = True
    keep = [a.solve(f=f, g=lambda pts, s=s: s * g(pts)) for s in (1.0, 2.0, 3.0, 4.0)]
    for s_, st in zip((1.0, 2.0, 3.0, 4.0), keep):
        np.testing.assert_allclose(st.u, s_ * sa.u - (s_ - 1.0) * a.solve(f=f, g=lambda pts: 0 * g(pts)).u,
                                   rtol=0, atol=1e-12 * np.abs(sa.u).max())


class TestUnionDomains:
    """Reference test_solver.py:295-311 (harmonic data reproduced on an L-shaped forest)."""
    L = ((0.0, 1.0, 0.0, 1.0), (1.0, 2.0, 0.0, 1.0), (0.0, 1.0, 1.0, 2.0))

    @pytest.mark.parametrize("refine", [False, True])
    def test_harmonic_on_lshape(self, refine):
        from paper_1612_02736_b200 import build_forest
        tree = build_forest(self.L, 2)
        if refine:
            refine_near_point(tree, (1.0, 1.0), 1)
        p, q = (10, 9) if not refine else (9, 8)
        solver = build_stage(tree, catalog("laplace"), p, q)
        f = lambda pts: pts[:, 0] ** 2 - pts[:, 1] ** 2
        st = solver.solve(f=f)
        for lf in tree.leaves():
            pts = orc.leaf_points(lf.bounds, p, q)
            assert np.abs(st.leaf_solutions[lf.id] - f(pts)).max() <= 1e-10
        ref = orc.solve(orc.build(tree, catalog("laplace"), p, q, enumerate_gauss_nodes(tree, q)), f)
        assert rel_maxdiff(st.u, ref["u"]) <= 1e-10
