"""The reference's behavioural tests for the build/solve path (pkg/tests/test_solver.py and the
acceptance criteria of pkg/tests/test_acceptance.py), restated against the B200 path with the
reference's own tolerances. Each test names the reference test it mirrors."""
import numpy as np
import pytest

from oracle import hps_oracle as orc
from paper_1612_02736_b200 import (ReferenceSolution, build_stage, build_uniform_tree, catalog, linf_error,
                                   refine_near_point)
from paper_1612_02736_b200.reference import state_boundary_values
from paper_1612_02736_b200.solver import downward_pass, solve, upward_pass

pytestmark = pytest.mark.gpu
UNIT = (0.0, 1.0, 0.0, 1.0)


def _tab_error(state, fn):
    """max over leaves of |u_leaf - fn(points)| (reference tests' tabulation_error)."""
    worst = 0.0
    tree, p, q = state.tree, state.p, state.q
    for lf in tree.leaves():
        pts = orc.leaf_points(lf.bounds, p, q)
        worst = max(worst, float(np.abs(np.asarray(state.leaf_solutions[lf.id]) - fn(pts)).max()))
    return worst


def test_single_leaf_tree():  # test_solver.py:95-99
    solver = build_stage(build_uniform_tree(UNIT, 1), catalog("laplace"), 10, 9)
    st = solver.solve(f=lambda pts: pts[:, 0])
    assert _tab_error(st, lambda pts: pts[:, 0]) <= 1e-12


def test_linearity():  # test_solver.py:113-122
    spec = catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)")
    solver = build_stage(build_uniform_tree(UNIT, 2), spec, 9, 8)
    full = solver.solve()
    f_only = solver.solve(g=lambda pts: np.zeros(len(pts)))
    g_only = solver.solve(f=lambda pts: np.zeros(len(pts)))
    scale = max(np.abs(full.u).max(), 1.0)
    assert np.abs(full.u - (f_only.u + g_only.u)).max() / scale <= 1e-12


def _normal_flux_exact(pts):
    pi = np.pi
    vertical = np.isclose(pts[:, 0], 0.0) | np.isclose(pts[:, 0], 1.0)
    return np.where(vertical, pi * np.cos(pi * pts[:, 0]) * np.sin(pi * pts[:, 1]),
                    pi * np.sin(pi * pts[:, 0]) * np.cos(pi * pts[:, 1]))


def test_upward_root_fluxes_manufactured():  # test_solver.py:140-151
    spec = catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)")
    solver = build_stage(build_uniform_tree(UNIT, 2), spec, 17, 16)
    st = upward_pass(solver)
    pts = solver.plan.coords[solver.plan.root_exterior()]
    np.testing.assert_allclose(st.h_root, _normal_flux_exact(pts), atol=1e-9)


def test_upward_interface_particular_solution():  # test_solver.py:153-163
    spec = catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)")
    tree = build_uniform_tree(UNIT, 2)
    solver = build_stage(tree, spec, 17, 16)
    st = upward_pass(solver)
    j3 = solver.plan.node[tree.root].j3
    pts = solver.plan.coords[j3]
    np.testing.assert_allclose(st.w[j3], np.sin(np.pi * pts[:, 0]) * np.sin(np.pi * pts[:, 1]), atol=1e-9)
    st = downward_pass(solver, None, st)
    assert _tab_error(st, spec.u_exact) <= 1e-9


def test_zero_load_upward_all_zero():  # test_solver.py:165-170
    solver = build_stage(build_uniform_tree(UNIT, 4), catalog("laplace"), 9, 8)
    st = upward_pass(solver)
    assert np.abs(st.h_root).max() == 0.0
    assert np.abs(st.w).max() == 0.0


def test_module_level_solve():  # test_solver.py:172-176
    solver = build_stage(build_uniform_tree(UNIT, 2), catalog("laplace"), 9, 8)
    st = solve(solver, f=lambda pts: pts[:, 1])
    assert _tab_error(st, lambda pts: pts[:, 1]) <= 1e-11


def test_interface_continuity():  # test_solver.py:178-204
    spec = catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)")
    tree = build_uniform_tree(UNIT, 4)
    p, q = 13, 12
    st = build_stage(tree, spec, p, q).solve()
    by_edge = {}
    for lf in tree.leaves():
        geo = orc.leaf_geometry(p, q, lf.bounds.width, lf.bounds.height)
        pts = orc.leaf_points(lf.bounds, p, q)
        vals = np.asarray(st.leaf_solutions[lf.id])
        for side in ("i_s", "i_e", "i_n", "i_w"):
            idx = geo[side]
            key = tuple(np.round(pts[idx], 12).ravel())
            by_edge.setdefault(key, []).append(vals[idx])
    shared = [c for c in by_edge.values() if len(c) == 2]
    assert len(shared) == 24  # interior edges of the 4x4 mesh
    assert max(np.abs(a - b).max() for a, b in shared) <= 1e-8


def test_merge_x_and_s_match_lu_form():  # test_solver.py:77-83 (X materialisation), :52-56
    """The GPU's explicit X (pivot column order + perm) inverts the interface block Delta of
    the oracle's children T maps, and its S matches the LU-based S."""
    p, q = 12, 11
    tree = build_uniform_tree(UNIT, 2)
    spec = catalog("varcoef_helmholtz", kappa=10.0)
    solver = build_stage(tree, spec, p, q)
    fns = orc.coef_functions(spec)
    grp = next(g for g in solver.parent_groups if g.depth == 1)
    for slot, nid in enumerate(grp.ids):
        ca, cb = tree.nodes[nid].children
        e = solver.plan.node[nid]
        ta = orc.leaf_ops(tree.nodes[ca].bounds, fns, p, q)["T"]
        tb = orc.leaf_ops(tree.nodes[cb].bounds, fns, p, q)["T"]
        delta = ta[np.ix_(e.pos3_a, e.pos3_a)] - tb[np.ix_(e.pos3_b, e.pos3_b)]
        m3 = grp.m3
        xs = grp.xs[slot].cpu().numpy()
        perm = grp.perm[slot].cpu().numpy()
        x = np.empty((m3, m3))
        x[:, perm] = xs[:, :m3]  # M[:, j] = inv[:, perm[j]]
        np.testing.assert_allclose(x @ delta, np.eye(m3), atol=1e-9)
        s_ref = orc.merge(ta, tb, e)["S"]
        assert np.abs(xs[:, m3:] - s_ref).max() <= 1e-10 * max(np.abs(s_ref).max(), 1.0)


def test_criterion_1_polynomial_exactness():  # test_acceptance.py:35-49
    spec = catalog("manufactured", u="x1**13 - 3*x1**5*x2**9 + 2*x2**13 - x1**2*x2**11 + x1*x2 - 4")
    ref = ReferenceSolution.analytic(spec.u_exact)
    worst = max(linf_error(build_stage(build_uniform_tree(UNIT, n), spec, 16, 15).solve(), ref) for n in (1, 2, 4))
    assert worst <= 1e-9


def test_criterion_2_manufactured_convergence():  # test_acceptance.py:52-66
    spec = catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)")
    ref = ReferenceSolution.analytic(spec.u_exact)
    errs = [linf_error(build_stage(build_uniform_tree(UNIT, n), spec, 9, 8).solve(), ref) for n in (2, 4, 8)]
    ratios = [errs[i] / errs[i + 1] for i in range(2)]
    assert all(r >= 100 for r in ratios) or errs[-1] <= 1e-10


def test_criterion_3_varcoef_helmholtz():  # test_acceptance.py:69-91
    spec = catalog("varcoef_helmholtz")
    ref_state = build_stage(build_uniform_tree(UNIT, 32), spec, 17, 16, "econ").solve()
    reference = ReferenceSolution.from_state(ref_state)
    amplitude = float(np.abs(state_boundary_values(ref_state)[1]).max())
    err_q4 = linf_error(build_stage(build_uniform_tree(UNIT, 16), spec, 5, 4).solve(), reference)
    err_q16 = linf_error(build_stage(build_uniform_tree(UNIT, 16), spec, 17, 16).solve(), reference)
    assert err_q4 > 1e-2 and err_q4 > 0.1 * amplitude
    assert err_q16 <= 1e-5


def test_criterion_4_discontinuous_aligned_load():  # test_acceptance.py:94-105
    spec = catalog("indicator_poisson")
    reference = ReferenceSolution.from_state(build_stage(build_uniform_tree(UNIT, 32), spec, 17, 16, "econ").solve())
    err = linf_error(build_stage(build_uniform_tree(UNIT, 16), spec, 17, 16).solve(), reference)
    assert err <= 1e-9


def test_criterion_5_refinement_parity():  # test_acceptance.py:108-131
    spec = catalog("concentrated_helmholtz")
    centre = tuple(spec.params["xhat"])

    def mesh(n, rounds):
        tree = build_uniform_tree(UNIT, n)
        if rounds:
            refine_near_point(tree, centre, rounds)
        return tree

    reference = ReferenceSolution.from_state(build_stage(mesh(16, 1), spec, 17, 16, "econ").solve())
    err_refined = linf_error(build_stage(mesh(4, 1), spec, 17, 16).solve(), reference)
    err_uniform = linf_error(build_stage(mesh(8, 0), spec, 17, 16).solve(), reference)
    assert err_refined <= 10 * err_uniform


def test_criterion_8_crank_nicolson_order():  # test_acceptance.py:171-195
    from paper_1612_02736_b200.problems import heat_exact, heat_problem
    from paper_1612_02736_b200.timestepping import TimeStepConfig, cn_run
    t_end = 0.1
    ks = [1 / 40, 1 / 80, 1 / 160, 1 / 320]
    errs, builds = [], 0
    for k in ks:
        run = cn_run(heat_problem(), build_uniform_tree(UNIT, 8), TimeStepConfig(k, t_end, (t_end,)), 9, 8)
        builds += run.build_count
        errs.append(linf_error(run.states[t_end], ReferenceSolution.analytic(lambda pts: heat_exact(pts, t_end))))
    slope = float(np.polyfit(np.log(ks), np.log(errs), 1)[0])
    assert abs(slope - 2.0) <= 0.3
    assert builds == len(ks)  # exactly one build per run


def test_criterion_10_shuffled_merge_order():  # test_acceptance.py:222-256 (second half)
    vspec = catalog("varcoef_helmholtz", kappa=10.0)
    t4 = build_uniform_tree(UNIT, 4)
    a = build_stage(t4, vspec, 9, 8)
    rng = np.random.default_rng(5)
    order = list(rng.permutation(len(t4.nodes)))
    order.sort(key=lambda nid: -t4.nodes[nid].level)
    b = build_stage(t4, vspec, 9, 8, order=order)
    f = lambda pts: np.sin(2 * pts[:, 0]) + pts[:, 1]
    assert np.abs(a.solve(f=f).u - b.solve(f=f).u).max() <= 1e-13
