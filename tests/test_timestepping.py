"""Time stepping on the GPU factorization (reference pkg/tests/test_timestepping.py inputs)."""
import numpy as np
import pytest

from hps_testutil import golden, rel_maxdiff
from oracle import hps_oracle as orc
from paper_1612_02736_b200 import build_stage, build_uniform_tree, catalog, problems
from paper_1612_02736_b200.model import CoefficientField
from paper_1612_02736_b200.timestepping import (ParabolicProblem, TimeStepConfig, cn_elliptic_spec, cn_rhs,
                                                cn_run, make_rhs_context)

UNIT = (0.0, 1.0, 0.0, 1.0)
PTS = np.array([[0.3, 0.4], [0.8, 0.1]])


class TestEllipticSpec:  # CPU: coefficient mapping (reference test_timestepping.py:17-47)
    def test_heat_mapping(self):
        spec = cn_elliptic_spec(problems.heat_problem(), 0.1)
        np.testing.assert_allclose(spec.coefficients.c11(PTS), 0.5)
        np.testing.assert_allclose(spec.coefficients.c22(PTS), 0.5)
        np.testing.assert_allclose(spec.coefficients.c(PTS), 10.0)

    def test_convection_diffusion_mapping(self):
        prob = ParabolicProblem.from_spec(catalog("convection_diffusion"))
        spec = cn_elliptic_spec(prob, 0.01)
        np.testing.assert_allclose(spec.coefficients.c11(PTS), 1 / 400)
        np.testing.assert_allclose(spec.coefficients.c1(PTS), 0.5)
        np.testing.assert_allclose(spec.coefficients.c(PTS), 100.0)

    def test_callable_coefficients_route(self):
        op = CoefficientField(lambda pts: -np.ones(len(pts)), 0, -1.0)
        prob = ParabolicProblem(operator=op, initial=lambda pts: np.zeros(len(pts)))
        spec = cn_elliptic_spec(prob, 0.5)
        np.testing.assert_allclose(spec.coefficients.c11(PTS), 0.5)
        np.testing.assert_allclose(spec.coefficients.c(PTS), 2.0)

    def test_rejects_bad_step(self):
        with pytest.raises(ValueError):
            cn_elliptic_spec(problems.heat_problem(), 0.0)

    def test_config_validation(self):
        with pytest.raises(ValueError):
            TimeStepConfig(-0.1, 1.0)
        cfg = TimeStepConfig(0.25, 1.0, (0.3, 1.0))
        assert cfg.steps == 4
        assert cfg.record_steps() == {1, 4}


def _tabulate(tree, p, q, fn):
    return {lf.id: fn(orc.leaf_points(lf.bounds, p, q)) for lf in tree.leaves()}


@pytest.mark.gpu
class TestRhs:
    def test_zero_state(self):
        tree = build_uniform_tree(UNIT, 2)
        ctx = make_rhs_context(problems.heat_problem(), tree, 9, 8)
        out = cn_rhs(problems.heat_problem(), 0.1, _tabulate(tree, 9, 8, lambda p_: np.zeros(len(p_))), ctx)
        assert all(np.abs(v).max() == 0.0 for v in out.values())

    def test_linear_state(self):
        tree = build_uniform_tree(UNIT, 2)
        k = 0.2
        ctx = make_rhs_context(problems.heat_problem(), tree, 9, 8)
        out = cn_rhs(problems.heat_problem(), k, _tabulate(tree, 9, 8, lambda p_: p_[:, 0]), ctx)
        for lf in tree.leaves():
            geo = orc.leaf_geometry(9, 8, lf.bounds.width, lf.bounds.height)
            expect = orc.leaf_points(lf.bounds, 9, 8)[geo["i_ci"], 0] / k
            np.testing.assert_allclose(out[lf.id], expect, atol=1e-10)

    def test_sine_mode(self):
        tree = build_uniform_tree(UNIT, 4)
        k, p, q = 0.05, 13, 12
        fn = lambda pts: np.sin(np.pi * pts[:, 0]) * np.sin(np.pi * pts[:, 1])
        ctx = make_rhs_context(problems.heat_problem(), tree, p, q)
        out = cn_rhs(problems.heat_problem(), k, _tabulate(tree, p, q, fn), ctx)
        for lf in tree.leaves():
            geo = orc.leaf_geometry(p, q, lf.bounds.width, lf.bounds.height)
            expect = (1 / k - np.pi ** 2) * fn(orc.leaf_points(lf.bounds, p, q)[geo["i_ci"]])
            np.testing.assert_allclose(out[lf.id], expect, atol=1e-9)

    def test_variable_operator_vs_dense(self):
        # all six coefficients active: compare with the dense collocation matrix of the oracle
        op = CoefficientField("1 + x1*x2", "x1/5", "1 + x2**2", "sin(x1)", "cos(x2)", "x1 - x2")
        prob = ParabolicProblem(operator=op, initial=lambda pts: np.zeros(len(pts)))
        tree = build_uniform_tree(UNIT, 2)
        p, q, k = 10, 9, 0.3
        fn = lambda pts: np.exp(pts[:, 0]) * np.cos(2 * pts[:, 1])
        out = cn_rhs(prob, k, _tabulate(tree, p, q, fn), make_rhs_context(prob, tree, p, q))
        fns = (op.c11, op.c12, op.c22, op.c1, op.c2, op.c)
        for lf in tree.leaves():
            geo = orc.leaf_geometry(p, q, lf.bounds.width, lf.bounds.height)
            pts = orc.leaf_points(lf.bounds, p, q)
            a = orc.assemble(fns, pts, geo)
            u = fn(pts)
            expect = (u / k + 0.5 * (a @ u))[geo["i_ci"]]
            assert rel_maxdiff(out[lf.id], expect) <= 1e-12


@pytest.mark.gpu
class TestRun:
    def test_zero_everything_stays_zero(self):
        prob = ParabolicProblem(operator=CoefficientField(-1.0, 0.0, -1.0), initial=lambda pts: np.zeros(len(pts)))
        run = cn_run(prob, build_uniform_tree(UNIT, 2), TimeStepConfig(0.05, 0.2, (0.1, 0.2)), 9, 8)
        for state in run.states.values():
            assert max(np.abs(v).max() for v in state.leaf_solutions.values()) == 0.0

    def test_single_build_many_steps(self):
        run = cn_run(problems.heat_problem(), build_uniform_tree(UNIT, 2), TimeStepConfig(0.01, 0.1), 9, 8)
        assert run.build_count == 1
        assert len(run.step_seconds) == 10

    def test_second_order_convergence(self):
        t_end = 0.1
        errs = []
        ks = [1 / 20, 1 / 40, 1 / 80]
        for k in ks:
            tree = build_uniform_tree(UNIT, 4)
            run = cn_run(problems.heat_problem(), tree, TimeStepConfig(k, t_end, (t_end,)), 9, 8)
            st = run.states[t_end]
            err = 0.0
            for lf in tree.leaves():
                geo = orc.leaf_geometry(9, 8, lf.bounds.width, lf.bounds.height)
                pts = orc.leaf_points(lf.bounds, 9, 8)[geo["i_ce"]]
                err = max(err, np.abs(st.leaf_solutions[lf.id][geo["i_ce"]] - problems.heat_exact(pts, t_end)).max())
            errs.append(err)
        slope = np.polyfit(np.log(ks), np.log(errs), 1)[0]
        assert slope == pytest.approx(2.0, abs=0.3)

    def test_matches_reference_golden(self):
        fx = golden("cn_heat.npz")
        tree = build_uniform_tree(UNIT, 2)
        run = cn_run(problems.heat_problem(), tree, TimeStepConfig(0.05, 0.2, (0.2,)), 9, 8)
        st = run.states[0.2]
        sol = np.stack([st.leaf_solutions[int(i)] for i in fx["leaf_ids"]])
        assert rel_maxdiff(sol, fx["leaf_sol"]) <= 1e-10

    def test_csv_snapshots(self, tmp_path):
        run = cn_run(problems.heat_problem(), build_uniform_tree(UNIT, 2), TimeStepConfig(0.05, 0.1, (0.05, 0.1)), 9, 8)
        out = tmp_path / "traj.csv"
        run.write_csv(out)
        lines = out.read_text().strip().splitlines()
        assert lines[0] == "time,x1,x2,u"
        assert len(lines) == 1 + 2 * run.solver.plan.n_gauss


@pytest.mark.gpu
def test_backward_euler_multi_rhs_matches_golden():
    import torch
    from paper_1612_02736_b200.timestepping import _leaf_points, be_run
    fx = golden("cfg5_n4.npz")
    dt = 1e-3
    tree = build_uniform_tree(UNIT, 4)
    solver = build_stage(tree, problems.config5_spec(dt), 16, 15)
    pts = _leaf_points(solver)
    u0 = np.stack([problems.config5_initial(r)(pts.reshape(-1, 2)).reshape(solver._n_leaves, -1)
                   for r in range(2)], axis=-1)
    bpts = solver.plan.coords[solver.plan.node[tree.root].ext]
    dirichlet = lambda t: torch.as_tensor(np.repeat(problems.config5_dirichlet(bpts, t)[:, None], 2, axis=1),
                                          device="cuda")
    st = be_run(solver, torch.as_tensor(u0, device="cuda"), dirichlet, dt, 2)
    tabs = st.leaf_tabulations().cpu().numpy()
    order = np.argsort(solver._leaf_ids)
    for r in range(2):
        assert rel_maxdiff(tabs[order, :, r], fx[f"rhs{r}_leaf_sol"]) <= 1e-10
