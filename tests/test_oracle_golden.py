"""Pin the CPU oracle (oracle/hps_oracle.py) to golden vectors produced by the reference."""
import numpy as np
import pytest

from hps_testutil import golden, rel_maxdiff
from oracle import hps_oracle as orc
from paper_1612_02736_b200 import problems
from paper_1612_02736_b200.geometry import (build_balanced_refined_tree, build_uniform_tree,
                                            enumerate_gauss_nodes, refine_near_point)
from paper_1612_02736_b200.model import catalog

UNIT = (0.0, 1.0, 0.0, 1.0)


@pytest.mark.parametrize("name,p,q,n", [("laplace_p12", 12, 11, 1), ("varcoef_p16", 16, 15, 4),
                                         ("helm_p16", 16, 15, 16)])
def test_leaf_ops(name, p, q, n):
    g = golden("leaf.npz")
    spec = {"laplace_p12": catalog("laplace"), "varcoef_p16": problems.config2_spec(),
            "helm_p16": catalog("helmholtz", kappa=40.0)}[name]
    tree = build_uniform_tree(UNIT, n)
    leaf = tree.nodes[int(g[name + "_leaf"][0])]
    ops = orc.leaf_ops(leaf.bounds, orc.coef_functions(spec), p, q)
    assert rel_maxdiff(ops["T"], g[name + "_T"]) < 1e-12
    assert rel_maxdiff(ops["H"], g[name + "_H"]) < 1e-12
    assert rel_maxdiff(ops["S"] @ g[name + "_vb"], g[name + "_Sv"]) < 1e-12
    assert rel_maxdiff(ops["F"] @ g[name + "_vm"], g[name + "_Fv"]) < 1e-12


def _solve_check(fx, tree, spec, p, q, f=None, g=None, prefix="", tol=1e-11):
    plan = enumerate_gauss_nodes(tree, q)
    ops = orc.build(tree, spec, p, q, plan)
    st = orc.solve(ops, f, g)
    ids = fx[prefix + "leaf_ids"]
    sol = np.stack([st["leaf_solutions"][int(i)] for i in ids])
    assert rel_maxdiff(sol, fx[prefix + "leaf_sol"]) < tol
    assert rel_maxdiff(st["u"], fx[prefix + "u"]) < tol
    if np.abs(fx[prefix + "h_root"]).max() > 0:
        assert rel_maxdiff(st["h_root"], fx[prefix + "h_root"]) < tol
    return ops, st


def test_config1():
    fx = golden("cfg1.npz")
    tree = build_uniform_tree(UNIT, 4)
    ops, _ = _solve_check(fx, tree, problems.config1_spec(), 16, 15)
    gfn = problems.config1_random_load(0)
    st = orc.solve(ops, f=lambda pts: np.zeros(len(pts)), g=gfn)
    sol = np.stack([st["leaf_solutions"][int(i)] for i in fx["rand_leaf_ids"]])
    assert rel_maxdiff(sol, fx["rand_leaf_sol"]) < 1e-11


def test_config2_small():
    _solve_check(golden("cfg2_n4.npz"), build_uniform_tree(UNIT, 4), problems.config2_spec(), 16, 15)


def test_config3_small():
    _solve_check(golden("cfg3_n4.npz"), build_uniform_tree(UNIT, 4), problems.config3_spec(), 32, 31,
                 tol=1e-10)


def test_config4_small():
    tree = build_balanced_refined_tree(4, (0.3, 0.7), 3)
    _solve_check(golden("cfg4_small.npz"), tree, problems.config4_spec(), 16, 14)


def test_refined_reference_native():
    tree = build_uniform_tree(UNIT, 4)
    refine_near_point(tree, (0.5, 0.5), 1)
    _solve_check(golden("refined_r4.npz"), tree, catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)"), 9, 8)


def test_config5_small_backward_euler():
    fx = golden("cfg5_n4.npz")
    dt = 1e-3
    tree = build_uniform_tree(UNIT, 4)
    plan = enumerate_gauss_nodes(tree, 15)
    ops = orc.build(tree, problems.config5_spec(dt), 16, 15, plan)
    for r in range(2):
        u0 = problems.config5_initial(r)
        tabs = {lf.id: u0(orc.leaf_points(lf.bounds, 16, 15)) for lf in tree.leaves()}
        for step in (1, 2):
            t = step * dt
            st = orc.solve(ops, f=lambda pts, _t=t: problems.config5_dirichlet(pts, _t),
                           g=orc.be_loads(tabs, tree, 16, 15, dt))
            tabs = st["leaf_solutions"]
        sol = np.stack([tabs[i] for i in sorted(tabs)])
        assert rel_maxdiff(sol, fx[f"rhs{r}_leaf_sol"]) < 1e-11


def test_be_drift_50_steps():
    """The oracle reproduces the reference's 50-step backward-Euler trajectory (16x16 leaves,
    seed 0; tests/golden/cfg5_drift_n16.npz) — pins the BE harness the GPU drift test checks."""
    fx = golden("cfg5_drift_n16.npz")
    dt, p, q = 1e-3, 16, 15
    tree = build_uniform_tree(UNIT, int(fx["n"][0]))
    plan = enumerate_gauss_nodes(tree, q)
    ops = orc.build(tree, problems.config5_spec(dt), p, q, plan)
    u0 = problems.config5_initial(0)
    tabs = {lf.id: u0(orc.leaf_points(lf.bounds, p, q)) for lf in tree.leaves()}
    bpts = plan.coords[plan.node[tree.root].ext]
    for k in range(1, int(fx["keep"][-1]) + 1):
        st = orc.solve(ops, problems.config5_dirichlet(bpts, k * dt), orc.be_loads(tabs, tree, p, q, dt))
        tabs = st["leaf_solutions"]
    ids = fx["leaf_ids"]
    assert rel_maxdiff(np.stack([tabs[int(i)] for i in ids]), fx["leaf_sol_final"]) < 1e-11
    assert rel_maxdiff(st["u"], fx["u_final"]) < 1e-11
