"""Generate golden fixtures by running the REFERENCE implementation (specdtn) itself.

Run in the build container (the reference exists only there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small ``.npz`` files next to this script. They pin (a) this package's host
constants/plan and (b) the CPU oracle; the GPU parity tests then compare the CUDA path
with the pinned oracle and with these vectors. Nothing here runs on the GPU box.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from specdtn import spectral as rs  # noqa: E402  (reference)
from specdtn.geometry import (RefinementSpec, build_uniform_tree, enumerate_gauss_nodes,  # noqa: E402
                              refine_near_point)
from specdtn.leaf import build_leaf_operators, leaf_geometry, stencil_for  # noqa: E402
from specdtn.model import CoefficientField, ProblemSpec, catalog  # noqa: E402
from specdtn.reference import ReferenceSolution, linf_error  # noqa: E402
from specdtn.solver import build_stage  # noqa: E402

from paper_1612_02736_b200.geometry import build_balanced_refined_tree  # noqa: E402
from paper_1612_02736_b200 import problems  # noqa: E402

UNIT = (0.0, 1.0, 0.0, 1.0)


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1024:.1f} KiB")


def spectral_fixture():
    out = {}
    for p, q, w, h in ((16, 15, 0.25, 0.25), (12, 11, 1.0, 1.0), (9, 8, 0.5, 0.25),
                       (16, 14, 1.0 / 2048, 1.0 / 2048), (32, 31, 1.0 / 32, 1.0 / 32)):
        key = f"p{p}q{q}w{w!r}h{h!r}"
        box = (0.0, w, 0.0, h)
        st = rs.leaf_stencil(p, q, box)
        d1, d2 = rs.tensor_diff_matrices(p, box)
        lift = rs.build_boundary_lift(p, q, box)
        flux = rs.build_flux_extractor(st, d1, d2)
        out[key + "_lift"] = lift
        out[key + "_dx"] = rs.diff_matrix_1d(rs.chebyshev_nodes(p, rs.Interval(0.0, w)))
        out[key + "_i_ce"] = st.i_ce
        out[key + "_i_ci"] = st.i_ci
        if p <= 16:
            out[key + "_flux"] = flux
        else:  # keep the fixture small: flux action on a seeded vector
            v = np.random.default_rng(5).standard_normal(p * p)
            out[key + "_fluxv"] = flux @ v
    for q in (8, 14):
        up, down = rs.build_edge_interpolators(q)
        out[f"edge{q}_up"] = up
        out[f"edge{q}_down"] = down
    save("spectral.npz", **out)


def plan_arrays(plan, tree):
    out = {"coords": plan.coords}
    for nid, e in plan.node.items():
        out[f"n{nid}_ext"] = e.ext
        out[f"n{nid}_extmo"] = e.ext_mergeorder
        if not tree.nodes[nid].is_leaf:
            for k in ("j3", "pos1_a", "pos3_a", "pos2_b", "pos3_b"):
                out[f"n{nid}_{k}"] = getattr(e, k)
            if e.wrap is not None:
                out[f"n{nid}_wperm"] = e.wrap.perm
                out[f"n{nid}_wfine"] = e.wrap.fine
                out[f"n{nid}_wext"] = e.wrap.ext
                out[f"n{nid}_wblocks"] = np.array([0 if b[0] == "identity" else 1 for b in e.wrap.blocks])
    return out


def plan_fixture():
    out = {}
    t = build_uniform_tree(UNIT, 4)
    for k, v in plan_arrays(enumerate_gauss_nodes(t, 15), t).items():
        out["u4q15_" + k] = v
    t = build_uniform_tree(UNIT, 4)
    refine_near_point(t, RefinementSpec((0.5, 0.5), 1))
    for k, v in plan_arrays(enumerate_gauss_nodes(t, 8), t).items():
        out["r4q8_" + k] = v
    t = build_balanced_refined_tree(8, (0.3, 0.7), 8, tree_factory=build_uniform_tree)
    for k, v in plan_arrays(enumerate_gauss_nodes(t, 14), t).items():
        out["cfg4q14_" + k] = v
    from specdtn.geometry import build_forest
    lshape = ((0.0, 1.0, 0.0, 1.0), (1.0, 2.0, 0.0, 1.0), (0.0, 1.0, 1.0, 2.0))
    t = build_forest(lshape, 2)
    refine_near_point(t, RefinementSpec((1.0, 1.0), 1))
    for k, v in plan_arrays(enumerate_gauss_nodes(t, 8), t).items():
        out["lshape_" + k] = v
    save("plans.npz", **out)


def leaf_fixture():
    out = {}
    rng = np.random.default_rng(7)
    cases = {
        "laplace_p12": (catalog("laplace"), 12, 11, 1),
        "varcoef_p16": (problems.config2_spec(), 16, 15, 4),
        "helm_p16": (catalog("helmholtz", kappa=40.0), 16, 15, 16),
    }
    for name, (spec, p, q, n) in cases.items():
        tree = build_uniform_tree(UNIT, n)
        leaf = tree.leaves()[min(5, len(tree.leaves()) - 1)]
        ops = build_leaf_operators(leaf, spec, p, q)
        out[name + "_leaf"] = np.array([leaf.id])
        out[name + "_T"] = ops.T
        out[name + "_H"] = ops.H
        vb = rng.standard_normal(4 * q)
        vm = rng.standard_normal((p - 2) ** 2)
        out[name + "_vb"] = vb
        out[name + "_vm"] = vm
        out[name + "_Sv"] = ops.S @ vb
        out[name + "_Fv"] = ops.F @ vm
        if p <= 12:
            out[name + "_S"] = ops.S
            out[name + "_F"] = ops.F
    save("leaf.npz", **out)


def state_arrays(state, solver):
    ids = sorted(state.leaf_solutions)
    return {"u": state.u, "w": state.w, "h_root": state.h_root, "leaf_ids": np.array(ids),
            "leaf_sol": np.stack([state.leaf_solutions[i] for i in ids]),
            "g_tab": np.stack([state.g_tab[i] for i in ids]),
            "root_ext": solver.plan.root_exterior()}


def solve_fixtures():
    # config 1 (full size): Poisson 4x4, p=16, manufactured harmonic u
    spec = problems.config1_spec()
    tree = build_uniform_tree(UNIT, 4)
    solver = build_stage(tree, spec, 16, 15)
    st = solver.solve()
    err = linf_error(st, ReferenceSolution.analytic(spec.u_exact))
    a = state_arrays(st, solver)
    a["linf_error"] = np.array([err])
    # random-RHS variant: 8 Gaussians, f = 0
    gfn = problems.config1_random_load(seed=0)
    st2 = solver.solve(f=lambda pts: np.zeros(len(pts)), g=gfn)
    for k, v in state_arrays(st2, solver).items():
        a["rand_" + k] = v
    save("cfg1.npz", **a)

    # config 2 shape at reduced size (n=4): variable coefficients, manufactured solution
    spec = problems.config2_spec()
    tree = build_uniform_tree(UNIT, 4)
    solver = build_stage(tree, spec, 16, 15)
    st = solver.solve()
    a = state_arrays(st, solver)
    a["linf_error"] = np.array([linf_error(st, ReferenceSolution.analytic(spec.u_exact))])
    save("cfg2_n4.npz", **a)

    # config 3 shape at reduced size (n=4, p=32): oscillatory Helmholtz, plane-wave data
    spec = problems.config3_spec()
    tree = build_uniform_tree(UNIT, 4)
    solver = build_stage(tree, spec, 32, 31)
    st = solver.solve()
    save("cfg3_n4.npz", **state_arrays(st, solver))

    # config 4 shape at reduced size: base 4x4, 3 rounds toward (0.3, 0.7), q=14
    spec = problems.config4_spec()
    tree = build_balanced_refined_tree(4, (0.3, 0.7), 3, tree_factory=build_uniform_tree)
    solver = build_stage(tree, spec, 16, 14)
    st = solver.solve()
    a = state_arrays(st, solver)
    a["n_leaves"] = np.array([len(tree.leaves())])
    save("cfg4_small.npz", **a)

    # refined mesh from the reference's own refine_near_point (wraps), manufactured
    spec = catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)")
    tree = build_uniform_tree(UNIT, 4)
    refine_near_point(tree, RefinementSpec((0.5, 0.5), 1))
    solver = build_stage(tree, spec, 9, 8)
    st = solver.solve()
    a = state_arrays(st, solver)
    a["linf_error"] = np.array([linf_error(st, ReferenceSolution.analytic(spec.u_exact))])
    save("refined_r4.npz", **a)

    # config 5 shape at reduced size: backward Euler n=4, dt=1e-3, 2 steps, 2 RHS
    dt = 1e-3
    spec = problems.config5_spec(dt)
    tree = build_uniform_tree(UNIT, 4)
    solver = build_stage(tree, spec, 16, 15)
    a = {}
    for r in range(2):
        u0 = problems.config5_initial(seed=r)
        tabs = {}
        for lf in tree.leaves():
            geo = leaf_geometry(16, 15, lf.bounds.width, lf.bounds.height)
            tabs[lf.id] = u0(stencil_for(lf.bounds, geo).cheb2d)
        for step in range(1, 3):
            t = step * dt
            g = {}
            for lf in tree.leaves():
                geo = leaf_geometry(16, 15, lf.bounds.width, lf.bounds.height)
                g[lf.id] = tabs[lf.id][geo.stencil0.i_ci] / dt
            st = solver.solve(f=lambda pts, _t=t: problems.config5_dirichlet(pts, _t), g=g)
            tabs = st.leaf_solutions
        ids = sorted(tabs)
        a[f"rhs{r}_leaf_sol"] = np.stack([tabs[i] for i in ids])
        a[f"rhs{r}_u"] = st.u
    save("cfg5_n4.npz", **a)


def fullsize_fixture():
    """BASELINE configs 2-5 at their full sizes, run by the reference itself. The full solutions
    are too large to commit, so the fixture keeps a fingerprint: norms of u, u on 2000 seeded
    Gauss nodes, the complete tabulations of 24 seeded leaves, and (config 2) the error against
    the manufactured solution."""
    rng = np.random.default_rng(2024)

    def fingerprint(tag, tree, spec, p, q, solve_kw=None, extra=None):
        import time
        t0 = time.perf_counter()
        solver = build_stage(tree, spec, p, q)
        st = solver.solve(**(solve_kw or {}))
        ids = sorted(st.leaf_solutions)
        pick = np.sort(rng.choice(len(ids), size=min(24, len(ids)), replace=False))
        upick = np.sort(rng.choice(len(st.u), size=min(2000, len(st.u)), replace=False))
        out = {"u_idx": upick, "u_vals": st.u[upick], "u_max": np.array([np.abs(st.u).max()]),
               "u_l2": np.array([np.linalg.norm(st.u)]), "leaf_ids": np.array([ids[i] for i in pick]),
               "leaf_sol": np.stack([st.leaf_solutions[ids[i]] for i in pick]),
               "leaf_max": np.array([max(np.abs(v).max() for v in st.leaf_solutions.values())])}
        if spec.u_exact is not None:
            out["linf_error"] = np.array([linf_error(st, ReferenceSolution.analytic(spec.u_exact))])
        out.update(extra or {})
        save(f"full_{tag}.npz", **out)
        print(tag, f"{time.perf_counter() - t0:.1f} s")

    fingerprint("cfg2", build_uniform_tree(UNIT, 64), problems.config2_spec(), 16, 15)
    fingerprint("cfg3", build_uniform_tree(UNIT, 32), problems.config3_spec(), 32, 31)
    fingerprint("cfg4", build_balanced_refined_tree(8, (0.3, 0.7), 8, tree_factory=build_uniform_tree),
                problems.config4_spec(), 16, 14)
    # config 5: the first backward-Euler step of RHS 0 (g = u0[i_ci] / dt, f at t = dt)
    dt = 1e-3
    tree = build_uniform_tree(UNIT, 128)
    u0 = problems.config5_initial(seed=0)
    g = {}
    for lf in tree.leaves():
        geo = leaf_geometry(16, 15, lf.bounds.width, lf.bounds.height)
        g[lf.id] = u0(stencil_for(lf.bounds, geo).cheb2d)[geo.stencil0.i_ci] / dt
    fingerprint("cfg5", tree, problems.config5_spec(dt), 16, 15,
                solve_kw={"f": lambda pts: problems.config5_dirichlet(pts, dt), "g": g})


def cn_fixture():
    from specdtn.experiments import heat_problem
    from specdtn.timestepping import TimeStepConfig, cn_run
    tree = build_uniform_tree(UNIT, 2)
    run = cn_run(heat_problem(), tree, TimeStepConfig(0.05, 0.2, (0.2,)), 9, 8)
    st = run.states[0.2]
    ids = sorted(st.leaf_solutions)
    save("cn_heat.npz", leaf_ids=np.array(ids), leaf_sol=np.stack([st.leaf_solutions[i] for i in ids]))


if __name__ == "__main__":
    import sys as _sys
    if "--only-cn" in _sys.argv:
        cn_fixture()
        raise SystemExit
    if "--only-plans" in _sys.argv:
        plan_fixture()
        raise SystemExit
    if "--only-full" in _sys.argv:
        fullsize_fixture()
        raise SystemExit
    cn_fixture()
    spectral_fixture()
    plan_fixture()
    leaf_fixture()
    solve_fixtures()
