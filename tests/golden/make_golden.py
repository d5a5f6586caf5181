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


PROJ_SEED = 99


def proj_weights(n):
    """Fixed seeded projection vector (standard normal) of length n, shared with the tests."""
    return np.random.default_rng([PROJ_SEED, n]).standard_normal(n)


def cover_all(st, q):
    """Fingerprint that covers EVERY leaf and every Gauss segment: per leaf, the max-norm and a
    seeded random projection w . u_c of its tabulation; per edge segment (q nodes, global ids
    seg*q + k), a projection of its q values. A wrong value anywhere moves one of them."""
    ids = sorted(st.leaf_solutions)
    tabs = np.stack([st.leaf_solutions[i] for i in ids])
    u = np.asarray(st.u)
    return {"all_leaf_ids": np.array(ids), "all_leaf_absmax": np.abs(tabs).max(axis=1),
            "all_leaf_proj": tabs @ proj_weights(tabs.shape[1]),
            "seg_proj": u.reshape(-1, q) @ proj_weights(q)}


def be_loads_ref(tabs, tree, p, q, dt):
    g = {}
    for lf in tree.leaves():
        geo = leaf_geometry(p, q, lf.bounds.width, lf.bounds.height)
        g[lf.id] = np.asarray(tabs[lf.id])[geo.stencil0.i_ci] / dt
    return g


def initial_tabs(tree, p, q, seed):
    u0 = problems.config5_initial(seed=seed)
    tabs = {}
    for lf in tree.leaves():
        geo = leaf_geometry(p, q, lf.bounds.width, lf.bounds.height)
        tabs[lf.id] = u0(stencil_for(lf.bounds, geo).cheb2d)
    return tabs


def cfg5_trajectory_fixture(nrhs=16, steps=3):
    """Config 5 at its real shape, run by the reference: 128x128 leaves, p=16, dt=1e-3, the 16
    seeded initial fields (seeds 0..15), `steps` backward-Euler steps each through the reference's
    own FactorizedSolver.solve loop (solver.py:337-354; g = u_c[i_ci]/dt, f = sin(2 pi t) x1 (1-x2)).
    Per step: every leaf of every RHS enters an RHS-mixed projection sum_r c_r (w . u_c^r); per
    RHS, u on 500 seeded Gauss nodes and max-norms. At the last step: the RHS-mixed projection of
    every Gauss segment and four complete leaf tabulations per RHS."""
    import time
    dt, p, q = 1e-3, 16, 15
    tree = build_uniform_tree(UNIT, 128)
    t0 = time.perf_counter()
    solver = build_stage(tree, problems.config5_spec(dt), p, q)
    print(f"cfg5 build {time.perf_counter() - t0:.1f} s")
    rng = np.random.default_rng(515)
    ids = sorted(lf.id for lf in tree.leaves())
    upick = np.sort(rng.choice(solver.plan.n_gauss, size=500, replace=False))
    lpick = np.sort(rng.choice(len(ids), size=4, replace=False))
    cmix = np.random.default_rng([PROJ_SEED, 16, 1]).standard_normal(nrhs)
    wP = proj_weights(p * p)
    out = {"u_idx": upick, "leaf_pick": np.array([ids[i] for i in lpick]), "leaf_ids": np.array(ids),
           "mix_proj": np.zeros((steps, len(ids))), "u_vals": np.zeros((steps, nrhs, upick.size)),
           "u_max": np.zeros((steps, nrhs)), "leaf_max": np.zeros((steps, nrhs)),
           "mix_seg": np.zeros(solver.plan.n_gauss // q),
           "leaf_sol": np.zeros((nrhs, lpick.size, p * p)), "steps": np.array([steps]),
           "nrhs": np.array([nrhs])}
    for r in range(nrhs):
        t1 = time.perf_counter()
        tabs = initial_tabs(tree, p, q, r)
        for k in range(1, steps + 1):
            t = k * dt
            st = solver.solve(f=lambda pts, _t=t: problems.config5_dirichlet(pts, _t),
                              g=be_loads_ref(tabs, tree, p, q, dt))
            tabs = st.leaf_solutions
            T = np.stack([tabs[i] for i in ids])
            out["mix_proj"][k - 1] += cmix[r] * (T @ wP)
            out["u_vals"][k - 1, r] = st.u[upick]
            out["u_max"][k - 1, r] = np.abs(st.u).max()
            out["leaf_max"][k - 1, r] = np.abs(T).max()
        out["mix_seg"] += cmix[r] * (st.u.reshape(-1, q) @ proj_weights(q))
        out["leaf_sol"][r] = T[lpick]
        print(f"  rhs {r}: {time.perf_counter() - t1:.1f} s")
    save("full_cfg5_traj.npz", **out)


def cfg5_drift_fixture(n=16, steps=50):
    """Long single-RHS backward-Euler trajectory (seed 0) at n x n leaves, for drift: fingerprints
    after steps 1, 10 and `steps`, plus the complete u and all leaf tabulations at the end."""
    dt, p, q = 1e-3, 16, 15
    tree = build_uniform_tree(UNIT, n)
    solver = build_stage(tree, problems.config5_spec(dt), p, q)
    tabs = initial_tabs(tree, p, q, 0)
    ids = sorted(lf.id for lf in tree.leaves())
    keep = (1, 10, steps)
    out = {"leaf_ids": np.array(ids), "keep": np.array(keep), "n": np.array([n])}
    for k in range(1, steps + 1):
        t = k * dt
        st = solver.solve(f=lambda pts, _t=t: problems.config5_dirichlet(pts, _t),
                          g=be_loads_ref(tabs, tree, p, q, dt))
        tabs = st.leaf_solutions
        if k in keep:
            for key, v in cover_all(st, q).items():
                out[f"s{k}_{key}"] = v
            out[f"s{k}_u_max"] = np.array([np.abs(st.u).max()])
    out["u_final"] = st.u
    out["leaf_sol_final"] = np.stack([tabs[i] for i in ids])
    save(f"cfg5_drift_n{n}.npz", **out)


def resonance_fixture():
    """A Helmholtz wavenumber at an interface resonance of the first merge, found with the
    reference's own leaf operators: on a 2x2 mesh (p=12, q=11) box 2 = [0.5,1]x[0,1] has the
    Dirichlet eigenvalue 5 pi^2, so kappa ~ sqrt(5) pi makes Delta = T33_a - T33_b singular. A
    secant iteration drives the eigenvalue of Delta nearest zero to round-off, then the
    reference's build_stage is run to record the box and message it raises
    (MergeSingularError, solver.py:108-119)."""
    from specdtn.solver import MergeSingularError
    tree = build_uniform_tree(UNIT, 2)
    p, q = 12, 11
    plan = enumerate_gauss_nodes(tree, q)
    par = [n for n in range(len(tree.nodes) - 1, -1, -1) if not tree.nodes[n].is_leaf][0]
    ca, cb = tree.nodes[par].children
    en = plan.node[par]

    def lam(k):
        spec = catalog("helmholtz", kappa=k)
        ta = build_leaf_operators(tree.nodes[ca], spec, p, q).T
        tb = build_leaf_operators(tree.nodes[cb], spec, p, q).T
        w = np.linalg.eigvals(ta[np.ix_(en.pos3_a, en.pos3_a)] - tb[np.ix_(en.pos3_b, en.pos3_b)])
        return w[np.argmin(np.abs(w))].real

    a, b = np.sqrt(5.0) * np.pi * 0.9999, np.sqrt(5.0) * np.pi
    fa, fb = lam(a), lam(b)
    for _ in range(30):
        if fb == fa:
            break
        a, fa, b = b, fb, b - fb * (b - a) / (fb - fa)
        fb = lam(b)
        if abs(fb) < 1e-14:
            break
    try:
        build_stage(tree, catalog("helmholtz", kappa=b), p, q)
        raise SystemExit("reference did not raise at the resonant kappa")
    except MergeSingularError as exc:
        msg = str(exc)
    box = int(msg.split("box ")[1].split()[0])
    print("resonance", repr(b), msg)
    save("resonance.npz", kappa=np.array([b]), p=np.array([p]), q=np.array([q]), n=np.array([2]),
         box=np.array([box]), lam=np.array([fb]))


def archive_fixture():
    """Archives written by the reference's own persist_operators (archive.py:65-101), stored and
    economy mode on a refined mesh (wrapped parents), plus the reference's solves from the
    reloaded solvers, for the GPU loader's interop test."""
    from specdtn.archive import load_operators, persist_operators
    for mode in ("stored", "econ"):
        tree = build_uniform_tree(UNIT, 2)
        refine_near_point(tree, RefinementSpec((0.1, 0.1), 1))
        solver = build_stage(tree, catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)"), 9, 8, mode)
        path = os.path.join(HERE, f"ref_archive_{mode}.sdtn")
        persist_operators(solver, path)
        loaded = load_operators(path)
        st = loaded.solve()
        g = {lf.id: np.cos(np.arange((9 - 2) ** 2) * 0.1 + lf.id) for lf in tree.leaves()}
        st2 = loaded.solve(f=lambda pts: pts[:, 0] * pts[:, 1], g=g)
        a = state_arrays(st, loaded)
        for k, v in state_arrays(st2, loaded).items():
            a["fg_" + k] = v
        save(f"ref_archive_{mode}_solution.npz", **a)
        print(f"ref_archive_{mode}.sdtn: {os.path.getsize(path) / 1024:.1f} KiB")


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
        out.update(cover_all(st, q))
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
    if "--only-archive" in _sys.argv:
        archive_fixture()
        raise SystemExit
    if "--only-resonance" in _sys.argv:
        resonance_fixture()
        raise SystemExit
    if "--only-traj" in _sys.argv:
        cfg5_drift_fixture()
        cfg5_trajectory_fixture()
        raise SystemExit
    if "--only-full" in _sys.argv:
        fullsize_fixture()
        raise SystemExit
    cn_fixture()
    spectral_fixture()
    plan_fixture()
    leaf_fixture()
    solve_fixtures()
