"""Implicit time stepping on one GPU-resident factorization (reference timestepping.py).

For du/dt = A u with time-independent coefficients (A in the elliptic sign convention):

  Crank–Nicolson   ((1/k) I - A/2) u_{n+1} = ((1/k) I + A/2) u_n         cn_run (timestepping.py:199-240)
  backward Euler   ((1/k) I - A)   u_{n+1} = (1/k) u_n                    be_run (config 5 harness)

The elliptic operator is built once (``build_stage``); every step is one ``hps_leaf_apply``
launch per leaf shape (the explicit side, computed from the previous step's leaf tabulations
that never leave HBM) followed by one replay of the CUDA-graph solve. Multi-RHS stepping
(config 5: 16 independent trajectories) runs all right-hand sides in the same launches.
"""

from __future__ import annotations

import csv
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _ext
from . import coeffs as coeff_mod
from . import solver as solver_mod
from .model import CoefficientField, ProblemSpec
from .solver import FactorizedSolver, SolveState


@dataclass(frozen=True)
class TimeStepConfig:
    """Step size, final time, recorded times (reference timestepping.py:36-60)."""

    k: float
    t_end: float
    record_times: tuple = ()

    def __post_init__(self):
        if not self.k > 0:
            raise ValueError(f"step size must be positive, got {self.k}")
        if self.t_end < 0:
            raise ValueError("final time must be nonnegative")

    @property
    def steps(self) -> int:
        return int(round(self.t_end / self.k))

    def record_steps(self) -> set[int]:
        return {min(self.steps, max(0, int(round(t / self.k)))) for t in self.record_times}


@dataclass
class ParabolicProblem:
    """du/dt = A u, u(.,0) = initial, Dirichlet f(pts, t) (reference timestepping.py:63-87)."""

    operator: CoefficientField
    initial: object
    dirichlet: object | None = None
    name: str = "parabolic"
    params: dict = field(default_factory=dict)

    @staticmethod
    def from_spec(spec: ProblemSpec, dirichlet=None) -> "ParabolicProblem":
        if spec.initial is None:
            raise ValueError(f"catalog entry {spec.name!r} has no initial condition")
        return ParabolicProblem(operator=spec.coefficients, initial=spec.initial, dirichlet=dirichlet,
                                name=spec.name, params=dict(spec.params))


def cn_elliptic_spec(problem: ParabolicProblem, k: float) -> ProblemSpec:
    """Coefficients of (1/k) I - (1/2) A (reference timestepping.py:90-114)."""
    if not k > 0:
        raise ValueError(f"step size must be positive, got {k}")
    a = problem.operator
    try:
        ce = a.symbolic()
        cf = CoefficientField(c11=-ce["c11"] / 2, c12=-ce["c12"] / 2, c22=-ce["c22"] / 2,
                              c1=-ce["c1"] / 2, c2=-ce["c2"] / 2, c=1.0 / k - ce["c"] / 2)
    except ValueError:
        def half_neg(fn):
            return lambda pts, _fn=fn: -0.5 * _fn(pts)
        cf = CoefficientField(half_neg(a.c11), half_neg(a.c12), half_neg(a.c22), half_neg(a.c1),
                              half_neg(a.c2), lambda pts, _fn=a.c: 1.0 / k - 0.5 * _fn(pts))
    return ProblemSpec(name=f"cn:{problem.name}", coefficients=cf, params={"k": k, **problem.params})


class RhsContext:
    """Device data for the explicit side on the leaves of a tree (reference
    timestepping.py:117-141 _RhsContext): per leaf shape, the 1D operators and the coefficient
    samples of the parabolic generator A. Leaf order = the solver's leaf-row order (leaf
    shapes grouped by first occurrence in id order, ids ascending within a shape).
    problem=None: no operator term (only alpha*u, backward Euler)."""

    def __init__(self, problem: ParabolicProblem | None, tree, p: int, q: int, device=None):
        from .spectral import shape_constants
        self.p, self.q = p, q
        dev = device or torch.device("cuda", torch.cuda.current_device())
        groups: dict = {}
        for nid, node in enumerate(tree.nodes):
            if node.is_leaf:
                key = (node.bounds.x1hi - node.bounds.x1lo, node.bounds.x2hi - node.bounds.x2lo)
                groups.setdefault(key, []).append(nid)
        self.groups = []
        self.leaf_ids = []
        row = 0
        for key, ids in groups.items():
            sc = shape_constants(p, q, float(key[0]), float(key[1]))
            consts = {k: torch.as_tensor(np.ascontiguousarray(getattr(sc, k)), dtype=torch.float64, device=dev)
                      for k in ("dx", "dy", "dxx", "dyy")}
            coef = None
            if problem is not None:
                org = torch.as_tensor(np.array([[tree.nodes[n].bounds.x1lo, tree.nodes[n].bounds.x2lo]
                                                for n in ids]), dtype=torch.float64, device=dev)
                pts = torch.as_tensor(sc.cheb2d(), dtype=torch.float64, device=dev)[None] + org[:, None, :]
                coef = coeff_mod.evaluate(problem.operator, pts).contiguous()
            self.groups.append(dict(ids=ids, first_row=row, consts=consts, coef=coef))
            self.leaf_ids.extend(ids)
            row += len(ids)
        self.n_leaves = row

    def apply_ptr(self, u: int, g: int, nrhs: int, alpha: float, beta: float):
        """g <- alpha u + beta A u for all leaves; u: (n_leaves, P, nrhs), g: (n_leaves, m, nrhs)
        device buffers given as raw pointers (leaf-row order)."""
        if beta != 0.0 and any(gr["coef"] is None for gr in self.groups):
            raise ValueError("this context has no operator (problem=None)")
        lib = _ext.load()
        p, m, P = self.p, (self.p - 2) ** 2, self.p ** 2
        stream = torch.cuda.current_stream().cuda_stream
        for gr in self.groups:
            cs = gr["consts"]
            args = _ext.LeafApplyArgs(len(gr["ids"]), p, nrhs, alpha, beta,
                                      gr["coef"].data_ptr() if beta != 0.0 else 0,
                                      cs["dx"].data_ptr(), cs["dy"].data_ptr(), cs["dxx"].data_ptr(),
                                      cs["dyy"].data_ptr(), u + 8 * gr["first_row"] * P * nrhs, P * nrhs,
                                      g + 8 * gr["first_row"] * m * nrhs, m * nrhs)
            _ext.check(lib.hps_leaf_apply(args, stream), "leaf apply")

    def apply(self, u: torch.Tensor, alpha: float, beta: float) -> torch.Tensor:
        """(n_leaves, P, nrhs) tabulations -> (n_leaves, m, nrhs) interior right-hand sides."""
        u = u.contiguous()
        nrhs = u.shape[-1]
        g = torch.empty((self.n_leaves, (self.p - 2) ** 2, nrhs), dtype=torch.float64, device=u.device)
        self.apply_ptr(u.data_ptr(), g.data_ptr(), nrhs, alpha, beta)
        return g


def make_rhs_context(problem: ParabolicProblem, tree, p: int, q: int) -> RhsContext:
    """Reference timestepping.py:159-161."""
    return RhsContext(problem, tree, p, q)


class DeviceStepper:
    """Device-resident stepping loop: each step = hps_leaf_apply + graph-replayed solve.

    alpha, beta: explicit side alpha*u + beta*A u (CN: 1/k, 1/2; BE: 1/k, 0).
    """

    def __init__(self, solver: FactorizedSolver, nrhs: int, alpha: float, beta: float,
                 ctx: RhsContext | None = None):
        if beta != 0.0 and ctx is None:
            raise ValueError("an explicit operator term needs an RhsContext")
        self.solver, self.nrhs, self.alpha, self.beta = solver, nrhs, alpha, beta
        self.ctx = ctx if ctx is not None else RhsContext(None, solver.tree, solver.p, solver.q, solver.device)
        if self.ctx.leaf_ids != list(solver._leaf_ids):
            raise ValueError("time-stepping context and solver disagree on the leaf order")
        # backward Euler with several right-hand sides: the solve's leaf steps read g = alpha u_n
        # straight from the leaf tabulations (one launch and 2 m doubles per leaf per RHS saved);
        # Crank-Nicolson (beta != 0) forms its load with hps_leaf_apply
        self.fold = beta == 0.0 and nrhs >= 3 and os.environ.get("HPS_BE_FOLD", "1") != "0"
        self.prog = solver._program(nrhs, be_alpha=alpha if self.fold else None)
        self.lay = solver._layout
        # folded program: the state alternates between two tabulation regions (parity = the
        # region holding the current state, read by the next step)
        self.parity = 0

    @property
    def pool(self):
        return self.prog["pool"]

    def leaf_tabulations(self) -> torch.Tensor:
        """(n_leaves, P, nrhs) view of the current leaf solutions (leaf-row order)."""
        s = self.solver
        P = s.p ** 2
        r0 = self.prog["uc_regions"][self.parity]
        return self.pool[r0:r0 + s._n_leaves * P].view(s._n_leaves, P, self.nrhs)

    def set_state(self, u_tabs: torch.Tensor):
        self.leaf_tabulations().copy_(u_tabs.reshape(self.leaf_tabulations().shape))

    def step(self, f: torch.Tensor):
        """Advance one step with Dirichlet data f ((|root ext|, nrhs), device) at t_{n+1}."""
        s, lay, n = self.solver, self.lay, self.nrhs
        if not self.fold:
            base = self.pool.data_ptr()
            self.ctx.apply_ptr(base + 8 * n * lay["UC"], base + 8 * n * lay["G"], n, self.alpha, self.beta)
        self.prog["f_in"].copy_(f.reshape(-1, self.nrhs))
        if self.fold:
            self.solver._execute(self.prog, parity=self.parity)
            self.parity ^= 1
        else:
            self.solver._execute(self.prog)


def _leaf_points(solver: FactorizedSolver) -> np.ndarray:
    """(n_leaves, P, 2) Chebyshev points in leaf-row order."""
    tree = solver.tree
    out = np.empty((solver._n_leaves, solver.p ** 2, 2))
    for grp in solver.leaf_groups:
        pts0 = grp.sc.cheb2d()
        for slot, nid in enumerate(grp.ids):
            b = tree.nodes[nid].bounds
            out[grp.first_row + slot] = pts0 + np.array([b.x1lo, b.x2lo])
    return out


def cn_rhs(problem: ParabolicProblem, k: float, u_tabs: dict, ctx: RhsContext) -> dict:
    """Interior tabulations of (1/k) u_n + (1/2) A u_n per leaf (reference timestepping.py:143-156)."""
    tabs = np.stack([np.asarray(u_tabs[n], dtype=float) for n in ctx.leaf_ids])
    u = torch.as_tensor(tabs, dtype=torch.float64).cuda().reshape(ctx.n_leaves, -1, 1)
    g = ctx.apply(u, 1.0 / k, 0.5)[:, :, 0].cpu().numpy()
    return {nid: g[i] for i, nid in enumerate(ctx.leaf_ids)}


@dataclass
class CnRun:
    """Trajectory of one Crank–Nicolson integration (reference timestepping.py:170-196)."""

    config: TimeStepConfig
    times: list
    states: dict
    build_count: int
    build_seconds: float
    step_seconds: list
    solver: FactorizedSolver

    def write_csv(self, path):
        coords = self.solver.plan.coords
        with open(path, "w", newline="") as fh:
            writer = csv.writer(fh)
            writer.writerow(["time", "x1", "x2", "u"])
            for t in sorted(self.states):
                u = self.states[t].u
                for j in range(coords.shape[0]):
                    writer.writerow([t, coords[j, 0], coords[j, 1], u[j]])


def _snapshot(solver: FactorizedSolver, stepper: DeviceStepper, j: int = 0) -> SolveState:
    lay, pool, N = stepper.lay, stepper.pool, solver.plan.n_gauss
    P, nl = solver.p ** 2, solver._n_leaves
    uw = pool[:2 * N, j].cpu().numpy()
    uc = pool[lay["UC"]:lay["UC"] + nl * P, j].cpu().numpy().reshape(nl, P)
    st = SolveState(u=uw[:N].copy(), w=uw[N:].copy(), tree=solver.tree, p=solver.p, q=solver.q)
    st.leaf_solutions = solver._leaf_view(uc)
    return st


def cn_run(problem: ParabolicProblem, tree, config: TimeStepConfig, p: int, q: int,
           mode: str = "stored") -> CnRun:
    """Crank–Nicolson with one GPU build and device-resident steps (reference timestepping.py:199-240)."""
    builds_before = solver_mod.BUILD_COUNT
    spec = cn_elliptic_spec(problem, config.k)
    solver = solver_mod.build_stage(tree, spec, p, q, mode)
    ctx = RhsContext(problem, tree, p, q, solver.device)
    stepper = DeviceStepper(solver, 1, 1.0 / config.k, 0.5, ctx)
    pts = _leaf_points(solver)
    u0 = np.asarray(problem.initial(pts.reshape(-1, 2)), dtype=float).reshape(solver._n_leaves, -1)
    stepper.set_state(torch.as_tensor(u0, device=solver.device))
    root_ext = solver.plan.node[tree.root].ext
    bpts = solver.plan.coords[root_ext]
    record = config.record_steps()
    states, step_seconds = {}, []
    if 0 in record:
        st0 = SolveState(u=np.full(solver.plan.n_gauss, np.nan), w=np.zeros(solver.plan.n_gauss),
                         tree=tree, p=p, q=q)
        st0.leaf_solutions = solver._leaf_view(u0.copy())
        states[0.0] = st0
    for step in range(1, config.steps + 1):
        t_next = step * config.k
        t0 = time.perf_counter()
        fv = (np.zeros(root_ext.size) if problem.dirichlet is None
              else np.asarray(problem.dirichlet(bpts, t_next), dtype=float))
        stepper.step(torch.as_tensor(fv, device=solver.device).reshape(-1, 1))
        torch.cuda.current_stream().synchronize()
        step_seconds.append(time.perf_counter() - t0)
        if step in record:
            states[t_next] = _snapshot(solver, stepper)
    return CnRun(config=config, times=[s_ * config.k for s_ in sorted(record)], states=states,
                 build_count=solver_mod.BUILD_COUNT - builds_before, build_seconds=solver.build_seconds,
                 step_seconds=step_seconds, solver=solver)


def be_run(solver: FactorizedSolver, u0: torch.Tensor, dirichlet, dt: float, steps: int,
           t0: float = 0.0, sync_every: int = 0) -> DeviceStepper:
    """Backward Euler on a solver built for (1/dt) I - A (config 5): g = u_n / dt.

    u0: (n_leaves, P, nrhs) device tabulations (leaf-row order); dirichlet(t) -> (|root ext|, nrhs)
    device tensor. Returns the stepper (its leaf_tabulations() hold u at t0 + steps*dt).
    """
    nrhs = u0.shape[-1]
    st = DeviceStepper(solver, nrhs, 1.0 / dt, 0.0)
    st.set_state(u0)
    for k in range(1, steps + 1):
        st.step(dirichlet(t0 + k * dt))
        if sync_every and k % sync_every == 0:
            torch.cuda.current_stream().synchronize()
    return st
