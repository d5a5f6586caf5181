"""Error metric and reference solutions (reference pkg/src/specdtn/reference.py:30-94), host side.

linf_error measures the max deviation over all leaf-boundary Chebyshev nodes, exactly as the
reference does, on SolveState objects of either package.
"""

from __future__ import annotations

import numpy as np

from .spectral import lagrange_matrix, shape_constants


class ReferenceSolution:
    """Evaluate a reference field at arbitrary points (reference.py:30-66)."""

    def __init__(self, evaluate, meta=None):
        self._evaluate = evaluate
        self.meta = meta or {}

    def evaluate(self, pts) -> np.ndarray:
        return self._evaluate(np.asarray(pts, dtype=float))

    @staticmethod
    def analytic(u_exact, meta=None) -> "ReferenceSolution":
        return ReferenceSolution(lambda pts: np.asarray(u_exact(pts), dtype=float),
                                 meta={"kind": "analytic", **(meta or {})})

    @staticmethod
    def from_state(state, meta=None) -> "ReferenceSolution":
        """Per-leaf tensor barycentric interpolation of a solved state."""
        tree, p, q = state.tree, state.p, state.q

        def evaluate(pts):
            out = np.empty(len(pts))
            by_leaf: dict = {}
            for j, pt in enumerate(pts):
                by_leaf.setdefault(tree.descend(pt).id, []).append(j)
            for nid, rows in by_leaf.items():
                rows = np.asarray(rows)
                b = tree.nodes[nid].bounds
                sc = shape_constants(p, q, b.x1hi - b.x1lo, b.x2hi - b.x2lo)
                wx = lagrange_matrix(sc.cx + b.x1lo, pts[rows, 0])
                wy = lagrange_matrix(sc.cy + b.x2lo, pts[rows, 1])
                vals = np.asarray(state.leaf_solutions[nid]).reshape(p, p)
                out[rows] = np.einsum("mi,mj,ji->m", wx, wy, vals)
            return out

        return ReferenceSolution(evaluate, meta={"kind": "self", **(meta or {})})


def state_boundary_values(state):
    """(points, values) at every leaf-boundary Chebyshev node (reference.py:79-88)."""
    tree, p, q = state.tree, state.p, state.q
    pts, vals = [], []
    for node in (n for n in tree.nodes if n.is_leaf):
        b = node.bounds
        sc = shape_constants(p, q, b.x1hi - b.x1lo, b.x2hi - b.x2lo)
        pts.append(sc.cheb2d(b.x1lo, b.x2lo)[sc.i_ce])
        vals.append(np.asarray(state.leaf_solutions[node.id])[sc.i_ce])
    return np.concatenate(pts), np.concatenate(vals)


def linf_error(state, reference: ReferenceSolution) -> float:
    """Max absolute deviation on all leaf-boundary Chebyshev nodes (reference.py:91-94)."""
    pts, vals = state_boundary_values(state)
    return float(np.abs(vals - reference.evaluate(pts)).max())
