"""CPU oracle for the HPS build/solve hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module, and only as the checker / CPU baseline; the
product package never does.

It is a numpy/scipy restatement of the reference algorithm (arXiv 1612.02736, package
``specdtn``), function by function:

  leaf_ops        <- pkg/src/specdtn/leaf.py:104-163  (LU + gecon, S/T/F/H)
  assemble        <- pkg/src/specdtn/model.py:153-177 (collocation matrix, row-scaled products)
  merge           <- pkg/src/specdtn/solver.py:108-143 (interface Schur complement)
  wrap            <- pkg/src/specdtn/solver.py:146-188 (2:1 edge interpolation)
  build           <- pkg/src/specdtn/solver.py:357-415 (children-first sweep)
  solve           <- pkg/src/specdtn/solver.py:241-354 (upward / downward passes)
  spectral consts <- pkg/src/specdtn/spectral.py:94-365

Parity is pinned against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``).
The index plan (global Gauss ids, pos arrays, wraps) is an input and is taken from the
caller's ``MergePlan`` (reference or this package's — both pinned by the same goldens).
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import get_lapack_funcs, lu_factor, lu_solve

RCOND_FLOOR = 1e-13


class OracleSingular(RuntimeError):
    pass


# --------------------------------------------------------------------------- spectral

def _cheb(p):
    k = np.arange(p)
    return np.sin(0.5 * np.pi * (2 * k - (p - 1)) / (p - 1))


def _gauss(q):
    return np.polynomial.legendre.leggauss(q)[0]


def _map(t, lo, hi):
    s = 0.5 * (t + 1.0)
    return lo * (1.0 - s) + hi * s


def _weights(x):
    if x.size == 1:
        return np.ones(1)
    d = (x[:, None] - x[None, :]) * (4.0 / (x.max() - x.min()))
    np.fill_diagonal(d, 1.0)
    w = 1.0 / d.prod(axis=1)
    return w / np.abs(w).max()


def _interp(src, dst):
    w = _weights(src)
    d = dst[:, None] - src[None, :]
    hr, hc = np.nonzero(d == 0.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = w[None, :] / d
        m = r / r.sum(axis=1, keepdims=True)
    if hr.size:
        m[hr] = 0.0
        m[hr, hc] = 1.0
    return m


def _diff(x):
    w = _weights(x)
    d = x[:, None] - x[None, :]
    np.fill_diagonal(d, 1.0)
    m = (w[None, :] / w[:, None]) / d
    np.fill_diagonal(m, 0.0)
    np.fill_diagonal(m, -m.sum(axis=1))
    return m


_GEO = {}


def leaf_geometry(p, q, w, h):
    """Dense shape constants (D1, D2, products, lift, flux, index sets) per leaf shape."""
    key = (p, q, w, h)
    if key in _GEO:
        return _GEO[key]
    cx, cy = _map(_cheb(p), 0.0, w), _map(_cheb(p), 0.0, h)
    gx, gy = _map(_gauss(q), 0.0, w), _map(_gauss(q), 0.0, h)
    d1 = np.kron(np.eye(p), _diff(cx))
    d2 = np.kron(_diff(cy), np.eye(p))
    idx = np.arange(p * p)
    a, b = idx % p, idx // p
    i_s, i_e, i_n, i_w = idx[b == 0], idx[a == p - 1], idx[b == p - 1], idx[a == 0]
    i_ce = np.concatenate([i_s[:-1], i_e[:-1], i_n[1:], i_w[1:]])
    i_ci = idx[(a > 0) & (a < p - 1) & (b > 0) & (b < p - 1)]
    mx, my = _interp(gx, cx), _interp(gy, cy)
    n = p - 1
    lift = np.zeros((4 * n, 4 * q))
    S, E, N, W = (slice(k * q, (k + 1) * q) for k in range(4))
    lift[:n, S] = mx[:n]
    lift[n:2 * n, E] = my[:n]
    lift[2 * n:3 * n, N] = mx[1:]
    lift[3 * n:, W] = my[1:]
    lift[0, S], lift[0, W] = 0.5 * mx[0], 0.5 * my[0]
    lift[n, E], lift[n, S] = 0.5 * my[0], 0.5 * mx[p - 1]
    lift[3 * n - 1, N], lift[3 * n - 1, E] = 0.5 * mx[p - 1], 0.5 * my[p - 1]
    lift[4 * n - 1, W], lift[4 * n - 1, N] = 0.5 * my[p - 1], 0.5 * mx[0]
    lx, ly = _interp(cx, gx), _interp(cy, gy)
    flux = np.vstack([lx @ d2[i_s], ly @ d1[i_e], lx @ d2[i_n], ly @ d1[i_w]])
    pts0 = np.column_stack([np.tile(cx, p), np.repeat(cy, p)])
    geo = dict(p=p, q=q, d1=d1, d2=d2, prods=(d1 @ d1, d1 @ d2, d2 @ d2), lift=lift, flux=flux,
               i_ce=i_ce, i_ci=i_ci, i_s=i_s, i_e=i_e, i_n=i_n, i_w=i_w, pts0=pts0,
               gx=gx, gy=gy)
    _GEO[key] = geo
    return geo


def edge_interpolators(q):
    g = _gauss(q)
    lo, hi = 0.5 * (g - 1.0), 0.5 * (g + 1.0)
    up = np.vstack([_interp(g, lo), _interp(g, hi)])
    h = q // 2
    down = np.zeros((q, 2 * q))
    down[:h, :q] = _interp(lo, g[:h])
    down[h:, q:] = _interp(hi, g[h:])
    return up, down


# --------------------------------------------------------------------------- leaf stage

def leaf_points(bounds, p, q):
    geo = leaf_geometry(p, q, bounds.x1hi - bounds.x1lo, bounds.x2hi - bounds.x2lo)
    return geo["pts0"] + np.array([bounds.x1lo, bounds.x2lo])


def assemble(coef_fns, pts, geo):
    """Collocation matrix with coefficient-scaled rows (reference model.py:153-177)."""
    d11, d12, d22 = geo["prods"]
    c = [np.asarray(fn(pts), dtype=float) * np.ones(len(pts)) for fn in coef_fns]
    a = -(c[0][:, None] * d11)
    a -= 2.0 * c[1][:, None] * d12
    a -= c[2][:, None] * d22
    a += c[3][:, None] * geo["d1"]
    a += c[4][:, None] * geo["d2"]
    a[np.diag_indices_from(a)] += c[5]
    if not np.all(np.isfinite(a)):
        raise ValueError("non-finite coefficient evaluation")
    return a


def _gecon_factor(mat):
    """LU with partial pivoting + LAPACK 1-norm rcond estimate."""
    anorm = np.linalg.norm(mat, 1)
    lu, piv = lu_factor(mat)
    rcond, info = get_lapack_funcs(("gecon",), (lu,))[0](lu, anorm)
    return (lu, piv), rcond, info


def leaf_ops(bounds, coef_fns, p, q):
    """S (P x 4q), T (4q x 4q), F (P x m), H (4q x m), rcond — reference leaf.py:138-163."""
    geo = leaf_geometry(p, q, bounds.x1hi - bounds.x1lo, bounds.x2hi - bounds.x2lo)
    pts = geo["pts0"] + np.array([bounds.x1lo, bounds.x2lo])
    a = assemble(coef_fns, pts, geo)
    ci, ce = geo["i_ci"], geo["i_ce"]
    lu_piv, rcond, info = _gecon_factor(a[np.ix_(ci, ci)])
    if info != 0 or not np.isfinite(rcond) or rcond < RCOND_FLOOR:
        raise OracleSingular(f"leaf interior block singular (rcond {rcond:.3e})")
    P = p * p
    s = np.empty((P, 4 * q))
    s[ce] = geo["lift"]
    s[ci] = lu_solve(lu_piv, -(a[np.ix_(ci, ce)] @ geo["lift"]))
    t = geo["flux"] @ s
    f = np.zeros((P, ci.size))
    f[ci] = lu_solve(lu_piv, np.eye(ci.size))
    h = geo["flux"] @ f
    return dict(S=s, T=t, F=f, H=h, rcond=rcond)


# --------------------------------------------------------------------------- merge stage

def merge(ta, tb, e):
    """Interface elimination (reference solver.py:108-143). Returns dict with X(dense), S, Tei, T."""
    p1a, p3a, p2b, p3b = e.pos1_a, e.pos3_a, e.pos2_b, e.pos3_b
    delta = ta[np.ix_(p3a, p3a)] - tb[np.ix_(p3b, p3b)]
    lu_piv, rcond, info = _gecon_factor(delta)
    if info != 0 or not np.isfinite(rcond) or rcond < RCOND_FLOOR:
        raise OracleSingular(f"interface singular (rcond {rcond:.3e})")
    s = lu_solve(lu_piv, np.hstack([-ta[np.ix_(p3a, p1a)], tb[np.ix_(p3b, p2b)]]))
    tei = np.vstack([ta[np.ix_(p1a, p3a)], tb[np.ix_(p2b, p3b)]])
    n1 = p1a.size
    tnew = tei @ s
    tnew[:n1, :n1] += ta[np.ix_(p1a, p1a)]
    tnew[n1:, n1:] += tb[np.ix_(p2b, p2b)]
    return dict(lu_piv=lu_piv, S=s, Tei=tei, T=tnew, rcond=rcond)


def wrap_matrices(wrap, q):
    """Dense block-diagonal P_up / P_down for a wrap plan (reference solver.py:157-174)."""
    up_ref, down_ref = edge_interpolators(q)
    ups, downs = [], []
    for blk in wrap.blocks:
        if blk[0] == "identity":
            ups.append(np.eye(blk[1]))
            downs.append(np.eye(blk[1]))
        else:
            ups.append(up_ref)
            downs.append(down_ref)
    rows_u = sum(u.shape[0] for u in ups)
    cols_u = sum(u.shape[1] for u in ups)
    pu = np.zeros((rows_u, cols_u))
    pd = np.zeros((cols_u, rows_u))
    r = c = 0
    for u, d in zip(ups, downs):
        pu[r:r + u.shape[0], c:c + u.shape[1]] = u
        pd[c:c + d.shape[0], r:r + d.shape[1]] = d
        r += u.shape[0]
        c += u.shape[1]
    return pu, pd


def coef_functions(spec):
    cf = spec.coefficients
    return (cf.c11, cf.c12, cf.c22, cf.c1, cf.c2, cf.c)


def build(tree, spec, p, q, plan):
    """Children-first sweep (reference solver.py:357-415). Returns an ops dict."""
    fns = coef_functions(spec)
    leaves, parents, tmap = {}, {}, {}
    for nid in range(len(tree.nodes) - 1, -1, -1):
        node = tree.nodes[nid]
        if node.is_leaf:
            ops = leaf_ops(node.bounds, fns, p, q)
            tmap[nid] = ops.pop("T")
            leaves[nid] = ops
            continue
        ca, cb = node.children
        e = plan.node[nid]
        ops = merge(tmap.pop(ca), tmap.pop(cb), e)
        if e.wrap is not None:
            pu, pd = wrap_matrices(e.wrap, q)
            perm = e.wrap.perm
            ops["T"] = pd @ ops["T"][np.ix_(perm, perm)] @ pu
            ops["S"] = ops["S"][:, perm] @ pu
            ops["wrap"] = (pu, pd, perm, e.wrap.fine)
        tmap[nid] = ops.pop("T")
        parents[nid] = ops
    return dict(tree=tree, plan=plan, p=p, q=q, leaves=leaves, parents=parents, spec=spec)


# --------------------------------------------------------------------------- solve stage

def solve(ops, f=None, g=None):
    """Upward then downward pass (reference solver.py:241-354).

    f: array over the root exterior (plan order) or callable or None (-> spec.dirichlet).
    g: dict leaf id -> (m,) interior tabulation, callable, or None (-> spec.body_load).
    """
    tree, plan, p, q, spec = ops["tree"], ops["plan"], ops["p"], ops["q"], ops["spec"]
    n = plan.n_gauss
    u, w = np.zeros(n), np.zeros(n)
    h, gtab = {}, {}
    if g is None:
        g = spec.body_load
    for nid in range(len(tree.nodes) - 1, -1, -1):
        node = tree.nodes[nid]
        e = plan.node[nid]
        if node.is_leaf:
            geo = leaf_geometry(p, q, node.bounds.x1hi - node.bounds.x1lo, node.bounds.x2hi - node.bounds.x2lo)
            m = geo["i_ci"].size
            if g is None:
                gci = np.zeros(m)
            elif callable(g):
                gci = np.asarray(g(leaf_points(node.bounds, p, q)[geo["i_ci"]]), dtype=float)
            else:
                gci = np.asarray(g[nid], dtype=float)
            gtab[nid] = gci
            h[nid] = ops["leaves"][nid]["H"] @ gci
            continue
        ca, cb = node.children
        ha, hb = h.pop(ca), h.pop(cb)
        po = ops["parents"][nid]
        w3 = lu_solve(po["lu_piv"], hb[e.pos3_b] - ha[e.pos3_a])
        hge = np.concatenate([ha[e.pos1_a], hb[e.pos2_b]]) + po["Tei"] @ w3
        if "wrap" in po:
            pu, pd, perm, _ = po["wrap"]
            hge = pd @ hge[perm]
        w[e.j3] = w3
        h[nid] = hge
    h_root = h[tree.root]
    root_ext = plan.node[tree.root].ext
    if f is None:
        f = spec.dirichlet
    if f is None:
        fv = np.zeros(root_ext.size)
    elif callable(f):
        fv = np.asarray(f(plan.coords[root_ext]), dtype=float)
    else:
        fv = np.asarray(f, dtype=float)
    u[root_ext] = fv
    sol = {}
    for nid in range(len(tree.nodes)):
        node = tree.nodes[nid]
        e = plan.node[nid]
        if node.is_leaf:
            lo = ops["leaves"][nid]
            sol[nid] = lo["S"] @ u[e.ext] + lo["F"] @ gtab[nid]
            continue
        po = ops["parents"][nid]
        if "wrap" in po:
            pu, _, _, fine = po["wrap"]
            uext = u[e.ext]
            u[fine] = pu @ uext
        else:
            uext = u[e.ext_mergeorder]
        u[e.j3] = po["S"] @ uext + w[e.j3]
    return dict(u=u, w=w, leaf_solutions=sol, g_tab=gtab, h_root=h_root)


def be_loads(leaf_solutions, tree, p, q, dt):
    """Backward-Euler body load g^{k+1} = u_c^k[i_ci] / dt (config-5 harness, not reference code;
    the nearest reference routine is the CN driver timestepping.py:199-240)."""
    out = {}
    for nid, vals in leaf_solutions.items():
        b = tree.nodes[nid].bounds
        geo = leaf_geometry(p, q, b.x1hi - b.x1lo, b.x2hi - b.x2lo)
        out[nid] = vals[geo["i_ci"]] / dt
    return out
