"""Host-side FP64 spectral constants for the leaf stage (computed once per leaf shape).

Clean-room restatement of the collocation primitives the reference builds in
``pkg/src/specdtn/spectral.py``; every array produced here is uploaded to the device
once per distinct leaf shape and then shared by all leaves of that shape.

Conventions (identical to the reference, which the GPU results must match):
  * tensor grids are x1-fastest: node k = i1 + p*i2          (spectral.py:16-17)
  * Gauss edge data runs S, E, N, W, each ascending           (spectral.py:18-19)
  * exterior Chebyshev list gives each corner to one side:
    SW->S, SE->E, NE->N, NW->W                                (spectral.py:20-21, 240-252)
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

SOUTH, EAST, NORTH, WEST = 0, 1, 2, 3


def cheb_ref(p: int) -> np.ndarray:
    """Chebyshev extreme points on [-1, 1] in sine form (reference spectral.py:94-103)."""
    if p < 2:
        raise ValueError(f"Chebyshev grid needs p >= 2, got {p}")
    j = np.arange(p, dtype=float)
    return np.sin(np.pi * (2.0 * j - (p - 1)) / (2.0 * (p - 1)))


def gauss_ref(q: int) -> np.ndarray:
    """Gauss-Legendre points on (-1, 1) ascending (reference spectral.py:106-111)."""
    if q < 1:
        raise ValueError(f"Gauss grid needs q >= 1, got {q}")
    return np.polynomial.legendre.leggauss(q)[0]


def to_interval(t: np.ndarray, lo: float, hi: float) -> np.ndarray:
    """Affine map [-1,1] -> [lo,hi] with exact endpoints (reference spectral.py:69-76)."""
    s = 0.5 * (np.asarray(t, dtype=float) + 1.0)
    return lo * (1.0 - s) + hi * s


def bary_weights(x: np.ndarray) -> np.ndarray:
    """Scaled barycentric weights, max |w| = 1 (reference spectral.py:126-142)."""
    x = np.asarray(x, dtype=float)
    if x.size == 1:
        return np.ones(1)
    span = 4.0 / (x.max() - x.min())
    diffs = (x[:, None] - x[None, :]) * span
    diffs[np.arange(x.size), np.arange(x.size)] = 1.0
    if (diffs == 0.0).any():
        raise ValueError("interpolation nodes must be pairwise distinct")
    w = 1.0 / np.prod(diffs, axis=1)
    return w / np.max(np.abs(w))


def lagrange_matrix(src: np.ndarray, dst: np.ndarray) -> np.ndarray:
    """Barycentric interpolation matrix src -> dst (reference spectral.py:145-164)."""
    src = np.asarray(src, dtype=float)
    dst = np.asarray(dst, dtype=float)
    w = bary_weights(src)
    gap = dst[:, None] - src[None, :]
    exact_r, exact_c = np.nonzero(gap == 0.0)
    with np.errstate(divide="ignore", invalid="ignore"):
        frac = w[None, :] / gap
        out = frac / frac.sum(axis=1, keepdims=True)
    if exact_r.size:
        out[exact_r] = 0.0
        out[exact_r, exact_c] = 1.0
    return out


def diff_1d(x: np.ndarray) -> np.ndarray:
    """Collocation derivative on nodes x, diagonal = -row sum (reference spectral.py:167-181)."""
    x = np.asarray(x, dtype=float)
    w = bary_weights(x)
    gap = x[:, None] - x[None, :]
    n = x.size
    gap[np.arange(n), np.arange(n)] = 1.0
    d = (w[None, :] / w[:, None]) / gap
    d[np.arange(n), np.arange(n)] = 0.0
    d[np.arange(n), np.arange(n)] = -d.sum(axis=1)
    return d


def grid_index_sets(p: int):
    """(i_ce, i_ci, i_s, i_e, i_n, i_w) of the p x p grid (reference spectral.py:240-252)."""
    k = np.arange(p * p)
    i1, i2 = k % p, k // p
    south, east = k[i2 == 0], k[i1 == p - 1]
    north, west = k[i2 == p - 1], k[i1 == 0]
    i_ce = np.concatenate([south[:-1], east[:-1], north[1:], west[1:]])
    inner = (i1 > 0) & (i1 < p - 1) & (i2 > 0) & (i2 < p - 1)
    return i_ce, k[inner], south, east, north, west


def lift_matrix(p: int, q: int, width: float, height: float) -> np.ndarray:
    """Gauss edge data (4q) -> exterior Chebyshev data (4(p-1)) with corner averaging.

    Restates reference spectral.py:282-319: each side interpolates from its own q Gauss
    nodes; every corner row is the mean of the two one-sided extrapolations.
    """
    if p < 3 or q < 2:
        raise ValueError("boundary lift needs p >= 3 and q >= 2")
    ix = lagrange_matrix(to_interval(gauss_ref(q), 0.0, width), to_interval(cheb_ref(p), 0.0, width))
    iy = lagrange_matrix(to_interval(gauss_ref(q), 0.0, height), to_interval(cheb_ref(p), 0.0, height))
    n = p - 1
    out = np.zeros((4 * n, 4 * q))
    cols = [slice(s * q, (s + 1) * q) for s in range(4)]
    # side blocks (rows follow the i_ce walk)
    out[0:n, cols[SOUTH]] = ix[:n]
    out[n:2 * n, cols[EAST]] = iy[:n]
    out[2 * n:3 * n, cols[NORTH]] = ix[1:]
    out[3 * n:4 * n, cols[WEST]] = iy[1:]
    # corners: SW (row 0), SE (row n), NE (row 3n-1), NW (row 4n-1)
    corner_rows = (0, n, 3 * n - 1, 4 * n - 1)
    corner_terms = (((SOUTH, ix[0]), (WEST, iy[0])),
                    ((EAST, iy[0]), (SOUTH, ix[p - 1])),
                    ((NORTH, ix[p - 1]), (EAST, iy[p - 1])),
                    ((WEST, iy[p - 1]), (NORTH, ix[0])))
    for row, terms in zip(corner_rows, corner_terms):
        for side, vals in terms:
            out[row, cols[side]] = 0.5 * vals
    return out


def edge_interpolators(q: int):
    """(P_up 2q x q, P_down q x 2q) between a coarse edge and its halves.

    Restates reference spectral.py:344-365 (needs even q).
    """
    if q < 2 or q % 2:
        raise ValueError(
            f"edge interpolators need an even q >= 2 (two q/2 blocks); got q={q}")
    g = gauss_ref(q)
    lo_half, hi_half = 0.5 * (g - 1.0), 0.5 * (g + 1.0)
    up = np.vstack([lagrange_matrix(g, lo_half), lagrange_matrix(g, hi_half)])
    h = q // 2
    down = np.zeros((q, 2 * q))
    down[:h, :q] = lagrange_matrix(lo_half, g[:h])
    down[h:, q:] = lagrange_matrix(hi_half, g[h:])
    return up, down


@dataclass(frozen=True)
class ShapeConstants:
    """Everything the device leaf stage needs for one (p, q, width, height) leaf shape.

    dx, dy, dxx, dyy : 1D operators (p x p) — the kernel rebuilds rows of
                       D1 = kron(I, dx), D2 = kron(dy, I) and their products on the fly.
    lift  : L (c x b)        flux : D_ge,c (b x P)
    dfi   : flux[:, i_ci] (b x m)   t0 : flux[:, i_ce] @ L (b x b)
    """

    p: int
    q: int
    width: float
    height: float
    cx: np.ndarray
    cy: np.ndarray
    gx: np.ndarray
    gy: np.ndarray
    dx: np.ndarray
    dy: np.ndarray
    dxx: np.ndarray
    dyy: np.ndarray
    i_ce: np.ndarray
    i_ci: np.ndarray
    i_s: np.ndarray
    i_e: np.ndarray
    i_n: np.ndarray
    i_w: np.ndarray
    lift: np.ndarray
    flux: np.ndarray
    dfi: np.ndarray
    t0: np.ndarray

    @property
    def m(self) -> int:
        return (self.p - 2) ** 2

    @property
    def b(self) -> int:
        return 4 * self.q

    @property
    def c(self) -> int:
        return 4 * (self.p - 1)

    def cheb2d(self, x1lo: float = 0.0, x2lo: float = 0.0) -> np.ndarray:
        """(P, 2) x1-fastest grid of the leaf anchored at (x1lo, x2lo)."""
        pts = np.empty((self.p * self.p, 2))
        pts[:, 0] = np.tile(self.cx + x1lo, self.p)
        pts[:, 1] = np.repeat(self.cy + x2lo, self.p)
        return pts


@lru_cache(maxsize=64)
def shape_constants(p: int, q: int, width: float, height: float) -> ShapeConstants:
    """Per-shape constants; mirrors reference leaf.py:66-80 (cached per p, q, w, h)."""
    if p < q + 1:
        raise ValueError(f"leaf order must satisfy p >= q+1, got p={p}, q={q}")
    if p < 3:
        raise ValueError(f"leaf stencil needs p >= 3, got {p}")
    if q < 2:
        raise ValueError(f"leaf stencil needs q >= 2, got {q}")
    cx = to_interval(cheb_ref(p), 0.0, width)
    cy = to_interval(cheb_ref(p), 0.0, height)
    gx = to_interval(gauss_ref(q), 0.0, width)
    gy = to_interval(gauss_ref(q), 0.0, height)
    dx, dy = diff_1d(cx), diff_1d(cy)
    i_ce, i_ci, i_s, i_e, i_n, i_w = grid_index_sets(p)
    lift = lift_matrix(p, q, width, height)
    # flux extractor: d/dx2 on S/N, d/dx1 on E/W, interpolated to Gauss nodes
    # (reference spectral.py:322-341), built from the kron structure of D1/D2.
    eye = np.eye(p)
    d1 = np.kron(eye, dx)
    d2 = np.kron(dy, eye)
    lx = lagrange_matrix(cx, gx)
    ly = lagrange_matrix(cy, gy)
    flux = np.vstack([lx @ d2[i_s], ly @ d1[i_e], lx @ d2[i_n], ly @ d1[i_w]])
    dfi = np.ascontiguousarray(flux[:, i_ci])
    t0 = flux[:, i_ce] @ lift
    return ShapeConstants(p, q, width, height, cx, cy, gx, gy, dx, dy, dx @ dx, dy @ dy,
                          i_ce, i_ci, i_s, i_e, i_n, i_w, lift, flux, dfi, t0)
