"""PDE description: coefficient fields, problem specs, catalog (host side, inputs).

Mirror of the reference's ``pkg/src/specdtn/model.py`` interface so a user of the
reference finds the same objects here:

    A u = -c11 u_x1x1 - 2 c12 u_x1x2 - c22 u_x2x2 + c1 u_x1 + c2 u_x2 + c u

``CoefficientField`` keeps the sympy expressions (``.exprs``) so the device path can
evaluate the coefficients on the GPU (``coeffs.py``); raw callables are evaluated on the
host and uploaded (documented fallback for inputs, not part of the timed hot path).
Reference objects (``specdtn.model.CoefficientField`` / ``ProblemSpec``) are accepted
by ``build_stage`` as well — only the attributes used here are read.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import sympy as sp

X1, X2 = sp.symbols("x1 x2", real=True)
COEF_NAMES = ("c11", "c12", "c22", "c1", "c2", "c")


def field_function(value):
    """constant / sympy expr / string -> (vectorised numpy callable, expr); callables pass through.

    Follows reference model.py:40-55.
    """
    if callable(value) and not isinstance(value, sp.Expr):
        return value, None
    expr = sp.sympify(value, locals={"x1": X1, "x2": X2})
    lam = sp.lambdify((X1, X2), expr, "numpy")

    def fn(pts, _lam=lam):
        pts = np.asarray(pts, dtype=float)
        out = np.asarray(_lam(pts[:, 0], pts[:, 1]), dtype=float)
        if out.shape != (pts.shape[0],):
            out = np.broadcast_to(out, (pts.shape[0],)).copy()
        return out

    return fn, expr


class CoefficientField:
    """Six vectorised coefficient functions (reference model.py:58-101)."""

    __slots__ = COEF_NAMES + ("exprs",)
    _NAMES = COEF_NAMES

    def __init__(self, c11=1, c12=0, c22=1, c1=0, c2=0, c=0):
        self.exprs = {}
        for name, value in zip(COEF_NAMES, (c11, c12, c22, c1, c2, c)):
            fn, expr = field_function(value)
            setattr(self, name, fn)
            if expr is not None:
                self.exprs[name] = expr

    def symbolic(self) -> dict:
        missing = [n for n in COEF_NAMES if n not in self.exprs]
        if missing:
            raise ValueError(f"coefficients {missing} have no symbolic form")
        return dict(self.exprs)

    def check_ellipticity(self, pts, label=""):
        import warnings
        pts = np.asarray(pts, dtype=float)
        a, b, d = self.c11(pts), self.c12(pts), self.c22(pts)
        bad = (a <= 0) | (d <= 0) | (a * d - b * b <= 0)
        if np.any(bad):
            k = int(np.argmax(bad))
            warnings.warn(
                f"second-order coefficients are not positive definite at sampled point "
                f"{tuple(pts[k])}{' (' + label + ')' if label else ''}", stacklevel=2)


@dataclass
class ProblemSpec:
    """Boundary value problem (reference model.py:108-131)."""

    name: str
    coefficients: CoefficientField
    body_load: object | None = None
    dirichlet: object | None = None
    params: dict = field(default_factory=dict)
    u_exact: object | None = None
    initial: object | None = None
    catalog_key: tuple | None = None

    def load(self, pts):
        return self.body_load(pts) if self.body_load is not None else np.zeros(len(pts))

    def boundary(self, pts):
        return self.dirichlet(pts) if self.dirichlet is not None else np.zeros(len(pts))


def _gauss_expr(alpha, center):
    return sp.exp(-alpha * ((X1 - center[0]) ** 2 + (X2 - center[1]) ** 2))


def _gauss_fn(alpha, center):
    cx, cy = center
    return lambda pts: np.exp(-alpha * ((np.asarray(pts)[:, 0] - cx) ** 2 + (np.asarray(pts)[:, 1] - cy) ** 2))


def manufactured_spec(u, coefficients: CoefficientField, name="manufactured") -> ProblemSpec:
    """g = A u symbolically, f = u on the boundary (reference model.py:303-321 generalised
    to any symbolic coefficient field, as config 2 needs)."""
    ue = sp.sympify(u, locals={"x1": X1, "x2": X2})
    ce = coefficients.symbolic()
    g = (-ce["c11"] * sp.diff(ue, X1, 2) - 2 * ce["c12"] * sp.diff(ue, X1, X2)
         - ce["c22"] * sp.diff(ue, X2, 2) + ce["c1"] * sp.diff(ue, X1)
         + ce["c2"] * sp.diff(ue, X2) + ce["c"] * ue)
    gfn, _ = field_function(sp.simplify(g))
    ufn, _ = field_function(ue)
    return ProblemSpec(name, coefficients, body_load=gfn, dirichlet=ufn, u_exact=ufn,
                       params={"u": str(u)})


def catalog(name: str, **params) -> ProblemSpec:
    """Catalog entries of reference model.py:230-360."""
    if name == "laplace":
        spec = ProblemSpec("laplace", CoefficientField(1, 0, 1), params=dict(params))
    elif name == "helmholtz":
        if "kappa" not in params:
            raise ValueError("catalog entry 'helmholtz' is missing parameter 'kappa'")
        spec = ProblemSpec("helmholtz", CoefficientField(1, 0, 1, c=-(params["kappa"] ** 2)),
                           params=dict(params))
    elif name == "varcoef_helmholtz":
        p = {"kappa": 40.0, "alpha": 300.0, "xhat": (0.25, 0.75), "alpha2": 200.0,
             "alpha3": 200.0, "xhat2": (7 / 20, 6 / 10), "xhat3": (6 / 10, 9 / 20)}
        p.update(params)
        scatter = (sp.Rational(1, 2) * _gauss_expr(p["alpha2"], p["xhat2"])
                   + sp.Rational(1, 2) * _gauss_expr(p["alpha3"], p["xhat3"]))
        cf = CoefficientField(1, 0, 1, c=-p["kappa"] ** 2 * (1 - scatter))
        spec = ProblemSpec("varcoef_helmholtz", cf, body_load=_gauss_fn(p["alpha"], p["xhat"]), params=p)
    elif name == "concentrated_helmholtz":
        p = {"kappa": 20.0, "alpha": 3000.0, "xhat": (0.5, 0.5)}
        p.update(params)
        spec = ProblemSpec("concentrated_helmholtz", CoefficientField(1, 0, 1, c=-p["kappa"] ** 2),
                           body_load=_gauss_fn(p["alpha"], p["xhat"]), params=p)
    elif name == "indicator_poisson":
        p = {"support": (0.25, 0.5, 0.25, 0.5)}
        p.update(params)
        a, b, c, d = p["support"]

        def g(pts):
            pts = np.asarray(pts, dtype=float)
            return ((pts[:, 0] >= a) & (pts[:, 0] <= b) & (pts[:, 1] >= c) & (pts[:, 1] <= d)).astype(float)

        spec = ProblemSpec("indicator_poisson", CoefficientField(1, 0, 1), body_load=g, params=p)
    elif name == "convection_diffusion":
        p = {"epsilon": 1 / 200, "alpha": 50.0, "xhat": (0.25, 0.25)}
        p.update(params)
        eps = p["epsilon"]
        spec = ProblemSpec("convection_diffusion", CoefficientField(-eps, 0, -eps, c1=-1.0),
                           initial=_gauss_fn(p["alpha"], p["xhat"]), params=p)
    elif name == "manufactured":
        p = {"operator": "laplace"}
        p.update(params)
        if "u" not in p:
            raise ValueError("manufactured entry needs a solution expression 'u'")
        base = catalog(p["operator"], **{k: v for k, v in p.items() if k not in ("u", "operator")})
        spec = manufactured_spec(p["u"], base.coefficients)
        spec.params = p
    else:
        raise KeyError(f"unknown catalog entry {name!r}")
    spec.catalog_key = (name, {k: v for k, v in spec.params.items() if not callable(v)})
    return spec
