"""The five BASELINE.json configurations as concrete, seeded inputs.

Decisions recorded here (the flagged items of SURVEY.md 8d):
  * Gaussian width w means exp(-|x-c|^2 / (2 w^2)) (sigma convention).
  * Seeded draws use ``numpy.random.default_rng(seed)``: centres first
    (``uniform(lo, hi, size=(k, 2))``), then amplitudes (``standard_normal(k)``).
  * config 1 random variant: f = 0 (isolates the body-load path), seed 0.
  * config 4: 2:1-balanced refinement, q = 14 (even q needed by the edge interpolators).
  * config 5: centres U[0,1]^2, seeds 0..15, one RHS per seed.
"""

from __future__ import annotations

import numpy as np

from .model import CoefficientField, ProblemSpec, catalog, manufactured_spec

UNIT = (0.0, 1.0, 0.0, 1.0)


def gaussian_sum(centres, amps, width):
    centres = np.asarray(centres, dtype=float)
    amps = np.asarray(amps, dtype=float)
    s2 = 2.0 * width * width

    def fn(pts):
        pts = np.asarray(pts, dtype=float)
        d2 = ((pts[:, None, :] - centres[None, :, :]) ** 2).sum(axis=2)
        return np.exp(-d2 / s2) @ amps

    fn.centres, fn.amps, fn.width = centres, amps, width
    return fn


def config1_spec() -> ProblemSpec:
    """Poisson, harmonic u = sin(pi x1) sinh(pi x2) (f = u on the boundary, g = 0)."""
    return catalog("manufactured", u="sin(pi*x1)*sinh(pi*x2)")


def config1_random_load(seed: int = 0):
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.1, 0.9, size=(8, 2))
    a = rng.standard_normal(8)
    return gaussian_sum(c, a, 0.05)


def config2_coefficients() -> CoefficientField:
    return CoefficientField(
        c11="1 + sin(2*pi*x1)*cos(2*pi*x2)/2",
        c12="sin(2*pi*(x1 + x2))/10",
        c22="1 + cos(4*pi*x1)*sin(2*pi*x2)/2",
        c1="cos(3*pi*x2)", c2="sin(3*pi*x1)", c=0)


def config2_spec() -> ProblemSpec:
    return manufactured_spec("exp(x1)*sin(5*pi*x2) + x1*x2", config2_coefficients(), name="cfg2")


def config3_spec(kappa: float = 80.0) -> ProblemSpec:
    cf = CoefficientField(1, 0, 1, c=f"-{kappa}**2*(1 - exp(-((x1 - 1/2)**2 + (x2 - 1/2)**2)/(2/100))/2)")
    def f(pts):
        pts = np.asarray(pts, dtype=float)
        return np.cos(kappa * (0.6 * pts[:, 0] + 0.8 * pts[:, 1]))
    return ProblemSpec("cfg3", cf, dirichlet=f, params={"kappa": kappa})


def config4_spec() -> ProblemSpec:
    def g(pts):
        pts = np.asarray(pts, dtype=float)
        return np.exp(-((pts[:, 0] - 0.3) ** 2 + (pts[:, 1] - 0.7) ** 2) / 1e-6) / 1e-6
    return ProblemSpec("cfg4", CoefficientField(1, 0, 1), body_load=g)


def config5_spec(dt: float = 1e-3) -> ProblemSpec:
    """Backward-Euler operator I/dt - Lap in the A-convention: c11 = c22 = 1, c = 1/dt."""
    return ProblemSpec("cfg5", CoefficientField(1, 0, 1, c=1.0 / dt), params={"dt": dt})


def config5_initial(seed: int):
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.0, 1.0, size=(32, 2))
    a = rng.standard_normal(32)
    return gaussian_sum(c, a, 0.02)


def config5_dirichlet(pts, t):
    pts = np.asarray(pts, dtype=float)
    return np.sin(2.0 * np.pi * t) * pts[:, 0] * (1.0 - pts[:, 1])


HEAT_DECAY = 2.0 * np.pi ** 2


def heat_problem():
    """Manufactured heat problem u = exp(-2 pi^2 t) sin(pi x1) sin(pi x2) (reference experiments.py:302-318)."""
    from .timestepping import ParabolicProblem

    def initial(pts):
        pts = np.asarray(pts, dtype=float)
        return np.sin(np.pi * pts[:, 0]) * np.sin(np.pi * pts[:, 1])

    def dirichlet(pts, t):
        return np.zeros(len(pts))

    return ParabolicProblem(operator=CoefficientField(-1.0, 0.0, -1.0), initial=initial,
                            dirichlet=dirichlet, name="heat")


def heat_exact(pts, t):
    pts = np.asarray(pts, dtype=float)
    return np.exp(-HEAT_DECAY * t) * np.sin(np.pi * pts[:, 0]) * np.sin(np.pi * pts[:, 1])
