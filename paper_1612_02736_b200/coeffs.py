"""On-device evaluation of the six PDE coefficients at the leaves' Chebyshev points.

Sympy expressions (``CoefficientField.exprs``, reference model.py:73-78) are lambdified to
torch and evaluated on CUDA tensors, so the [6, L, P] coefficient table the leaf-assembly
kernel reads is produced on the GPU. Raw callables without a symbolic form (allowed by
the reference, model.py:40-43) are evaluated on the host and uploaded — documented
input-preparation fallback, outside the timed hot path.
"""

from __future__ import annotations

import numpy as np
import sympy as sp
import torch

from .model import COEF_NAMES, X1, X2

_LAMBDA_CACHE: dict = {}


def _torch_fn(expr):
    key = sp.srepr(expr)
    fn = _LAMBDA_CACHE.get(key)
    if fn is None:
        syms = sorted(expr.free_symbols, key=lambda s: s.name)
        subs = {s: (X1 if s.name == "x1" else X2) for s in syms if s.name in ("x1", "x2")}
        expr = expr.xreplace(subs)
        fn = sp.lambdify((X1, X2), expr, modules="torch")
        _LAMBDA_CACHE[key] = fn
    return fn


def evaluate(coefficients, pts: torch.Tensor) -> torch.Tensor:
    """pts: (..., 2) float64 CUDA tensor -> (6, ...) coefficient table on the same device."""
    out = torch.empty((6,) + tuple(pts.shape[:-1]), dtype=torch.float64, device=pts.device)
    x1, x2 = pts[..., 0], pts[..., 1]
    exprs = getattr(coefficients, "exprs", {}) or {}
    for k, name in enumerate(COEF_NAMES):
        expr = exprs.get(name)
        if expr is not None:
            val = _torch_fn(expr)(x1, x2)
            if isinstance(val, torch.Tensor):
                out[k] = val.to(torch.float64).expand_as(x1)
            else:
                out[k].fill_(float(val))
        else:
            host = pts.detach().cpu().numpy().reshape(-1, 2)
            vals = np.asarray(getattr(coefficients, name)(host), dtype=np.float64)
            vals = np.broadcast_to(vals, (host.shape[0],))
            out[k] = torch.from_numpy(np.ascontiguousarray(vals)).to(pts.device).reshape(x1.shape)
    return out
