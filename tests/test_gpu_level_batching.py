"""Padded level batching of small parent steps (FactorizedSolver._merge_levels): on a refined
mesh every wrapped parent is its own shape group, so one tree level used to cost several
launches. Batched, the solve must give the same values (padding meets a zero pool row and a
scratch output row) and the config-4 program must need far fewer launches."""
import numpy as np
import pytest
import torch

from paper_1612_02736_b200 import build_balanced_refined_tree, build_stage, catalog, problems
from paper_1612_02736_b200.solver import downward_pass, upward_pass

pytestmark = pytest.mark.gpu


def _pair(tree, spec, p, q):
    merged = build_stage(tree, spec, p, q)
    plain = build_stage(tree, spec, p, q)
    plain.MERGE_BYTES = 0  # instance override: no level batching
    return merged, plain


@pytest.mark.parametrize("nrhs", [1, 4])
def test_config4_batched_levels_match_unbatched(nrhs):
    tree = build_balanced_refined_tree(8, (0.3, 0.7), 8)
    merged, plain = _pair(tree, problems.config4_spec(), 16, 14)
    nm = len(merged._program(nrhs)["up"]) + len(merged._program(nrhs)["down"])
    npl = len(plain._program(nrhs)["up"]) + len(plain._program(nrhs)["down"])
    assert nm < 0.5 * npl, (nm, npl)
    root_ext = merged.plan.node[tree.root].ext
    rng = np.random.default_rng(3)
    f = torch.as_tensor(rng.standard_normal((root_ext.size, nrhs)), device="cuda")
    g = torch.as_tensor(rng.standard_normal((merged._n_leaves * 196, nrhs)), device="cuda")
    a = {k: v.clone() for k, v in merged.solve_device(f, g).items()}
    b = plain.solve_device(f, g)
    scale = b["uc"].abs().max().item()
    for k in ("u", "w", "uc"):
        assert (a[k] - b[k]).abs().max().item() <= 1e-13 * scale, k


def test_refined_host_api_and_passes_batched():
    spec = catalog("varcoef_helmholtz", kappa=10.0)
    tree = build_balanced_refined_tree(4, (0.3, 0.6), 3)
    merged, plain = _pair(tree, spec, 10, 8)
    f = lambda pts: np.sin(2 * pts[:, 0]) + pts[:, 1]  # noqa: E731
    a, b = merged.solve(f=f), plain.solve(f=f)
    scale = np.abs(b.u).max()
    assert np.abs(a.u - b.u).max() <= 1e-13 * scale
    st_a = downward_pass(merged, f, upward_pass(merged))
    st_b = downward_pass(plain, f, upward_pass(plain))
    assert np.abs(st_a.u - st_b.u).max() <= 1e-13 * scale
    assert np.abs(np.asarray(st_a.w) - np.asarray(st_b.w)).max() <= 1e-13 * max(np.abs(st_b.w).max(), 1.0)
