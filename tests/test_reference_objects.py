"""Reference objects through the drop-in boundary: specdtn's own
DomainTree, MergePlan and ProblemSpec (geometry.py:139-193, 444-472; model.py:58-131) are accepted
unchanged by this package's build_stage. Runs only where the reference package is importable (the
build container, from /root/reference); skipped elsewhere (the GPU box has no /root/reference).

What is checked on the host: the plan-derived merge tables built from the reference's plan equal
the ones built from this package's plan; the on-device coefficient evaluation (sympy -> torch, here
on CPU tensors) of the reference's CoefficientField equals the reference's own callables; and
build_stage walks the reference objects through plan checks, ellipticity and order validation up to
the device boundary. With a GPU present the same objects build and solve, checked against the
reference's own solve."""
import os
import sys

import numpy as np
import pytest
import torch

REF_SRC = "/root/reference/pkg/src"
if os.path.isdir(REF_SRC) and REF_SRC not in sys.path:
    sys.path.append(REF_SRC)
specdtn = pytest.importorskip("specdtn")

from specdtn import geometry as rgeo  # noqa: E402
from specdtn import model as rmodel  # noqa: E402

from paper_1612_02736_b200 import build_stage, build_uniform_tree, enumerate_gauss_nodes, problems  # noqa: E402
from paper_1612_02736_b200 import coeffs  # noqa: E402
from paper_1612_02736_b200.solver import _plan_tables  # noqa: E402

UNIT = (0.0, 1.0, 0.0, 1.0)


def _ref_mesh():
    tree = rgeo.build_uniform_tree(UNIT, 4)
    rgeo.refine_near_point(tree, rgeo.RefinementSpec((0.3, 0.7), 1))
    return tree


def _our_mesh():
    from paper_1612_02736_b200 import RefinementSpec, refine_near_point
    tree = build_uniform_tree(UNIT, 4)
    refine_near_point(tree, RefinementSpec((0.3, 0.7), 1))
    return tree


def test_plan_tables_from_reference_plan():
    rt, ot = _ref_mesh(), _our_mesh()
    rp, op = rgeo.enumerate_gauss_nodes(rt, 8), enumerate_gauss_nodes(ot, 8)
    a, b = _plan_tables(rt, rp), _plan_tables(ot, op)
    assert list(a["leaf_groups"].items()) == list(b["leaf_groups"].items())
    assert a["depth"] == b["depth"]
    assert len(a["levels"]) == len(b["levels"])
    for (da, ia, ga), (db, ib, gb) in zip(a["levels"], b["levels"]):
        assert da == db and ia == ib and len(ga) == len(gb)
        for (ids1, r1, s1), (ids2, r2, s2) in zip(ga, gb):
            assert ids1 == ids2 and s1 == s2 and np.array_equal(r1, r2)


def test_reference_coefficients_evaluate_on_torch():
    cf = rmodel.CoefficientField(
        c11="1 + sin(2*pi*x1)*cos(2*pi*x2)/2", c12="sin(2*pi*(x1 + x2))/10",
        c22="1 + cos(4*pi*x1)*sin(2*pi*x2)/2", c1="cos(3*pi*x2)", c2="sin(3*pi*x1)", c=0)
    pts = np.random.default_rng(3).uniform(size=(500, 2))
    got = coeffs.evaluate(cf, torch.as_tensor(pts)).numpy()
    want = np.stack([getattr(cf, n)(pts) * np.ones(len(pts)) for n in ("c11", "c12", "c22", "c1", "c2", "c")])
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-14)


def test_build_stage_accepts_reference_objects():
    tree = _ref_mesh()
    plan = rgeo.enumerate_gauss_nodes(tree, 8)
    spec = rmodel.catalog("manufactured", u="sin(pi*x1)*sin(pi*x2)")
    if not torch.cuda.is_available():
        # every host-side step runs on the foreign objects; the first device step is the boundary
        with pytest.raises(RuntimeError, match="needs a CUDA device"):
            build_stage(tree, spec, 9, 8, plan=plan)
        return
    from specdtn.solver import build_stage as ref_build
    ours = build_stage(tree, spec, 9, 8, plan=plan).solve()
    ref = ref_build(tree, spec, 9, 8, plan=plan).solve()
    scale = np.abs(ref.u).max()
    assert np.abs(ours.u - ref.u).max() <= 1e-10 * scale
    for nid, v in ref.leaf_solutions.items():
        assert np.abs(ours.leaf_solutions[nid] - v).max() <= 1e-10 * scale


def test_problem_catalog_matches_reference():
    # the configs' problem definitions evaluate identically through either package
    ours = problems.config2_spec()
    pts = np.random.default_rng(4).uniform(size=(300, 2))
    ref_cf = rmodel.CoefficientField(
        c11="1 + sin(2*pi*x1)*cos(2*pi*x2)/2", c12="sin(2*pi*(x1 + x2))/10",
        c22="1 + cos(4*pi*x1)*sin(2*pi*x2)/2", c1="cos(3*pi*x2)", c2="sin(3*pi*x1)", c=0)
    for n in ("c11", "c12", "c22", "c1", "c2", "c"):
        np.testing.assert_allclose(getattr(ours.coefficients, n)(pts) * np.ones(len(pts)),
                                   getattr(ref_cf, n)(pts) * np.ones(len(pts)), rtol=0, atol=1e-15)


@pytest.mark.parametrize("mode", ["stored", "econ"])
def test_reference_loads_gpu_written_archive(mode):
    """The reverse interop direction: archives written on the B200 by
    persist_operators(..., flavor="reference") (tools/write_gpu_archive.py, committed as
    tests/golden/gpu_archive_*.sdtn with the GPU's own solve) load in the reference's own
    load_operators (archive.py:113-177), and the reference's solve reproduces the GPU solve."""
    from specdtn.archive import load_operators as ref_load
    from hps_testutil import GOLDEN, golden
    solver = ref_load(os.path.join(GOLDEN, f"gpu_archive_{mode}.sdtn"))
    assert solver.mode == mode
    st = solver.solve(f=lambda pts: pts[:, 0] - 2 * pts[:, 1])
    fx = golden(f"gpu_archive_{mode}_solution.npz")
    scale = np.abs(fx["u"]).max()
    assert np.abs(st.u - fx["u"]).max() <= 1e-12 * scale
    for k, nid in enumerate(fx["leaf_ids"]):
        assert np.abs(st.leaf_solutions[int(nid)] - fx["leaf_sol"][k]).max() <= 1e-12 * scale
