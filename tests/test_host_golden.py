"""Host constants and the merge plan of this package vs golden vectors from the reference."""
import numpy as np
import pytest

from paper_1612_02736_b200 import spectral
from paper_1612_02736_b200.geometry import (MeshSpec, build_balanced_refined_tree, build_forest, build_mesh,
                                            build_uniform_tree, count_chebyshev_dofs, enumerate_gauss_nodes,
                                            refine_near_point)
from hps_testutil import golden

SHAPES = ((16, 15, 0.25, 0.25), (12, 11, 1.0, 1.0), (9, 8, 0.5, 0.25),
          (16, 14, 1.0 / 2048, 1.0 / 2048), (32, 31, 1.0 / 32, 1.0 / 32))


@pytest.mark.parametrize("shape", SHAPES)
def test_shape_constants_match_reference(shape):
    p, q, w, h = shape
    g = golden("spectral.npz")
    key = f"p{p}q{q}w{w!r}h{h!r}"
    sc = spectral.shape_constants(p, q, w, h)
    np.testing.assert_array_equal(sc.i_ce, g[key + "_i_ce"])
    np.testing.assert_array_equal(sc.i_ci, g[key + "_i_ci"])
    np.testing.assert_allclose(sc.lift, g[key + "_lift"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(sc.dx, g[key + "_dx"], rtol=1e-14, atol=1e-14 * np.abs(sc.dx).max())
    if key + "_flux" in g:
        ref = g[key + "_flux"]
        np.testing.assert_allclose(sc.flux, ref, rtol=0, atol=1e-13 * np.abs(ref).max())
    else:
        v = np.random.default_rng(5).standard_normal(p * p)
        ref = g[key + "_fluxv"]
        np.testing.assert_allclose(sc.flux @ v, ref, rtol=0, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("q", [8, 14])
def test_edge_interpolators(q):
    g = golden("spectral.npz")
    up, down = spectral.edge_interpolators(q)
    np.testing.assert_allclose(up, g[f"edge{q}_up"], atol=1e-14)
    np.testing.assert_allclose(down, g[f"edge{q}_down"], atol=1e-14)
    with pytest.raises(ValueError, match="even q"):
        spectral.edge_interpolators(q + 1)


def _check_plan(prefix, tree, plan):
    g = golden("plans.npz")
    np.testing.assert_array_equal(plan.coords, g[prefix + "coords"])
    for nid in range(len(tree.nodes)):
        e = plan.node[nid]
        np.testing.assert_array_equal(e.ext, g[f"{prefix}n{nid}_ext"])
        np.testing.assert_array_equal(e.ext_mergeorder, g[f"{prefix}n{nid}_extmo"])
        if tree.nodes[nid].is_leaf:
            continue
        for k in ("j3", "pos1_a", "pos3_a", "pos2_b", "pos3_b"):
            np.testing.assert_array_equal(getattr(e, k), g[f"{prefix}n{nid}_{k}"])
        if f"{prefix}n{nid}_wperm" in g:
            assert e.wrap is not None
            np.testing.assert_array_equal(e.wrap.perm, g[f"{prefix}n{nid}_wperm"])
            np.testing.assert_array_equal(e.wrap.fine, g[f"{prefix}n{nid}_wfine"])
            np.testing.assert_array_equal(e.wrap.ext, g[f"{prefix}n{nid}_wext"])
            kinds = np.array([0 if b[0] == "identity" else 1 for b in e.wrap.blocks])
            np.testing.assert_array_equal(kinds, g[f"{prefix}n{nid}_wblocks"])
        else:
            assert e.wrap is None


def test_plan_uniform():
    t = build_uniform_tree((0, 1, 0, 1), 4)
    _check_plan("u4q15_", t, enumerate_gauss_nodes(t, 15))


def test_plan_refined_reference_native():
    t = build_uniform_tree((0, 1, 0, 1), 4)
    refine_near_point(t, (0.5, 0.5), 1)
    _check_plan("r4q8_", t, enumerate_gauss_nodes(t, 8))


def test_plan_config4_balanced():
    t = build_balanced_refined_tree(8, (0.3, 0.7), 8)
    assert len(t.leaves()) == 175 and len(t.nodes) == 349
    plan = enumerate_gauss_nodes(t, 14)
    assert plan.n_gauss == 6804
    assert sum(e.wrap is not None for e in plan.node.values()) == 32
    _check_plan("cfg4q14_", t, plan)


def test_chebyshev_dof_count():
    t = build_uniform_tree((0, 1, 0, 1), 4)
    assert count_chebyshev_dofs(t, 16) == (4 * 15 + 1) ** 2 == 3721


def test_plan_refined_lshape_forest():
    lshape = ((0.0, 1.0, 0.0, 1.0), (1.0, 2.0, 0.0, 1.0), (0.0, 1.0, 1.0, 2.0))
    t = build_forest(lshape, 2)
    refine_near_point(t, (1.0, 1.0), 1)
    _check_plan("lshape_", t, enumerate_gauss_nodes(t, 8))


def test_mesh_spec_round_trip():
    lshape = ((0.0, 1.0, 0.0, 1.0), (1.0, 2.0, 0.0, 1.0), (0.0, 1.0, 1.0, 2.0))
    t = build_forest(lshape, 2)
    refine_near_point(t, (1.0, 1.0), 1)
    t2 = build_mesh(MeshSpec.from_json(t.mesh_spec.to_json()))
    assert [n.bounds for n in t.nodes] == [n.bounds for n in t2.nodes]
    assert [n.children for n in t.nodes] == [n.children for n in t2.nodes]
