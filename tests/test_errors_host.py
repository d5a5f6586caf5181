"""The reference's error contract on the host side of the drop-in (SURVEY.md 8b "errors" row).
These failures are raised by build_stage before any device work, so they run without a GPU:
invalid merge order (reference solver.py:384-400, test_solver.py:219-224), 2:1 violations and
disjoint forest glue (geometry.py:517-521, 628-630; test_geometry.py:200, 235), bad mode / p < q+1
(solver.py:368-371), RefinementSpec validation (geometry.py:208-213)."""
import math

import numpy as np
import pytest

from paper_1612_02736_b200 import (MeshConformityError, RefinementSpec, build_forest, build_stage,
                                   build_uniform_tree, catalog, enumerate_gauss_nodes, refine_near_point)

UNIT = (0.0, 1.0, 0.0, 1.0)


def test_invalid_order_rejected():  # test_solver.py:219-224
    tree = build_uniform_tree(UNIT, 2)
    with pytest.raises(ValueError, match="before its children"):
        build_stage(tree, catalog("laplace"), 9, 8, order=range(len(tree.nodes)))


def test_order_not_a_permutation():  # solver.py:384-386
    tree = build_uniform_tree(UNIT, 2)
    with pytest.raises(ValueError, match="permutation"):
        build_stage(tree, catalog("laplace"), 9, 8, order=[0, 1, 2])


def test_mode_and_order_checks():  # solver.py:368-371
    tree = build_uniform_tree(UNIT, 2)
    with pytest.raises(ValueError, match="unknown mode"):
        build_stage(tree, catalog("laplace"), 9, 8, mode="lazy")
    with pytest.raises(ValueError, match="p >= q\\+1"):
        build_stage(tree, catalog("laplace"), 8, 8)


def test_ratio_above_two_rejected():  # test_geometry.py:192-199
    tree = build_uniform_tree(UNIT, 2)
    refine_near_point(tree, RefinementSpec((0.45, 0.25), 2, threshold=1e-6))
    with pytest.raises(MeshConformityError, match="2:1"):
        enumerate_gauss_nodes(tree, 4)
    with pytest.raises(MeshConformityError, match="2:1"):
        build_stage(tree, catalog("laplace"), 9, 8)


def test_disjoint_glue_rejected():  # test_geometry.py:231-235
    tree = build_forest([(0.0, 1.0, 0.0, 1.0), (2.0, 3.0, 0.0, 1.0)], 2)
    with pytest.raises(MeshConformityError, match="share no interface"):
        enumerate_gauss_nodes(tree, 4)
    with pytest.raises(MeshConformityError, match="share no interface"):
        build_stage(tree, catalog("laplace"), 9, 8)


def test_refinement_spec_contract():  # geometry.py:196-213, 333-357
    with pytest.raises(ValueError, match=">= 0"):
        RefinementSpec((0.5, 0.5), -1)
    with pytest.raises(ValueError, match="positive"):
        RefinementSpec((0.5, 0.5), 1, threshold=0.0)
    assert RefinementSpec((0.5, 0.5), 1).threshold == math.sqrt(2.0)
    a, b = build_uniform_tree(UNIT, 4), build_uniform_tree(UNIT, 4)
    refine_near_point(a, RefinementSpec((0.3, 0.7), 2))   # reference calling convention
    refine_near_point(b, (0.3, 0.7), 2)                    # positional form
    assert [n.bounds for n in a.nodes] == [n.bounds for n in b.nodes]
    with pytest.raises(ValueError, match="outside the domain"):
        refine_near_point(a, RefinementSpec((2.0, 0.5), 1))
    assert a.mesh_spec.refinements[-1] == RefinementSpec((0.3, 0.7), 2)


def test_load_shape_mismatch_message():  # solver.py:249-252 (host-side table check)
    from paper_1612_02736_b200.solver import FactorizedSolver
    s = FactorizedSolver.__new__(FactorizedSolver)
    tree = build_uniform_tree(UNIT, 2)
    s.p, s.q, s.spec, s.tree = 9, 8, catalog("laplace"), tree
    s._leaf_ids = [n.id for n in tree.leaves()]
    s._n_leaves = len(s._leaf_ids)
    g = {n: np.zeros(49) for n in s._leaf_ids}
    assert s._leaf_table(g).shape == (4, 49)
    g[s._leaf_ids[2]] = np.zeros(48)
    with pytest.raises(ValueError, match=f"leaf {s._leaf_ids[2]} load has shape \\(48,\\), expected \\(49,\\)"):
        s._leaf_table(g)
