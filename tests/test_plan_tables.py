"""Host tables of build_stage (solver._plan_tables): merge groups with their stacked child-position
rows must equal the per-node plan, be cached on the plan object, and work for a plan object that
refuses new attributes."""
import numpy as np

from paper_1612_02736_b200 import build_balanced_refined_tree, build_uniform_tree, enumerate_gauss_nodes
from paper_1612_02736_b200.solver import _depths, _plan_tables


def _check(tree, plan):
    t = _plan_tables(tree, plan)
    leaves = sorted(n for ids in t["leaf_groups"].values() for n in ids)
    assert leaves == sorted(lf.id for lf in tree.leaves())
    assert t["depth"] == _depths(tree)
    seen = []
    prev = None
    for d, level_ids, groups in t["levels"]:
        assert prev is None or d < prev  # deepest level first
        prev = d
        assert sorted(level_ids) == sorted(n for n, dd in t["depth"].items() if dd == d and not tree.nodes[n].is_leaf)
        for ids, rows, same in groups:
            seen.extend(ids)
            for slot, nid in enumerate(ids):
                en = plan.node[nid]
                want = np.concatenate([en.pos1_a, en.pos3_a, en.pos2_b, en.pos3_b])
                got = rows if same else rows[slot]
                np.testing.assert_array_equal(got, want)
    assert sorted(seen) == sorted(n for n in range(len(tree.nodes)) if not tree.nodes[n].is_leaf)
    return t


def test_uniform_tree_tables_and_cache():
    tree = build_uniform_tree((0.0, 1.0, 0.0, 1.0), 8)
    plan = enumerate_gauss_nodes(tree, 15)
    t = _check(tree, plan)
    assert all(same for _, _, groups in t["levels"] for _, _, same in groups)  # uniform: shared rows
    assert _plan_tables(tree, plan) is t  # cached on the plan


def test_refined_tree_tables():
    tree = build_balanced_refined_tree(4, (0.3, 0.7), 3)
    _check(tree, enumerate_gauss_nodes(tree, 14))


def test_plan_without_attribute_support():
    tree = build_uniform_tree((0.0, 1.0, 0.0, 1.0), 4)
    plan = enumerate_gauss_nodes(tree, 15)

    class Frozen:
        __slots__ = ("node",)

    fp = Frozen()
    fp.node = plan.node
    _check(tree, fp)
