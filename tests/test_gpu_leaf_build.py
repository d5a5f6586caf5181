"""hps_leaf_build operators vs the oracle's leaf_ops (reference leaf.py:124-163) for a
variable-coefficient operator with a mixed-derivative term (config 2's coefficients), on every
assembly path: the fused shared-memory kernel with 16-byte row stores (p = 16), with scalar
stores (odd p: odd row length), and the two-kernel assembly + GEMM path (p = 26 > 24)."""
import numpy as np
import pytest

from oracle import hps_oracle as orc
from paper_1612_02736_b200 import build_stage, build_uniform_tree, problems

pytestmark = pytest.mark.gpu
UNIT = (0.0, 1.0, 0.0, 1.0)


@pytest.mark.parametrize("n,p,q", [(2, 16, 15), (2, 9, 8), (4, 13, 11), (2, 26, 25), (8, 16, 15)])
def test_leaf_operators_match_oracle(n, p, q):
    tree = build_uniform_tree(UNIT, n)
    spec = problems.config2_spec()
    solver = build_stage(tree, spec, p, q)
    cf = orc.coef_functions(spec)
    tol = 1e-10 if p < 32 else 1e-9
    leaves = [nd.id for nd in tree.nodes if nd.is_leaf]
    for nid in leaves[:: max(1, len(leaves) // 6)]:
        ref = orc.leaf_ops(tree.nodes[nid].bounds, cf, p, q)
        got = solver.leaf_ops[nid]
        for name in ("S", "F", "H"):
            a, b = getattr(got, name), ref[name]
            assert a.shape == b.shape
            assert np.abs(a - b).max() <= tol * np.abs(b).max(), (name, nid)
