"""Archive interop, host side (no GPU): archives written by the reference's own
persist_operators (tests/golden/ref_archive_*.sdtn, make_golden.py --only-archive) parse with
this package's reader (framing, checksums, Fortran-ordered LAPACK sections), and the CPU oracle
solving with those archived operators reproduces the reference's own solve of the reloaded
archive (reference archive.py:113-177)."""
import json
import os

import numpy as np
import pytest

from hps_testutil import GOLDEN, golden, oracle_ops_from_archive, rel_maxdiff
from oracle import hps_oracle as orc
from paper_1612_02736_b200.archive import ArchiveError, read_archive
from paper_1612_02736_b200.geometry import MeshSpec, build_mesh, enumerate_gauss_nodes
from paper_1612_02736_b200.model import catalog


def _mesh(header):
    tree = build_mesh(MeshSpec.from_json(json.dumps(header["mesh"])))
    return tree, enumerate_gauss_nodes(tree, header["q"])


def test_reference_archive_sections():
    header, arrays = read_archive(os.path.join(GOLDEN, "ref_archive_stored.sdtn"))
    assert "flavor" not in header and header["mode"] == "stored" and header["p"] == 9
    tree, plan = _mesh(header)
    assert any(plan.node[n.id].wrap is not None for n in tree.nodes if not n.is_leaf)
    for node in tree.nodes:
        if node.is_leaf:
            assert arrays[f"leaf/{node.id}/S"].shape == (81, 32)
            assert arrays[f"leaf/{node.id}/F"].shape == (81, 49)
        else:
            lu = arrays[f"parent/{node.id}/lu"]
            assert lu.flags.f_contiguous and lu.shape[0] == plan.node[node.id].j3.size


@pytest.mark.parametrize("mode", ["stored", "econ"])
def test_oracle_solves_reference_archive(mode):
    header, arrays = read_archive(os.path.join(GOLDEN, f"ref_archive_{mode}.sdtn"))
    tree, plan = _mesh(header)
    spec = catalog(header["spec"]["name"], **header["spec"]["params"])
    if mode == "econ":
        ops = orc.build(tree, spec, header["p"], header["q"], plan)  # leaves refactored, as econ does
        ops["parents"] = oracle_ops_from_archive(header, arrays, tree, plan, spec)["parents"]
    else:
        ops = oracle_ops_from_archive(header, arrays, tree, plan, spec)
    fx = golden(f"ref_archive_{mode}_solution.npz")
    st = orc.solve(ops)
    assert rel_maxdiff(st["u"], fx["u"]) < 1e-12
    g = {lf.id: np.cos(np.arange(49) * 0.1 + lf.id) for lf in tree.leaves()}
    st2 = orc.solve(ops, lambda pts: pts[:, 0] * pts[:, 1], g)
    assert rel_maxdiff(st2["u"], fx["fg_u"]) < 1e-12
    ids = fx["fg_leaf_ids"]
    assert rel_maxdiff(np.stack([st2["leaf_solutions"][int(i)] for i in ids]), fx["fg_leaf_sol"]) < 1e-12


def test_reader_rejects_corruption(tmp_path):
    data = bytearray(open(os.path.join(GOLDEN, "ref_archive_econ.sdtn"), "rb").read())
    bad = tmp_path / "bad.sdtn"
    bad.write_bytes(bytes(data[:-25]))
    with pytest.raises(ArchiveError, match="truncated|checksum"):
        read_archive(bad)
    data[len(data) // 2] ^= 0x40
    bad.write_bytes(bytes(data))
    with pytest.raises(ArchiveError, match="checksum"):
        read_archive(bad)
