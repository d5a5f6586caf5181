"""Shared helpers for the test suite (golden fixture access, tree helpers)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def rel_maxdiff(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    scale = max(np.abs(b).max(), 1e-300)
    return float(np.abs(a - b).max() / scale)


def oracle_ops_from_archive(header, arrays, tree, plan, spec):
    """Oracle ops dict (oracle/hps_oracle.py build() layout) from reference-layout archive
    sections (reference archive.py:47-62), so the CPU oracle can solve with archived operators."""
    from oracle import hps_oracle as orc
    leaves, parents = {}, {}
    q = header["q"]
    for node in tree.nodes:
        nid = node.id
        if node.is_leaf:
            if header["mode"] == "stored":
                leaves[nid] = {k: arrays[f"leaf/{nid}/{k}"] for k in ("S", "F", "H")}
            continue
        po = {"lu_piv": (arrays[f"parent/{nid}/lu"], arrays[f"parent/{nid}/piv"].astype(np.int32)),
              "S": arrays[f"parent/{nid}/S"], "Tei": arrays[f"parent/{nid}/Tei"]}
        e = plan.node[nid]
        if e.wrap is not None:
            pu, pd = orc.wrap_matrices(e.wrap, q)
            po["wrap"] = (pu, pd, e.wrap.perm, e.wrap.fine)
        parents[nid] = po
    return dict(tree=tree, plan=plan, p=header["p"], q=q, leaves=leaves, parents=parents, spec=spec)
