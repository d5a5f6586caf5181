"""Persist / reload a GPU-built solver (reference archive.py:1-177, same container framing).

Layout (little-endian), as the reference's SDTNARC1:

    magic b"SDTNARC1" | u64 header length | header JSON | u32 crc32(header)
    per array section, in header order: u64 payload length | raw bytes | u32 crc32(payload)

The header carries ``"flavor": "b200"``: the sections are this package's level-batched device
operators (per leaf shape group: [F_ii | S_ie], H, column order; per merge group: [X | S], T_ei,
column order, wrap interpolators) rather than the reference's per-node LU factors. The mesh is
rebuilt deterministically from its MeshSpec, so index sets match bit for bit and a reloaded
solver reproduces in-memory solves exactly. Economy-mode archives store the coefficient
samples instead of the leaf operators.
"""

from __future__ import annotations

import json
import struct
import zlib

import numpy as np
import torch

from .geometry import MeshSpec, build_mesh, enumerate_gauss_nodes
from .model import catalog
from .spectral import shape_constants
from . import solver as S

MAGIC = b"SDTNARC1"


class ArchiveError(RuntimeError):
    """Archive is malformed, truncated, or from an incompatible version."""


def _arrays(solver) -> dict:
    out = {}
    for i, g in enumerate(solver.leaf_groups):
        if solver.mode == "econ":
            out[f"lg{i}/coef"] = g.coef
        else:
            out[f"lg{i}/fs"] = g.fs
            out[f"lg{i}/h"] = g.h
            out[f"lg{i}/perm"] = g.perm
    for i, g in enumerate(solver.parent_groups):
        out[f"pg{i}/tei"] = g.tei
        out[f"pg{i}/perm"] = g.perm
        if g.wrap is not None:
            out[f"pg{i}/xsw"] = g.wrap["xsw"]
            out[f"pg{i}/qd"] = g.wrap["qd_dev"]
            out[f"pg{i}/pu"] = g.wrap["pu_dev"]
            out[f"pg{i}/pd"] = torch.as_tensor(g.wrap["pd"])
        else:
            out[f"pg{i}/xs"] = g.xs
    return {k: np.ascontiguousarray(v.detach().cpu().numpy()) for k, v in out.items()}


def persist_operators(solver, path) -> None:
    """Write the solver to ``path`` (checksummed sections, bit-exact reload)."""
    mesh = getattr(solver.tree, "mesh_spec", None)
    if mesh is None:
        raise ArchiveError("solver's tree carries no mesh description")
    key = getattr(solver.spec, "catalog_key", None)
    if key is None and solver.mode == "econ":
        raise ArchiveError("economy-mode archives need a catalog-reconstructible problem "
                           "(coefficient callables cannot be serialized)")
    arrays = _arrays(solver)
    order = sorted(arrays)
    header = {
        "version": 1, "flavor": "b200", "mode": solver.mode, "p": solver.p, "q": solver.q,
        "mesh": json.loads(mesh.to_json()),
        "spec": None if key is None else {"name": key[0], "params": key[1]},
        "build_seconds": solver.build_seconds,
        "leaf_groups": [{"key": list(map(float, g.key)), "ids": list(map(int, g.ids)), "first_row": g.first_row}
                        for g in solver.leaf_groups],
        "parent_groups": [{"depth": g.depth, "ids": list(map(int, g.ids)), "m3": g.m3, "n1": g.n1, "n2": g.n2,
                           "lda": g.lda, "ldb": g.ldb, "ec": None if g.wrap is None else g.wrap["ec"]}
                          for g in solver.parent_groups],
        "arrays": [{"key": k, "dtype": arrays[k].dtype.str, "shape": list(arrays[k].shape)} for k in order],
    }
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        blob = json.dumps(header).encode()
        fh.write(struct.pack("<Q", len(blob)))
        fh.write(blob)
        fh.write(struct.pack("<I", zlib.crc32(blob)))
        for k in order:
            payload = arrays[k].astype(arrays[k].dtype.newbyteorder("<"), copy=False).tobytes()
            fh.write(struct.pack("<Q", len(payload)))
            fh.write(payload)
            fh.write(struct.pack("<I", zlib.crc32(payload)))


def _read_exact(fh, size: int, what: str) -> bytes:
    data = fh.read(size)
    if len(data) != size:
        raise ArchiveError(f"archive truncated while reading {what}")
    return data


def load_operators(path, spec=None):
    """Rebuild a GPU solver from an archive written by persist_operators."""
    with open(path, "rb") as fh:
        if _read_exact(fh, len(MAGIC), "magic") != MAGIC:
            raise ArchiveError("not a solver archive (bad magic)")
        (hlen,) = struct.unpack("<Q", _read_exact(fh, 8, "header length"))
        blob = _read_exact(fh, hlen, "header")
        (crc,) = struct.unpack("<I", _read_exact(fh, 4, "header checksum"))
        if zlib.crc32(blob) != crc:
            raise ArchiveError("header checksum mismatch")
        header = json.loads(blob)
        if header.get("version") != 1 or header.get("flavor") != "b200":
            raise ArchiveError(f"unsupported archive version/flavor {header.get('version')}/{header.get('flavor')}")
        arrays = {}
        for meta in header["arrays"]:
            (plen,) = struct.unpack("<Q", _read_exact(fh, 8, meta["key"]))
            payload = _read_exact(fh, plen, meta["key"])
            (crc,) = struct.unpack("<I", _read_exact(fh, 4, meta["key"] + " checksum"))
            if zlib.crc32(payload) != crc:
                raise ArchiveError(f"checksum mismatch in section {meta['key']}")
            arrays[meta["key"]] = np.frombuffer(payload, dtype=np.dtype(meta["dtype"])).reshape(meta["shape"]).copy()

    tree = build_mesh(MeshSpec.from_json(json.dumps(header["mesh"])))
    p, q = header["p"], header["q"]
    plan = enumerate_gauss_nodes(tree, q)
    if spec is None:
        if header["spec"] is None:
            raise ArchiveError("archive has no catalog key; pass the problem spec explicitly")
        spec = catalog(header["spec"]["name"], **header["spec"]["params"])
    solver = S.FactorizedSolver(tree, plan, spec, p, q, header["mode"])
    solver.build_seconds = header.get("build_seconds", 0.0)
    dev = solver.device

    def dev_t(k, dtype=None):
        try:
            a = arrays[k]
        except KeyError:
            raise ArchiveError(f"archive is missing section {k!r}") from None
        return torch.as_tensor(a, device=dev) if dtype is None else torch.as_tensor(a, dtype=dtype, device=dev)

    leaf_ids = []
    for i, g in enumerate(header["leaf_groups"]):
        w, h = g["key"]
        sc = shape_constants(p, q, float(w), float(h))
        grp = S._LeafGroup((w, h), g["ids"], sc, first_row=g["first_row"])
        grp.consts = S._leaf_consts(sc, dev)
        L = len(g["ids"])
        grp.anorm = torch.empty(L, dtype=torch.float64, device=dev)
        grp.ainvnorm = torch.empty(L, dtype=torch.float64, device=dev)
        grp.status = torch.zeros(L, dtype=torch.int32, device=dev)
        if header["mode"] == "econ":
            grp.coef = dev_t(f"lg{i}/coef")
            # the leaf stage re-runs per solve; one run here recovers the column order (perm)
            S._leaf_build_call(grp, p, q, S._ext.load(), S._stream_ptr())
        else:
            grp.fs, grp.h, grp.perm = dev_t(f"lg{i}/fs"), dev_t(f"lg{i}/h"), dev_t(f"lg{i}/perm")
        for slot, nid in enumerate(g["ids"]):
            solver.leaf_loc[nid] = (i, slot)
        leaf_ids.extend(g["ids"])
        solver.leaf_groups.append(grp)
    solver._leaf_ids = leaf_ids
    solver._n_leaves = len(leaf_ids)
    for i, g in enumerate(header["parent_groups"]):
        grp = S._ParentGroup(g["depth"], g["ids"], g["m3"], g["n1"], g["n2"], g["lda"], g["ldb"])
        grp.tei, grp.perm = dev_t(f"pg{i}/tei"), dev_t(f"pg{i}/perm")
        if g["ec"] is not None:
            grp.wrap = {"ec": g["ec"], "xsw": dev_t(f"pg{i}/xsw"), "qd_dev": dev_t(f"pg{i}/qd"),
                        "pu_dev": dev_t(f"pg{i}/pu"), "pd": arrays[f"pg{i}/pd"],
                        "pu": arrays[f"pg{i}/pu"]}
        else:
            grp.xs = dev_t(f"pg{i}/xs")
        solver.parent_groups.append(grp)
    solver.depth = S._depths(tree)
    solver._layout = S._layout(solver)
    if header["mode"] == "econ":
        for grp in solver.leaf_groups:
            grp.fs = grp.h = None
    return solver
