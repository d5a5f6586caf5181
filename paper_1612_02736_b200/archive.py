"""Persist / reload a GPU-built solver (reference archive.py:1-177, same container framing).

Layout (little-endian), as the reference's SDTNARC1:

    magic b"SDTNARC1" | u64 header length | header JSON | u32 crc32(header)
    per array section, in header order: u64 payload length | raw bytes | u32 crc32(payload)

Two payload flavors share that framing:

* ``flavor="reference"`` (no ``flavor`` key in the header, exactly what specdtn writes): per-node
  sections ``leaf/{id}/S,F,H`` and ``parent/{id}/lu,piv,S,Tei`` (reference archive.py:47-62).
  ``load_operators`` reads archives written by the reference itself: leaf operators go to the
  device as [F_ii | S_ie] and H, each box's X = Delta^-1 is formed from the archived LAPACK
  (lu, piv). ``persist_operators(..., flavor="reference")`` writes an archive the reference's
  own ``load_operators`` accepts; the (lu, piv) sections are LAPACK's factors of the device's
  interface blocks (FactorizedSolver.parent_ops).
* ``flavor="b200"`` (default): this package's level-batched device operators (per leaf shape
  group: [F_ii | S_ie], H, column order; per merge group: [X | S], T_ei, column order, wrap
  interpolators); bit-exact reload of the GPU solver, not readable by the reference.

The mesh is rebuilt deterministically from its MeshSpec, so index sets match bit for bit.
Economy-mode archives store no leaf operators (b200: the coefficient samples instead).
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
FLAVORS = ("b200", "reference")


class ArchiveError(RuntimeError):
    """Archive is malformed, truncated, or from an incompatible version."""


def _mem_order(arr: np.ndarray) -> str:
    """Memory order of a section (reference archive.py:38-44): LAPACK factors are Fortran."""
    return "F" if (arr.flags.f_contiguous and not arr.flags.c_contiguous) else "C"


def reference_arrays(solver) -> dict:
    """Per-node sections in the reference's layout (reference archive.py:47-62)."""
    arrays = {}
    for nid, ops in solver.leaf_ops.items():
        arrays[f"leaf/{nid}/S"] = ops.S
        arrays[f"leaf/{nid}/F"] = ops.F
        arrays[f"leaf/{nid}/H"] = ops.H
    for nid, ops in solver.parent_ops.items():
        arrays[f"parent/{nid}/lu"] = ops.lu_piv[0]
        arrays[f"parent/{nid}/piv"] = ops.lu_piv[1]
        arrays[f"parent/{nid}/S"] = ops.s_gi_ge
        arrays[f"parent/{nid}/Tei"] = ops.t_ei
    return arrays


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


def _write(path, header: dict, arrays: dict, order: list) -> None:
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        blob = json.dumps(header).encode()
        fh.write(struct.pack("<Q", len(blob)))
        fh.write(blob)
        fh.write(struct.pack("<I", zlib.crc32(blob)))
        for k in order:
            arr = arrays[k]
            if arr.dtype.byteorder == ">":
                arr = arr.astype(arr.dtype.newbyteorder("<"))
            if not (arr.flags.c_contiguous or arr.flags.f_contiguous):
                arr = np.ascontiguousarray(arr)
            payload = arr.tobytes(order="A")
            fh.write(struct.pack("<Q", len(payload)))
            fh.write(payload)
            fh.write(struct.pack("<I", zlib.crc32(payload)))


def persist_operators(solver, path, flavor: str = "b200") -> None:
    """Write the solver to ``path`` (checksummed sections). flavor "b200": bit-exact reload of
    this GPU solver; flavor "reference": the reference's per-node layout, loadable by specdtn's
    own load_operators (reference archive.py:65-101)."""
    if flavor not in FLAVORS:
        raise ValueError(f"unknown archive flavor {flavor!r}; expected one of {FLAVORS}")
    mesh = getattr(solver.tree, "mesh_spec", None)
    if mesh is None:
        raise ArchiveError("solver's tree carries no mesh description")
    key = getattr(solver.spec, "catalog_key", None)
    if key is None and solver.mode == "econ":
        raise ArchiveError("economy-mode archives need a catalog-reconstructible problem "
                           "(coefficient callables cannot be serialized)")
    header = {"version": 1, "mode": solver.mode, "p": solver.p, "q": solver.q,
              "mesh": json.loads(mesh.to_json()),
              "spec": None if key is None else {"name": key[0], "params": key[1]},
              "build_seconds": solver.build_seconds}
    if flavor == "reference":
        arrays = reference_arrays(solver)
        order = sorted(arrays)
        header["arrays"] = [{"key": k, "dtype": arrays[k].dtype.str, "shape": list(arrays[k].shape),
                             "order": _mem_order(arrays[k])} for k in order]
        _write(path, header, arrays, order)
        return
    arrays = _arrays(solver)
    order = sorted(arrays)
    header.update({
        "flavor": "b200",
        "leaf_groups": [{"key": list(map(float, g.key)), "ids": list(map(int, g.ids)), "first_row": g.first_row}
                        for g in solver.leaf_groups],
        "parent_groups": [{"depth": g.depth, "ids": list(map(int, g.ids)), "m3": g.m3, "n1": g.n1, "n2": g.n2,
                           "lda": g.lda, "ldb": g.ldb, "ec": None if g.wrap is None else g.wrap["ec"]}
                          for g in solver.parent_groups],
        "arrays": [{"key": k, "dtype": arrays[k].dtype.str, "shape": list(arrays[k].shape)} for k in order]})
    _write(path, header, arrays, order)


def _read_exact(fh, size: int, what: str) -> bytes:
    data = fh.read(size)
    if len(data) != size:
        raise ArchiveError(f"archive truncated while reading {what}")
    return data


def read_archive(path):
    """(header, {key: ndarray}) of an SDTNARC1 archive of either flavor, checksums verified."""
    with open(path, "rb") as fh:
        if _read_exact(fh, len(MAGIC), "magic") != MAGIC:
            raise ArchiveError("not a solver archive (bad magic)")
        (hlen,) = struct.unpack("<Q", _read_exact(fh, 8, "header length"))
        blob = _read_exact(fh, hlen, "header")
        (crc,) = struct.unpack("<I", _read_exact(fh, 4, "header checksum"))
        if zlib.crc32(blob) != crc:
            raise ArchiveError("header checksum mismatch")
        header = json.loads(blob)
        if header.get("version") != 1 or header.get("flavor", "reference") not in FLAVORS:
            raise ArchiveError(f"unsupported archive version/flavor {header.get('version')}/{header.get('flavor')}")
        arrays = {}
        for meta in header["arrays"]:
            (plen,) = struct.unpack("<Q", _read_exact(fh, 8, meta["key"]))
            payload = _read_exact(fh, plen, meta["key"])
            (crc,) = struct.unpack("<I", _read_exact(fh, 4, meta["key"] + " checksum"))
            if zlib.crc32(payload) != crc:
                raise ArchiveError(f"checksum mismatch in section {meta['key']}")
            arr = np.frombuffer(payload, dtype=np.dtype(meta["dtype"]))
            arrays[meta["key"]] = arr.reshape(meta["shape"], order=meta.get("order", "C")).copy(order="A")
    return header, arrays


def load_operators(path, spec=None):
    """Rebuild a GPU solver from an archive written by persist_operators (either flavor) or by
    the reference's own persist_operators (reference archive.py:113-177)."""
    header, arrays = read_archive(path)
    tree = build_mesh(MeshSpec.from_json(json.dumps(header["mesh"])))
    p, q = header["p"], header["q"]
    plan = enumerate_gauss_nodes(tree, q)
    if spec is None:
        if header["spec"] is None:
            raise ArchiveError("archive has no catalog key; pass the problem spec explicitly")
        spec = catalog(header["spec"]["name"], **header["spec"]["params"])
    solver = S.FactorizedSolver(tree, plan, spec, p, q, header["mode"])
    solver.build_seconds = header.get("build_seconds", 0.0)
    if header.get("flavor", "reference") == "reference":
        _load_reference(solver, arrays)
    else:
        _load_b200(solver, header, arrays)
    return solver


def _section(arrays, k):
    try:
        return arrays[k]
    except KeyError:
        raise ArchiveError(f"archive is missing section {k!r}") from None


def _load_reference(solver, arrays):
    """Per-node reference sections -> the device layout: leaf [F_ii | S_ie] rows in i_ci order
    (columns in natural order, perm = identity), H; parent [X | S] with X = lu_solve(lu, I) from
    the archived LAPACK factors, T_ei; wrap interpolators rebuilt from the plan."""
    from scipy.linalg import lu_solve
    p, q, dev = solver.p, solver.q, solver.device
    m, b = (p - 2) ** 2, 4 * q
    S._skeleton(solver)
    for grp in solver.leaf_groups:
        L = len(grp.ids)
        ci = grp.sc.i_ci
        if solver.mode == "econ":
            grp.coef = S._leaf_coefficients(solver, grp)
            S._leaf_build_call(grp, p, q, S._ext.load(), S._stream_ptr())  # column order (perm)
            continue
        fs = np.empty((L, m, m + b))
        h = np.empty((L, b, m))
        for slot, nid in enumerate(grp.ids):
            fs[slot, :, :m] = _section(arrays, f"leaf/{nid}/F")[ci]
            fs[slot, :, m:] = _section(arrays, f"leaf/{nid}/S")[ci]
            h[slot] = _section(arrays, f"leaf/{nid}/H")
        grp.fs, grp.h = S._op_f64(fs, dev), S._op_f64(h, dev)
        grp.perm = torch.arange(m, dtype=torch.int32, device=dev).repeat(L, 1).contiguous()
    for grp in solver.parent_groups:
        m3, e, n = grp.m3, grp.e, len(grp.ids)
        tei = np.empty((n, e, m3))
        xs = []
        for slot, nid in enumerate(grp.ids):
            lu = _section(arrays, f"parent/{nid}/lu")
            piv = _section(arrays, f"parent/{nid}/piv").astype(np.int32)
            x = lu_solve((lu, piv), np.eye(m3))
            xs.append(np.hstack([x, _section(arrays, f"parent/{nid}/S")]))
            tei[slot] = _section(arrays, f"parent/{nid}/Tei")
        grp.tei = S._f64(tei, dev)
        grp.perm = torch.arange(m3, dtype=torch.int32, device=dev).repeat(n, 1).contiguous()
        en = solver.plan.node[grp.ids[0]]
        if en.wrap is not None:
            pu, pd = S._wrap_dense(en.wrap, q)
            ec = pu.shape[1]
            qd = np.zeros((ec, e))
            qd[:, en.wrap.perm] = pd
            grp.wrap = {"pu": pu, "pd": pd, "ec": ec, "qd_dev": S._op_f64(qd, dev), "pu_dev": S._op_f64(pu, dev),
                        "xsw": S._op_f64(xs[0], dev)}
        else:
            grp.xs = S._op_f64(np.stack(xs), dev)
    solver._layout = S._layout(solver)
    if solver.mode == "econ":
        for grp in solver.leaf_groups:
            grp.fs = grp.h = None


def _load_b200(solver, header, arrays):
    p, q, dev = solver.p, solver.q, solver.device
    tree = solver.tree

    def dev_t(k, dtype=None):
        a = _section(arrays, k)
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
            grp.fs = S._op_f64(_section(arrays, f"lg{i}/fs"), dev)
            grp.h = S._op_f64(_section(arrays, f"lg{i}/h"), dev)
            grp.perm = dev_t(f"lg{i}/perm")
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
            grp.wrap = {"ec": g["ec"], "xsw": S._op_f64(_section(arrays, f"pg{i}/xsw"), dev),
                        "qd_dev": S._op_f64(_section(arrays, f"pg{i}/qd"), dev),
                        "pu_dev": S._op_f64(_section(arrays, f"pg{i}/pu"), dev), "pd": arrays[f"pg{i}/pd"],
                        "pu": arrays[f"pg{i}/pu"]}
        else:
            grp.xs = S._op_f64(_section(arrays, f"pg{i}/xs"), dev)
        solver.parent_groups.append(grp)
    solver.depth = S._depths(tree)
    solver._layout = S._layout(solver)
    if header["mode"] == "econ":
        for grp in solver.leaf_groups:
            grp.fs = grp.h = None
