"""ctypes binding of the C ABI in include/hps_b200.h (the in-tree _hps_b200.so).

There is no fallback: if the library cannot be loaded (or built in-tree with nvcc) every
GPU entry point raises. The structs below mirror include/hps_b200.h field by field.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import build_ext

c_dp = C.POINTER(C.c_double)


class MatBatch(C.Structure):
    _fields_ = [("base", C.c_void_p), ("stride", C.c_longlong), ("ptrs", C.c_void_p),
                ("ld", C.c_int), ("off", C.c_longlong)]


class LeafBatch(C.Structure):
    _fields_ = [("nleaf", C.c_int), ("p", C.c_int), ("q", C.c_int),
                ("coef", C.c_void_p), ("dx", C.c_void_p), ("dy", C.c_void_p),
                ("dxx", C.c_void_p), ("dyy", C.c_void_p), ("int_pos", C.c_void_p),
                ("ext_pos", C.c_void_p), ("lift", C.c_void_p), ("dfi", C.c_void_p),
                ("t0", C.c_void_p), ("fs", C.c_void_p), ("h", C.c_void_p), ("t", C.c_void_p),
                ("anorm", C.c_void_p), ("ainvnorm", C.c_void_p), ("status", C.c_void_p),
                ("perm", C.c_void_p), ("workspace", C.c_void_p)]


class MergeBatch(C.Structure):
    _fields_ = [("npar", C.c_int), ("m3", C.c_int), ("n1", C.c_int), ("n2", C.c_int),
                ("ta", C.c_void_p), ("tb", C.c_void_p), ("lda", C.c_int), ("ldb", C.c_int),
                ("idx", C.c_void_p), ("idx_stride", C.c_longlong), ("xs", C.c_void_p),
                ("tei", C.c_void_p), ("tnew", C.c_void_p), ("dnorm", C.c_void_p),
                ("xnorm", C.c_void_p), ("status", C.c_void_p), ("perm", C.c_void_p),
                ("workspace", C.c_void_p), ("delta", C.c_void_p)]


class GemvBatch(C.Structure):
    _fields_ = [("nitems", C.c_int), ("R", C.c_int), ("K", C.c_int), ("nrhs", C.c_int),
                ("A", MatBatch), ("pool", C.c_void_p), ("xidx", C.c_void_p),
                ("x2idx", C.c_void_p), ("aidx", C.c_void_p), ("oidx", C.c_void_p),
                ("mode2", C.c_int), ("R2", C.c_int), ("K2", C.c_int), ("A2", MatBatch),
                ("a2idx", C.c_void_p), ("o2idx", C.c_void_p), ("kparts", C.c_int),
                ("kscale", C.c_int), ("xscale", C.c_double)]


class LeafApplyArgs(C.Structure):
    _fields_ = [("nleaf", C.c_int), ("p", C.c_int), ("nrhs", C.c_int), ("alpha", C.c_double),
                ("beta", C.c_double), ("coef", C.c_void_p), ("dx", C.c_void_p), ("dy", C.c_void_p),
                ("dxx", C.c_void_p), ("dyy", C.c_void_p), ("u", C.c_void_p), ("u_stride", C.c_longlong),
                ("g", C.c_void_p), ("g_stride", C.c_longlong)]


EXPORTS = ("hps_abi_version", "hps_status_string", "hps_gemm_batched", "hps_gj_workspace_bytes",
           "hps_gj_invert_batched", "hps_leaf_workspace_bytes", "hps_leaf_build",
           "hps_merge_workspace_bytes", "hps_merge_build", "hps_sweep_gemv", "hps_leaf_apply")

ABI_VERSION = 7
_lib = None
_lock = threading.Lock()


class ExtensionError(RuntimeError):
    pass


def lib_path() -> str:
    return build_ext.LIB


def load(build_if_missing: bool = True):
    """Load (building in-tree if needed) the sm_100a extension; raises if unavailable."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("HPS_B200_LIB") or build_ext.LIB  # override: A/B tuning builds only
        if path == build_ext.LIB and (not os.path.exists(path) or not build_ext.up_to_date()):
            if not build_if_missing:
                raise ExtensionError(f"HPS CUDA extension missing: {path}")
            build_ext.build()
        lib = C.CDLL(path)
        lib.hps_abi_version.restype = C.c_int
        lib.hps_status_string.restype = C.c_char_p
        lib.hps_status_string.argtypes = [C.c_int]
        lib.hps_gemm_batched.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                         C.POINTER(MatBatch), C.POINTER(MatBatch), C.c_double,
                                         C.POINTER(MatBatch), C.c_void_p, C.c_int, C.c_void_p]
        lib.hps_gj_workspace_bytes.restype = C.c_longlong
        lib.hps_gj_workspace_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
        lib.hps_gj_invert_batched.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(MatBatch),
                                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p, C.c_void_p]
        lib.hps_leaf_workspace_bytes.restype = C.c_longlong
        lib.hps_leaf_workspace_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
        lib.hps_leaf_build.argtypes = [C.POINTER(LeafBatch), C.c_void_p]
        lib.hps_merge_workspace_bytes.restype = C.c_longlong
        lib.hps_merge_workspace_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
        lib.hps_merge_build.argtypes = [C.POINTER(MergeBatch), C.c_void_p]
        lib.hps_sweep_gemv.argtypes = [C.POINTER(GemvBatch), C.c_void_p]
        lib.hps_leaf_apply.argtypes = [C.POINTER(LeafApplyArgs), C.c_void_p]
        for name in EXPORTS:
            getattr(lib, name)
        if lib.hps_abi_version() != ABI_VERSION:
            raise ExtensionError("HPS extension ABI version mismatch")
        _lib = lib
        return lib


def check(rc: int, what: str):
    if rc != 0:
        msg = load().hps_status_string(rc).decode()
        raise ExtensionError(f"{what} failed: {msg} (status {rc})")


def mat(tensor_or_ptr, stride: int, ld: int, off: int = 0, ptrs=None) -> MatBatch:
    """Build an hps_mat_batch from a torch tensor (or raw pointer) and element strides."""
    base = tensor_or_ptr if isinstance(tensor_or_ptr, int) else tensor_or_ptr.data_ptr()
    return MatBatch(base, stride, 0 if ptrs is None else ptrs.data_ptr(), ld, off)


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


_host = False


def host_module():
    """The optional CPython helper `_hps_host` (threaded gather of body-load mappings), or None."""
    global _host
    if _host is False:
        _host = None
        try:
            path = build_ext.build_host()
            if path:
                import importlib.machinery
                import importlib.util
                loader = importlib.machinery.ExtensionFileLoader("_hps_host", path)
                spec = importlib.util.spec_from_loader("_hps_host", loader)
                mod = importlib.util.module_from_spec(spec)
                loader.exec_module(mod)
                _host = mod
        except Exception:
            _host = None
    return _host

