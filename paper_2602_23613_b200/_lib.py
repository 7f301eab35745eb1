"""ctypes binding of libhcamg (include/hcamg.h).

The shared library is built in-tree (``paper_2602_23613_b200/lib/libhcamg.so``,
see Makefile / ``__graft_entry__.build``).  There is no fallback: if the
library or a CUDA device is missing, every solver entry point raises
:class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libhcamg.so")

OK, EINVAL, ENOTSPD, EBREAKDOWN, ENOMEM, ECUDA, ENOTSYM, EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6, -7

# every symbol declared in include/hcamg.h (checked by tests/test_lib_exports.py)
EXPORTS = [
    "hcamg_create", "hcamg_destroy", "hcamg_last_error", "hcamg_error_index", "hcamg_version",
    "hcamg_setup_alg", "hcamg_setup_ref", "hcamg_hier_begin", "hcamg_hier_push", "hcamg_hier_end",
    "hcamg_hier_end_with", "hcamg_info_get", "hcamg_notes", "hcamg_level", "hcamg_export_csr",
    "hcamg_export_splitting", "hcamg_export_l1", "hcamg_export_patches", "hcamg_export_coarse_cols",
    "hcamg_vcycle", "hcamg_pcg", "hcamg_amg_solve", "hcamg_pcg_device", "hcamg_graph_launches",
    "hcamg_stream", "hcamg_pcg_generic", "hcamg_spmv", "hcamg_profile_vcycle", "hcamg_export_dense", "hcamg_component_solve", "hcamg_kuhn_assemble", "hcamg_kuhn_export", "hcamg_split_alg", "hcamg_split_export",
    "hcamg_dist_prepare", "hcamg_dist_connect", "hcamg_dist_connect_ptrs", "hcamg_dist_disconnect", "hcamg_dist_info",
    "hcamg_set_option", "hcamg_get_option", "hcamg_coarse_solve", "hcamg_solve_status", "hcamg_cholesky_factor",
    "hcamg_smoother_setup", "hcamg_smooth",
    "hcamg_rows_prepare", "hcamg_rows_connect", "hcamg_rows_connect_ptrs", "hcamg_rows_disconnect", "hcamg_rows_info",
    "hcamg_rows_emulate", "hcamg_rows_owner", "hcamg_plan_create", "hcamg_plan_destroy", "hcamg_plan_set_vector",
    "hcamg_plan_invalidate", "hcamg_plan_step", "hcamg_plan_counts", "hcamg_plan_pushes",
]


class NativeUnavailable(RuntimeError):
    """libhcamg.so (or a CUDA device) is not available — there is no CPU path."""


class CSR(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("indptr", C.c_void_p),
                ("indices", C.c_void_p), ("data", C.c_void_p)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int32), ("zero_rhs", C.c_int32),
                ("diverged", C.c_int32), ("pad", C.c_int32), ("final_relres", C.c_double)]


class Info(C.Structure):
    _fields_ = [("depth", C.c_int32), ("stalled", C.c_int32), ("method", C.c_int32), ("pad", C.c_int32),
                ("operator_complexity", C.c_double), ("setup_seconds", C.c_double), ("setup_flops", C.c_double)]


class LevelInfo(C.Structure):
    _fields_ = [(name, C.c_int64) for name in (
        "n", "nnz_A", "ncols_G", "nnz_G", "nnz_P", "n_pairs", "n_interior", "n_coarse_nodes",
        "n_patches", "n_patch_entries", "n_waves", "n_gc_cols", "coarsest", "n_components",
        "max_component", "pad", "factor_bytes", "factor_steps", "factor_tma")]


PRECOND_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64, C.c_void_p)

_lib = None


def load(required=True):
    """Load libhcamg.so once; raise NativeUnavailable when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if required:
            raise NativeUnavailable(f"{LIB_PATH} not built (run __graft_entry__.build())")
        return None
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "hcamg_create": (C.c_int, [C.POINTER(P), C.c_int, P]),
        "hcamg_destroy": (None, [P]),
        "hcamg_last_error": (C.c_char_p, [P]),
        "hcamg_error_index": (C.c_int64, [P]),
        "hcamg_version": (C.c_int, []),
        "hcamg_setup_alg": (C.c_int, [P, C.POINTER(CSR), C.POINTER(CSR), C.c_int32, C.c_int64, C.c_double,
                                      C.POINTER(Info)]),
        "hcamg_setup_ref": (C.c_int, [P, C.POINTER(CSR), C.POINTER(CSR), C.c_int32, P, P, P, P, C.c_int32,
                                      C.c_int64, C.POINTER(Info)]),
        "hcamg_hier_begin": (C.c_int, [P]),
        "hcamg_hier_push": (C.c_int, [P, C.POINTER(CSR), C.POINTER(CSR), C.POINTER(CSR)]),
        "hcamg_hier_end": (C.c_int, [P, C.POINTER(Info)]),
        "hcamg_hier_end_with": (C.c_int, [P, C.POINTER(CSR), C.POINTER(Info)]),
        "hcamg_info_get": (C.c_int, [P, C.POINTER(Info)]),
        "hcamg_notes": (C.c_int, [P, C.c_char_p, C.c_int64]),
        "hcamg_level": (C.c_int, [P, C.c_int32, C.POINTER(LevelInfo)]),
        "hcamg_export_csr": (C.c_int, [P, C.c_int32, C.c_int32, P, P, P]),
        "hcamg_export_splitting": (C.c_int, [P, C.c_int32, P, P, P]),
        "hcamg_export_l1": (C.c_int, [P, C.c_int32, P]),
        "hcamg_export_patches": (C.c_int, [P, C.c_int32, P, P, P]),
        "hcamg_export_coarse_cols": (C.c_int, [P, C.c_int32, P]),
        "hcamg_vcycle": (C.c_int, [P, P, P, P]),
        "hcamg_pcg": (C.c_int, [P, P, P, C.c_double, C.c_int64, P, P, C.POINTER(Report)]),
        "hcamg_amg_solve": (C.c_int, [P, P, P, C.c_double, C.c_int64, P, P, C.POINTER(Report)]),
        "hcamg_pcg_device": (C.c_int, [P, P, P, C.c_double, C.c_int64, P, C.POINTER(Report)]),
        "hcamg_graph_launches": (C.c_int64, [P, C.c_int32]),
        "hcamg_stream": (P, [P]),
        "hcamg_pcg_generic": (C.c_int, [P, C.POINTER(CSR), P, P, C.c_double, C.c_int64, PRECOND_FN, P, P, P,
                                        C.POINTER(Report)]),
        "hcamg_spmv": (C.c_int, [P, C.POINTER(CSR), P, P]),
        "hcamg_profile_vcycle": (C.c_int, [P, C.c_int32, C.c_int32, P, P, P, P, P]),
        "hcamg_export_dense": (C.c_int, [P, C.c_int32, C.c_int32, P]),
        "hcamg_component_solve": (C.c_int, [P, C.c_int32, P, P]),
        "hcamg_kuhn_assemble": (C.c_int, [P, C.c_int64, P, C.c_double, P, P, P]),
        "hcamg_kuhn_export": (C.c_int, [P, P, P, P, P, P, P, P, P]),
        "hcamg_split_alg": (C.c_int, [P, C.POINTER(CSR), C.POINTER(CSR), C.c_double, P]),
        "hcamg_split_export": (C.c_int, [P, P, P, P]),
        "hcamg_dist_prepare": (C.c_int, [P, C.c_int32, C.c_int32, P, C.POINTER(C.c_void_p)]),
        "hcamg_dist_connect": (C.c_int, [P, P]),
        "hcamg_dist_connect_ptrs": (C.c_int, [P, P]),
        "hcamg_dist_disconnect": (C.c_int, [P]),
        "hcamg_dist_info": (C.c_int, [P, P, P, P, P]),
        "hcamg_set_option": (C.c_int, [P, C.c_char_p, C.c_double]),
        "hcamg_get_option": (C.c_int, [P, C.c_char_p, C.POINTER(C.c_double)]),
        "hcamg_coarse_solve": (C.c_int, [P, C.c_int32, P, P]),
        "hcamg_solve_status": (C.c_int, [P, C.POINTER(Report)]),
        "hcamg_cholesky_factor": (C.c_int, [P, C.c_int32, P, P]),
        "hcamg_smoother_setup": (C.c_int, [P, C.POINTER(CSR), C.POINTER(CSR)]),
        "hcamg_smooth": (C.c_int, [P, C.c_int32, C.c_int32, P, P, P]),
        "hcamg_rows_prepare": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int64, P, C.POINTER(C.c_void_p)]),
        "hcamg_rows_connect": (C.c_int, [P, P]),
        "hcamg_rows_connect_ptrs": (C.c_int, [P, P]),
        "hcamg_rows_disconnect": (C.c_int, [P]),
        "hcamg_rows_info": (C.c_int, [P, P, C.c_int32]),
        "hcamg_rows_emulate": (C.c_int, [P, C.c_int32, C.c_int32, P, P, C.c_double, C.c_int64, C.c_int32,
                                         C.POINTER(Report)]),
        "hcamg_rows_owner": (C.c_int, [C.c_int64, P, P, C.c_int32, P]),
        "hcamg_plan_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, P]),
        "hcamg_plan_destroy": (C.c_int, [P]),
        "hcamg_plan_set_vector": (C.c_int, [P, C.c_int32, C.c_int32, P]),
        "hcamg_plan_invalidate": (C.c_int, [P, C.c_int32]),
        "hcamg_plan_step": (C.c_int, [P, P, P, P, P, P, P]),
        "hcamg_plan_counts": (C.c_int, [P, P]),
        "hcamg_plan_pushes": (C.c_int, [P, P, P]),
        # debug entry points (not in the public header)
        "hcamg_debug_dist_piece": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int32, P, P]),
        "hcamg_debug_apply_p": (C.c_int, [P, C.c_int32, C.c_int32, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class HostCSR:
    """Keeps the int64/int32/fp64 copies alive for the duration of a call."""

    def __init__(self, M):
        M = M.tocsr()
        if not M.has_sorted_indices:
            M = M.sorted_indices()
        self.indptr = np.ascontiguousarray(M.indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(M.indices, dtype=np.int32)
        self.data = np.ascontiguousarray(M.data, dtype=np.float64)
        self.view = CSR(M.shape[0], M.shape[1], ptr(self.indptr), ptr(self.indices), ptr(self.data))

    def ref(self):
        return C.byref(self.view)
