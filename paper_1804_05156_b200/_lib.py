"""ctypes binding of libfemlite_b200.so (the C-ABI in include/femlite_b200.h).

There is no fallback: if the shared library is missing or no sm_100 device is
present, every entry point raises.  The library is built in-tree by
``paper_1804_05156_b200/build.py`` (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import Error, ErrorCode

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfemlite_b200.so")

# enum fl_mem / fl_field_kind / fl_output / fl_array (femlite_b200.h)
MEM_HOST, MEM_DEVICE = 0, 1
FIELD_NONE, FIELD_CONST, FIELD_SINSIN, FIELD_X, FIELD_XYZ, FIELD_SAMPLES, FIELD_COEF_C5 = 0, 1, 2, 3, 4, 6, 7
OUT_STIFFNESS, OUT_LOAD, OUT_PARTITION, OUT_SYSTEM, REPLAN = 1, 2, 4, 8, 16
(A_COL_PTR, A_ROW_IDX, A_VALUES, B, U0, B_MOD, DIR_NODES, FREE_NODES,
 AFF_COL_PTR, AFF_ROW_IDX, AFF_VALUES, B_F, DIR_FACES, DIR_FACE_ELEM, DIR_FACE_LOCAL,
 NEU_FACES, NEU_FACE_ELEM, NEU_FACE_LOCAL) = range(18)

FL_ERR_ARGUMENT, FL_ERR_CUDA, FL_ERR_NO_DEVICE, FL_ERR_OUT_OF_MEMORY, FL_ERR_UNSUPPORTED = 100, 101, 102, 103, 104

# (symbol, restype, argtypes) -- every symbol declared in include/femlite_b200.h
_vp = C.c_void_p
SIGNATURES = {
    "fl_abi_version": (C.c_int, []),
    "fl_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "fl_destroy": (C.c_int, [_vp]),
    "fl_last_error": (C.c_char_p, []),
    "fl_set_stream": (C.c_int, [_vp, _vp]),
    "fl_synchronize": (C.c_int, [_vp]),
    "fl_mesh_create": (C.c_int, [_vp, C.c_int, C.c_int32, C.c_int32, _vp, _vp, _vp, C.c_int,
                                 C.POINTER(_vp)]),
    "fl_mesh_set_nodes": (C.c_int, [_vp, _vp, _vp, C.c_int]),
    "fl_mesh_set_flags": (C.c_int, [_vp, _vp, _vp, C.c_int]),
    "fl_mesh_set_elems": (C.c_int, [_vp, _vp, _vp, C.c_int]),
    "fl_mesh_validate": (C.c_int, [_vp, _vp]),
    "fl_mesh_plan": (C.c_int, [_vp, _vp]),
    "fl_mesh_set_columns": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32]),
    "fl_result_counts_async": (C.c_int, [_vp, _vp]),
    "fl_boundary_faces": (C.c_int, [_vp, _vp, _vp]),
    "fl_cg_solve": (C.c_int, [_vp, C.c_int32, _vp, _vp, _vp, _vp, C.c_int, _vp, _vp, _vp, _vp, _vp]),
    "fl_solve_system": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int, _vp, _vp]),
    "fl_from_triplets": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int64, _vp, _vp, _vp, C.c_int, _vp]),
    "fl_apply_dirichlet": (C.c_int, [_vp, _vp, C.c_int32, C.c_int32, _vp, _vp, _vp, C.c_int64, _vp, C.c_int,
                                     _vp, _vp]),
    "fl_accumulate": (C.c_int, [_vp, C.c_int64, _vp, _vp, C.c_int32, _vp, C.c_int]),
    "fl_solve_neumann": (C.c_int, [_vp, _vp, _vp, C.c_int32, _vp, _vp, C.c_int, _vp, _vp]),
    "fl_matvec": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp, _vp, C.c_int]),
    "fl_boundary_faces_copy": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int]),
    "fl_mesh_set_boundary_flags": (C.c_int, [_vp, _vp, _vp, C.c_int8, C.c_int]),
    "fl_mesh_destroy": (C.c_int, [_vp]),
    "fl_result_create": (C.c_int, [_vp, C.POINTER(_vp)]),
    "fl_result_destroy": (C.c_int, [_vp]),
    "fl_assemble": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, C.c_uint32, _vp]),
    "fl_result_sizes": (C.c_int, [_vp, _vp]),
    "fl_result_copy": (C.c_int, [_vp, C.c_int, _vp, C.c_int64, C.c_int]),
    "fl_result_device_ptr": (C.c_int, [_vp, C.c_int, C.POINTER(_vp), C.POINTER(C.c_int64)]),
    "fl_submatrix": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, _vp, C.c_int32, _vp,
                               C.c_int32, _vp, C.c_int, _vp]),
    "fl_launch_count": (C.c_int64, [_vp]),
    "fl_last_timings": (C.c_int, [_vp, _vp]),
    "fl_last_kernel_timings": (C.c_int, [_vp, _vp]),
    "fl_selftest_div": (C.c_int, [_vp, C.c_int64, _vp, _vp, _vp, _vp, C.c_int]),
    "fl_phase_cycles": (C.c_int, [_vp, _vp]),
    "fl_host_sample": (C.c_int, [C.c_int, C.c_int32, C.c_int32, _vp, _vp, C.c_int, C.c_int,
                                 C.c_double, _vp]),
    "fl_host_points": (C.c_int, [C.c_int, C.c_int32, C.c_int32, _vp, _vp, C.c_int, _vp]),
    "fl_text_create": (C.c_int, [_vp, C.POINTER(_vp)]),
    "fl_text_destroy": (C.c_int, [_vp]),
    "fl_text_size": (C.c_int, [_vp, C.POINTER(C.c_int64)]),
    "fl_text_copy": (C.c_int, [_vp, _vp, C.c_int64, C.c_int]),
    "fl_text_device_ptr": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(C.c_int64)]),
    "fl_write_matrix_market": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, _vp, C.c_int, _vp]),
    "fl_write_mesh": (C.c_int, [_vp, _vp, _vp]),
    "fl_format_reals": (C.c_int, [_vp, C.c_int64, _vp, C.c_int, C.c_uint32, _vp]),
}


class Field(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mem", C.c_int32), ("value", C.c_double),
                ("samples", _vp), ("n_samples", C.c_int64)]


class CgOptions(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_iter", C.c_int64), ("preconditioner", C.c_int32),
                ("pad", C.c_int32)]


class Sizes(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_dir", C.c_int32), ("n_free", C.c_int32),
                ("n_dir_faces", C.c_int32), ("n_neu_faces", C.c_int32), ("n_free_cols", C.c_int32),
                ("nnz", C.c_int64), ("nnz_ff", C.c_int64)]


_lib = None


def lib():
    """Load libfemlite_b200.so (raises if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise Error(ErrorCode.io_error,
                        f"{LIB_PATH} not built: run __graft_entry__.build() "
                        "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().fl_last_error().decode(errors="replace")


def check(rc: int, what: str = ""):
    """Map an ABI status onto the reference's exception type (error.hpp:28-37)."""
    if rc == 0:
        return
    msg = last_error()
    if 1 <= rc <= 15:
        raise Error(ErrorCode(rc - 1), msg)
    raise Error(None, f"{what}: status {rc}: {msg}", status=rc)
