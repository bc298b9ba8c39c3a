"""ctypes face of the CHECKERS (test infrastructure only).

Two libraries, same call shapes:

* ``build/libfemlite_oracle.so`` -- the plain-C restatement (femlite_oracle.c);
* ``_ref/libfemlite_ref.so``     -- the unmodified femlite reference compiled from
  /root/reference through ref_shim.cpp (absent if the reference was never
  compiled here; it travels to the GPU box as a prebuilt .so).

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) import this module.  The product package
``paper_1804_05156_b200`` never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libfemlite_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfemlite_ref.so")

# field kinds (shared numbering with oracle/femlite_oracle.h and the product ABI)
FIELD_NONE, FIELD_CONST, FIELD_SINSIN, FIELD_X, FIELD_XYZ, FIELD_CALLBACK, FIELD_SAMPLES = 0, 1, 2, 3, 4, 5, 6
# classifiers (oracle/femlite_oracle.c classify == oracle/ref_shim.cpp make_classifier)
CLS_DIRICHLET, CLS_NEUMANN, CLS_MIXED, CLS_LSHAPE, CLS_NONE, CLS_BOTTOM_NEU, CLS_ZFACE_NEU, CLS_ROBIN = range(8)
SHAPE_SQUARE, SHAPE_CUBE, SHAPE_LSHAPE = 0, 1, 2

_i32p = C.POINTER(C.c_int32)
_f64p = C.POINTER(C.c_double)
_i8p = C.POINTER(C.c_int8)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


@dataclass
class Csc:
    m: int
    n: int
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])


class _fo_csc(C.Structure):
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("nnz", C.c_int32),
                ("col_ptr", _i32p), ("row_idx", _i32p), ("values", _f64p)]


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def _arr_i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _arr_f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _arr_i8(a):
    return np.ascontiguousarray(a, dtype=np.int8)


_libs: dict = {}


def lib(which: str = "oracle"):
    if which not in _libs:
        path = ORACLE_SO if which == "oracle" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        _libs[which] = C.CDLL(path)
    return _libs[which]


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def _take(ptr, n, dtype, free):
    if n == 0:
        out = np.zeros(0, dtype=dtype)
    else:
        out = np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)
    free(ptr)
    return out


def _check(rc, which="oracle"):
    if rc != 0:
        msg = ""
        if which == "ref":
            f = lib("ref").ref_last_error
            f.restype = C.c_char_p
            msg = f().decode()
        raise OracleError(rc, msg)


# ---------------------------------------------------------------------------
# meshes
# ---------------------------------------------------------------------------
def generate_mesh(shape: int, n: int, which: str = "oracle"):
    L = lib(which)
    dim, nn, ne = C.c_int32(), C.c_int32(), C.c_int32()
    nodes, elems = _f64p(), _i32p()
    fn = L.fo_generate_mesh if which == "oracle" else L.ref_generate_mesh
    _check(fn(C.c_int(shape), C.c_int(n), C.byref(dim), C.byref(nn), C.byref(ne),
              C.byref(nodes), C.byref(elems)), which)
    free = L.fo_free if which == "oracle" else L.ref_free
    free.argtypes = [C.c_void_p]
    d = dim.value
    nodes_np = _take(nodes, nn.value * d, np.float64, free).reshape(nn.value, d)
    elems_np = _take(elems, ne.value * (d + 1), np.int32, free).reshape(ne.value, d + 1)
    return d, nodes_np, elems_np


def set_boundary_flags(dim, nodes, elems, classifier: int, which: str = "oracle"):
    L = lib(which)
    nodes, elems = _arr_f64(nodes), _arr_i32(elems)
    nn, ne = nodes.shape[0], elems.shape[0]
    flags = np.zeros((ne, dim + 1), dtype=np.int8)
    fn = L.fo_set_boundary_flags if which == "oracle" else L.ref_set_boundary_flags
    _check(fn(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p), _p(elems, _i32p),
              C.c_int(classifier), _p(flags, _i8p)), which)
    return flags


def validate_mesh(dim, nodes, elems, flags=None, which: str = "oracle") -> int:
    L = lib(which)
    nodes, elems = _arr_f64(nodes), _arr_i32(elems)
    flags = _arr_i8(flags) if flags is not None else None
    fn = L.fo_validate_mesh if which == "oracle" else L.ref_validate_mesh
    return fn(C.c_int(dim), C.c_int32(nodes.shape[0]), C.c_int32(elems.shape[0]),
              _p(nodes, _f64p), _p(elems, _i32p), _p(flags, _i8p))


# ---------------------------------------------------------------------------
# sparse / assembly
# ---------------------------------------------------------------------------
def _csc_from_fo(L, out: _fo_csc) -> Csc:
    L.fo_free.argtypes = [C.c_void_p]
    nnz = out.nnz
    col_ptr = np.ctypeslib.as_array(out.col_ptr, shape=(out.n + 1,)).copy()
    row_idx = np.ctypeslib.as_array(out.row_idx, shape=(max(nnz, 1),))[:nnz].copy()
    values = np.ctypeslib.as_array(out.values, shape=(max(nnz, 1),))[:nnz].copy()
    L.fo_csc_free(C.byref(out))
    return Csc(out.m, out.n, col_ptr, row_idx, values)


def _csc_from_ref(L, m, n, nnz, cp, ri, va) -> Csc:
    L.ref_free.argtypes = [C.c_void_p]
    col_ptr = _take(cp, n + 1, np.int32, L.ref_free)
    row_idx = _take(ri, nnz, np.int32, L.ref_free)
    values = _take(va, nnz, np.float64, L.ref_free)
    return Csc(m, n, col_ptr, row_idx, values)


def assemble_blockwise(dim, nodes, elems, coef=None, which: str = "oracle") -> Csc:
    L = lib(which)
    nodes, elems = _arr_f64(nodes), _arr_i32(elems)
    coef = _arr_f64(coef) if coef is not None else None
    nn, ne = nodes.shape[0], elems.shape[0]
    if which == "oracle":
        out = _fo_csc()
        _check(L.fo_assemble_blockwise(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                                       _p(elems, _i32p), _p(coef, _f64p), C.byref(out)))
        return _csc_from_fo(L, out)
    nnz, cp, ri, va = C.c_int32(), _i32p(), _i32p(), _f64p()
    if coef is None:
        rc = L.ref_assemble(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                            _p(elems, _i32p), C.c_int(2), C.c_int(0), C.byref(nnz), C.byref(cp),
                            C.byref(ri), C.byref(va))
    else:
        rc = L.ref_assemble_blockwise_coef(C.c_int(dim), C.c_int32(nn), C.c_int32(ne),
                                           _p(nodes, _f64p), _p(elems, _i32p), _p(coef, _f64p),
                                           C.byref(nnz), C.byref(cp), C.byref(ri), C.byref(va))
    _check(rc, which)
    return _csc_from_ref(L, nn, nn, nnz.value, cp, ri, va)


def ref_assemble_strategy(dim, nodes, elems, strategy: int, symmetric_fill: bool = False) -> Csc:
    """The reference's assemble(mesh, strategy) (assembly.hpp:302): 0 dense, 1 triplet, 2 blockwise."""
    L = lib("ref")
    nodes, elems = _arr_f64(nodes), _arr_i32(elems)
    nn, ne = nodes.shape[0], elems.shape[0]
    nnz, cp, ri, va = C.c_int32(), _i32p(), _i32p(), _f64p()
    _check(L.ref_assemble(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                          _p(elems, _i32p), C.c_int(strategy), C.c_int(int(symmetric_fill)),
                          C.byref(nnz), C.byref(cp), C.byref(ri), C.byref(va)), "ref")
    return _csc_from_ref(L, nn, nn, nnz.value, cp, ri, va)


def assemble_columns(dim, nodes, elems, cols, coef=None) -> Csc:
    L = lib("oracle")
    nodes, elems, cols = _arr_f64(nodes), _arr_i32(elems), _arr_i32(cols)
    coef = _arr_f64(coef) if coef is not None else None
    out = _fo_csc()
    _check(L.fo_assemble_columns(C.c_int(dim), C.c_int32(nodes.shape[0]), C.c_int32(elems.shape[0]),
                                 _p(nodes, _f64p), _p(elems, _i32p), _p(coef, _f64p),
                                 C.c_int32(cols.shape[0]), _p(cols, _i32p), C.byref(out)))
    return _csc_from_fo(L, out)


def from_triplets(m, n, ii, jj, ss, which: str = "oracle") -> Csc:
    L = lib(which)
    ii, jj, ss = _arr_i32(ii), _arr_i32(jj), _arr_f64(ss)
    cnt = ii.shape[0]
    if which == "oracle":
        out = _fo_csc()
        _check(L.fo_from_triplets(C.c_int32(m), C.c_int32(n), C.c_int64(cnt), _p(ii, _i32p),
                                  _p(jj, _i32p), _p(ss, _f64p), C.byref(out)))
        return _csc_from_fo(L, out)
    nnz, cp, ri, va = C.c_int32(), _i32p(), _i32p(), _f64p()
    _check(L.ref_from_triplets(C.c_int32(m), C.c_int32(n), C.c_int64(cnt), _p(ii, _i32p),
                               _p(jj, _i32p), _p(ss, _f64p), C.byref(nnz), C.byref(cp),
                               C.byref(ri), C.byref(va)), "ref")
    return _csc_from_ref(L, m, n, nnz.value, cp, ri, va)


def _fo_from(a: Csc) -> _fo_csc:
    s = _fo_csc()
    s.m, s.n, s.nnz = a.m, a.n, a.nnz
    s.col_ptr = _p(a.col_ptr, _i32p)
    s.row_idx = _p(a.row_idx, _i32p)
    s.values = _p(a.values, _f64p)
    return s


def submatrix(a: Csc, rows, cols, which: str = "oracle") -> Csc:
    L = lib(which)
    rows, cols = _arr_i32(rows), _arr_i32(cols)
    a = Csc(a.m, a.n, _arr_i32(a.col_ptr), _arr_i32(a.row_idx), _arr_f64(a.values))
    if which == "oracle":
        out = _fo_csc()
        src = _fo_from(a)
        _check(L.fo_submatrix(C.byref(src), C.c_int32(rows.shape[0]), _p(rows, _i32p),
                              C.c_int32(cols.shape[0]), _p(cols, _i32p), C.byref(out)))
        return _csc_from_fo(L, out)
    nnz, cp, ri, va = C.c_int32(), _i32p(), _i32p(), _f64p()
    _check(L.ref_submatrix(C.c_int32(a.m), C.c_int32(a.n), _p(a.col_ptr, _i32p), _p(a.row_idx, _i32p),
                           _p(a.values, _f64p), C.c_int32(rows.shape[0]), _p(rows, _i32p),
                           C.c_int32(cols.shape[0]), _p(cols, _i32p), C.byref(nnz), C.byref(cp),
                           C.byref(ri), C.byref(va)), "ref")
    return _csc_from_ref(L, rows.shape[0], cols.shape[0], nnz.value, cp, ri, va)


def accumulate(idx, vals, size, which: str = "oracle"):
    L = lib(which)
    idx, vals = _arr_i32(idx), _arr_f64(vals)
    out = np.zeros(size, dtype=np.float64)
    fn = L.fo_accumulate if which == "oracle" else L.ref_accumulate
    _check(fn(C.c_int64(idx.shape[0]), _p(idx, _i32p), _p(vals, _f64p), C.c_int32(size),
              _p(out, _f64p)), which)
    return out


def local_stiffness_normals(dim, verts, which: str = "oracle"):
    L = lib(which)
    verts = _arr_f64(verts).ravel()
    meas = C.c_double()
    if which == "oracle":
        out = np.zeros((dim + 1) * (dim + 1), dtype=np.float64)
        _check(L.fo_local_stiffness_normals(C.c_int(dim), _p(verts, _f64p), _p(out, _f64p),
                                            C.byref(meas)))
        return out.reshape(dim + 1, dim + 1), meas.value
    out = np.zeros(16, dtype=np.float64)
    _check(L.ref_local_stiffness(C.c_int(dim), _p(verts, _f64p), C.c_int(1), _p(out, _f64p),
                                 C.byref(meas)), "ref")
    return out[: (dim + 1) ** 2].reshape(dim + 1, dim + 1), meas.value


# ---------------------------------------------------------------------------
# system
# ---------------------------------------------------------------------------
def sample_load_points(dim, nodes, elems, f_kind, f_value=0.0):
    L = lib("oracle")
    nodes, elems = _arr_f64(nodes), _arr_i32(elems)
    ne = elems.shape[0]
    out = np.zeros(ne * (dim + 1), dtype=np.float64)
    _check(L.fo_sample_load_points(C.c_int(dim), C.c_int32(nodes.shape[0]), C.c_int32(ne),
                                   _p(nodes, _f64p), _p(elems, _i32p), C.c_int(f_kind),
                                   C.c_double(f_value), _p(out, _f64p)))
    return out


def assemble_load(dim, nodes, elems, f_kind, f_value=0.0, samples=None, which: str = "oracle"):
    L = lib(which)
    nodes, elems = _arr_f64(nodes), _arr_i32(elems)
    nn, ne = nodes.shape[0], elems.shape[0]
    b = np.zeros(nn, dtype=np.float64)
    if which == "oracle":
        samples = _arr_f64(samples) if samples is not None else None
        _check(L.fo_assemble_load(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                                  _p(elems, _i32p), C.c_int(f_kind), C.c_double(f_value),
                                  _p(samples, _f64p), _p(b, _f64p)))
        return b
    if f_kind == FIELD_SAMPLES:
        raise ValueError("reference takes callables, not samples")
    _check(L.ref_assemble_load(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                               _p(elems, _i32p), C.c_int(f_kind), C.c_double(f_value), None, None,
                               _p(b, _f64p)), "ref")
    return b


def partition_boundary(dim, nodes, elems, flags, which: str = "oracle"):
    L = lib(which)
    nodes, elems, flags = _arr_f64(nodes), _arr_i32(elems), _arr_i8(flags)
    nn, ne = nodes.shape[0], elems.shape[0]
    nd, nf, ndf, nnf = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    dn, fn_ = _i32p(), _i32p()
    if which == "oracle":
        _check(L.fo_partition_boundary(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(elems, _i32p),
                                       _p(flags, _i8p), C.byref(nd), C.byref(dn), C.byref(nf),
                                       C.byref(fn_), C.byref(ndf), C.byref(nnf)))
        free = L.fo_free
    else:
        _check(L.ref_partition_boundary(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                                        _p(elems, _i32p), _p(flags, _i8p), C.byref(nd), C.byref(dn),
                                        C.byref(nf), C.byref(fn_), C.byref(ndf), C.byref(nnf)), "ref")
        free = L.ref_free
    free.argtypes = [C.c_void_p]
    return (_take(dn, nd.value, np.int32, free), _take(fn_, nf.value, np.int32, free),
            ndf.value, nnf.value)


def boundary_faces(dim, nodes, elems, flags, value: int, which: str = "oracle"):
    """boundary_faces(mesh, value) (mesh.hpp:222-246) -> (faces [n, dim], parent_elem, local_face)."""
    L = lib(which)
    nodes, elems, flags = _arr_f64(nodes), _arr_i32(elems), _arr_i8(flags)
    nn, ne = nodes.shape[0], elems.shape[0]
    n = C.c_int32()
    fa, pa, la = _i32p(), _i32p(), _i32p()
    if which == "oracle":
        _check(L.fo_boundary_faces(C.c_int(dim), C.c_int32(ne), _p(elems, _i32p), _p(flags, _i8p),
                                   C.c_int(value), C.byref(n), C.byref(fa), C.byref(pa), C.byref(la)))
        free = L.fo_free
    else:
        _check(L.ref_boundary_faces(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                                    _p(elems, _i32p), _p(flags, _i8p), C.c_int(value), C.byref(n),
                                    C.byref(fa), C.byref(pa), C.byref(la)), "ref")
        free = L.ref_free
    free.argtypes = [C.c_void_p]
    k = n.value
    return (_take(fa, k * dim, np.int32, free).reshape(k, dim), _take(pa, k, np.int32, free),
            _take(la, k, np.int32, free))


def apply_dirichlet(dim, nodes, elems, flags, a: Csc, b, g_kind, g_value=0.0, g_samples=None,
                    which: str = "oracle"):
    L = lib(which)
    nodes, elems, flags, b = _arr_f64(nodes), _arr_i32(elems), _arr_i8(flags), _arr_f64(b)
    a = Csc(a.m, a.n, _arr_i32(a.col_ptr), _arr_i32(a.row_idx), _arr_f64(a.values))
    nn, ne = nodes.shape[0], elems.shape[0]
    u0 = np.zeros(nn, dtype=np.float64)
    bo = np.zeros(nn, dtype=np.float64)
    if which == "oracle":
        src = _fo_from(a)
        g_samples = _arr_f64(g_samples) if g_samples is not None else None
        _check(L.fo_apply_dirichlet(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                                    _p(elems, _i32p), _p(flags, _i8p), C.byref(src), _p(b, _f64p),
                                    C.c_int(g_kind), C.c_double(g_value), _p(g_samples, _f64p),
                                    _p(u0, _f64p), _p(bo, _f64p)))
    else:
        _check(L.ref_apply_dirichlet(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                                     _p(elems, _i32p), _p(flags, _i8p), _p(a.col_ptr, _i32p),
                                     _p(a.row_idx, _i32p), _p(a.values, _f64p), _p(b, _f64p),
                                     C.c_int(g_kind), C.c_double(g_value), None, None,
                                     _p(u0, _f64p), _p(bo, _f64p)), "ref")
    return u0, bo


def apply_neumann(dim, nodes, elems, flags, b, g_kind, g_value=0.0, which: str = "oracle"):
    L = lib(which)
    nodes, elems, flags = _arr_f64(nodes), _arr_i32(elems), _arr_i8(flags)
    out = _arr_f64(b).copy()
    nn, ne = nodes.shape[0], elems.shape[0]
    if which == "oracle":
        _check(L.fo_apply_neumann(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                                  _p(elems, _i32p), _p(flags, _i8p), C.c_int(g_kind),
                                  C.c_double(g_value), _p(out, _f64p)))
    else:
        _check(L.ref_apply_neumann(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                                   _p(elems, _i32p), _p(flags, _i8p), C.c_int(g_kind),
                                   C.c_double(g_value), None, None, _p(out, _f64p)), "ref")
    return out


def coefficient_c5(dim, nodes, elems):
    L = lib("oracle")
    nodes, elems = _arr_f64(nodes), _arr_i32(elems)
    out = np.zeros(elems.shape[0], dtype=np.float64)
    _check(L.fo_coefficient_c5(C.c_int(dim), C.c_int32(elems.shape[0]), _p(nodes, _f64p),
                               _p(elems, _i32p), _p(out, _f64p)))
    return out


def ref_time_system(dim, nodes, elems, flags, f_kind, f_value=0.0, coef=None, reps=1):
    """Time the reference's own solve_poisson pre-solve path (ref_shim.cpp ref_time_system)."""
    L = lib("ref")
    nodes, elems, flags = _arr_f64(nodes), _arr_i32(elems), _arr_i8(flags)
    coef = _arr_f64(coef) if coef is not None else None
    secs = np.zeros(reps, dtype=np.float64)
    nnz, nnz_ff = C.c_int64(), C.c_int64()
    _check(L.ref_time_system(C.c_int(dim), C.c_int32(nodes.shape[0]), C.c_int32(elems.shape[0]),
                             _p(nodes, _f64p), _p(elems, _i32p), _p(flags, _i8p), C.c_int(f_kind),
                             C.c_double(f_value), _p(coef, _f64p), C.c_int(reps), _p(secs, _f64p),
                             C.byref(nnz), C.byref(nnz_ff)), "ref")
    return secs, nnz.value, nnz_ff.value


def ref_time_system_mt(dim, nodes, elems, flags, f_kind, f_value=0.0, coef=None, reps=1, threads=1):
    """The reference pipeline on `threads` host threads concurrently (throughput);
    per-round wall seconds (ref_shim.cpp ref_time_system_mt)."""
    L = lib("ref")
    nodes, elems, flags = _arr_f64(nodes), _arr_i32(elems), _arr_i8(flags)
    coef = _arr_f64(coef) if coef is not None else None
    secs = np.zeros(reps, dtype=np.float64)
    _check(L.ref_time_system_mt(C.c_int(dim), C.c_int32(nodes.shape[0]), C.c_int32(elems.shape[0]),
                                _p(nodes, _f64p), _p(elems, _i32p), _p(flags, _i8p), C.c_int(f_kind),
                                C.c_double(f_value), _p(coef, _f64p), C.c_int(reps), C.c_int(threads),
                                _p(secs, _f64p)), "ref")
    return secs


def ref_matvec(a: Csc, x):
    """The reference's matvec (sparse.hpp:129-141)."""
    L = lib("ref")
    x = _arr_f64(x)
    y = np.zeros(a.m, dtype=np.float64)
    _check(L.ref_matvec(C.c_int32(a.m), C.c_int32(a.n), _p(_arr_i32(a.col_ptr), _i32p),
                        _p(_arr_i32(a.row_idx), _i32p), _p(_arr_f64(a.values), _f64p), _p(x, _f64p),
                        _p(y, _f64p)), "ref")
    return y


def ref_cg_solve(a: Csc, b, rel_tol=1e-10, max_iter=0, precond=2):
    """The reference's cg_solve (solver.hpp:63-136): (x, iterations, relres, converged)."""
    L = lib("ref")
    b = _arr_f64(b)
    x = np.zeros(a.n, dtype=np.float64)
    it, rr, cv = C.c_int64(), C.c_double(), C.c_int32()
    cp, ri, va = _arr_i32(a.col_ptr), _arr_i32(a.row_idx), _arr_f64(a.values)
    _check(L.ref_cg_solve(C.c_int32(a.n), _p(cp, _i32p), _p(ri, _i32p), _p(va, _f64p), _p(b, _f64p),
                          C.c_double(rel_tol), C.c_int64(max_iter), C.c_int(precond), _p(x, _f64p),
                          C.byref(it), C.byref(rr), C.byref(cv)), "ref")
    return x, it.value, rr.value, bool(cv.value)


def ref_solve_poisson(dim, nodes, elems, flags, f_kind, f_value, g_kind, g_value, rel_tol=1e-10):
    """The reference's solve_poisson on a Dirichlet mesh: (u, iterations, relres, seconds)."""
    L = lib("ref")
    nodes, elems, flags = _arr_f64(nodes), _arr_i32(elems), _arr_i8(flags)
    u = np.zeros(nodes.shape[0], dtype=np.float64)
    it, rr, sec = C.c_int64(), C.c_double(), C.c_double()
    _check(L.ref_solve_poisson(C.c_int(dim), C.c_int32(nodes.shape[0]), C.c_int32(elems.shape[0]),
                               _p(nodes, _f64p), _p(elems, _i32p), _p(flags, _i8p), C.c_int(f_kind),
                               C.c_double(f_value), C.c_int(g_kind), C.c_double(g_value),
                               C.c_double(rel_tol), _p(u, _f64p), C.byref(it), C.byref(rr),
                               C.byref(sec)), "ref")
    return u, it.value, rr.value, sec.value


# ---------------------------------------------------------------------------
# text writers
# ---------------------------------------------------------------------------
def _take_text(L, ptr, n, free) -> bytes:
    free.argtypes = [C.c_void_p]
    data = C.string_at(ptr, n) if n else b""
    free(ptr)
    return data


def write_matrix_market(a: Csc, which: str = "oracle", timing: bool = False):
    """matrix_market.hpp:15-24 -> bytes (timing=True: (bytes, seconds), ref only)."""
    L = lib(which)
    txt, n = C.c_void_p(), C.c_int64()
    if which == "oracle":
        s = _fo_from(a)
        _check(L.fo_write_matrix_market(C.byref(s), C.byref(txt), C.byref(n)))
        out = _take_text(L, txt, n.value, L.fo_free)
        return (out, float("nan")) if timing else out
    a_cp, a_ri, a_va = _arr_i32(a.col_ptr), _arr_i32(a.row_idx), _arr_f64(a.values)
    sec = C.c_double()
    _check(L.ref_write_matrix_market(C.c_int32(a.m), C.c_int32(a.n), _p(a_cp, _i32p), _p(a_ri, _i32p),
                                     _p(a_va, _f64p), C.byref(txt), C.byref(n), C.byref(sec)), "ref")
    out = _take_text(L, txt, n.value, L.ref_free)
    return (out, sec.value) if timing else out


def write_mesh(dim, nodes, elems, flags=None, which: str = "oracle", timing: bool = False):
    """mesh_io.hpp:125-142 -> bytes (timing=True: (bytes, seconds), ref only)."""
    L = lib(which)
    nodes, elems = _arr_f64(nodes), _arr_i32(elems)
    fl = _arr_i8(flags) if flags is not None else None
    nn, ne = nodes.shape[0], elems.shape[0]
    txt, n = C.c_void_p(), C.c_int64()
    if which == "oracle":
        _check(L.fo_write_mesh(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p),
                               _p(elems, _i32p), _p(fl, _i8p), C.byref(txt), C.byref(n)))
        out = _take_text(L, txt, n.value, L.fo_free)
        return (out, float("nan")) if timing else out
    sec = C.c_double()
    _check(L.ref_write_mesh(C.c_int(dim), C.c_int32(nn), C.c_int32(ne), _p(nodes, _f64p), _p(elems, _i32p),
                            _p(fl, _i8p), C.byref(txt), C.byref(n), C.byref(sec)), "ref")
    out = _take_text(L, txt, n.value, L.ref_free)
    return (out, sec.value) if timing else out
