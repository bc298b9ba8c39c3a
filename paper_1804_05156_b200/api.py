"""The reference's hot-path API, running on the B200 path.

Names, argument meaning and error behaviour follow femlite
(/root/reference/proj/include/femlite/): assemble_blockwise / assemble
(assembly.hpp:261,302), assemble_load (system.hpp:71), partition_boundary
(system.hpp:50), apply_neumann (system.hpp:123), apply_dirichlet
(system.hpp:182), submatrix (sparse.hpp:159), plus ``assemble_system`` -- the
fused pre-solve sequence of solve_poisson (solver.hpp:226-242) in one pass.

Every function calls libfemlite_b200.so; there is no host fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import sys
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .context import Context
from .errors import Error, ErrorCode
from .mesh import TET_FACES, TRI_FACES, Mesh

# quadrature.hpp:65-71
TET4_A = 0.58541019662496845
TET4_B = 0.13819660112501051


class AssemblyStrategy(enum.IntEnum):  # assembly.hpp:41 + the GPU tag
    dense_oracle = 0
    triplet_loop = 1
    blockwise = 2
    b200 = 3


@dataclass
class CscMatrix:  # sparse.hpp:50-59
    m: int
    n: int
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray

    def nnz(self) -> int:
        return int(self.values.shape[0])

    def __eq__(self, other) -> bool:  # bitwise, like `bool operator==` = default
        return (self.m == other.m and self.n == other.n
                and np.array_equal(self.col_ptr, other.col_ptr)
                and np.array_equal(self.row_idx, other.row_idx)
                and self.values.tobytes() == other.values.tobytes())


@dataclass
class FaceList:  # mesh.hpp:101-109
    dim: int
    faces: np.ndarray        # [M, dim] vertices in kTriFaces / kTetFaces order
    parent_elem: np.ndarray  # [M]
    local_face: np.ndarray   # [M]

    def size(self) -> int:
        return int(self.parent_elem.shape[0])

    def __eq__(self, other) -> bool:
        return (self.dim == other.dim and np.array_equal(self.faces, other.faces)
                and np.array_equal(self.parent_elem, other.parent_elem)
                and np.array_equal(self.local_face, other.local_face))


@dataclass
class BoundaryPartition:  # system.hpp:39-44
    dirichlet_nodes: np.ndarray
    free_nodes: np.ndarray
    dirichlet_faces: FaceList
    neumann_faces: FaceList

    @property
    def n_dirichlet_faces(self) -> int:
        return self.dirichlet_faces.size()

    @property
    def n_neumann_faces(self) -> int:
        return self.neumann_faces.size()


@dataclass
class DirichletSystem:  # system.hpp:174-178
    u0: np.ndarray
    b: np.ndarray
    partition: BoundaryPartition


@dataclass
class PoissonSystem:
    """Everything solve_poisson builds before the solve (solver.hpp:226-242)."""
    a: CscMatrix
    b: np.ndarray
    u0: np.ndarray
    b_mod: np.ndarray
    partition: BoundaryPartition
    a_ff: CscMatrix
    b_f: np.ndarray


# ---------------------------------------------------------------------------
# fields
# ---------------------------------------------------------------------------
_NAMED = {"sinsin": _lib.FIELD_SINSIN, "x": _lib.FIELD_X, "xyz": _lib.FIELD_XYZ,
          "coef_c5": _lib.FIELD_COEF_C5}


def _load_points(mesh: Mesh):
    """Cartesian points of the load rule, with the reference's formulas:
    2-D edge midpoints (system.hpp:86-90), 3-D tet4 points (system.hpp:103-107)."""
    X = mesh.nodes[mesh.elems]  # [NT, d+1, d]
    if mesh.dim == 2:
        a, b = TRI_FACES[:, 0], TRI_FACES[:, 1]
        mid = (X[:, a, :] + X[:, b, :]) / 2.0
        return mid[..., 0], mid[..., 1], np.zeros(mid.shape[:2])
    pts = np.zeros((X.shape[0], 4, 3))
    for q in range(4):
        for k in range(4):
            lam = TET4_A if k == q else TET4_B
            pts[:, q, :] = pts[:, q, :] + lam * X[:, k, :]
    return pts[..., 0], pts[..., 1], pts[..., 2]


def _face_points(mesh: Mesh):
    """Neumann rule points per (t, lf): 2-D midpoint, 3-D barycentre (system.hpp:143,160)."""
    table = TRI_FACES if mesh.dim == 2 else TET_FACES
    X = mesh.nodes[mesh.elems[:, table]]  # [NT, d+1, d, d]
    if mesh.dim == 2:
        m = (X[:, :, 0, :] + X[:, :, 1, :]) / 2.0
        return m[..., 0], m[..., 1], np.zeros(m.shape[:2])
    b = (X[:, :, 0, :] + X[:, :, 1, :] + X[:, :, 2, :]) / 3.0
    return b[..., 0], b[..., 1], b[..., 2]


def _field_struct(spec, mesh: Mesh, role: str):
    """-> (fl_field, keepalive).  role: load | coef | dirichlet | neumann."""
    f = _lib.Field()
    keep = None
    if spec is None:
        f.kind = _lib.FIELD_NONE
    elif isinstance(spec, (int, float)) and not isinstance(spec, bool):
        f.kind, f.value = _lib.FIELD_CONST, float(spec)
    elif isinstance(spec, str):
        if spec not in _NAMED:
            raise Error(ErrorCode.invalid_parameter, f"unknown field '{spec}'")
        f.kind = _NAMED[spec]
    else:
        if callable(spec) and not isinstance(spec, np.ndarray):
            # a host callable (the reference's std::function): sample it at the
            # rule's points with the reference's point formulas
            if role == "load":
                x, y, z = _load_points(mesh)
            elif role == "neumann":
                x, y, z = _face_points(mesh)
            elif role == "dirichlet":
                n = mesh.nodes
                x, y = n[:, 0], n[:, 1]
                z = n[:, 2] if mesh.dim == 3 else np.zeros(n.shape[0])
            else:
                raise Error(ErrorCode.invalid_parameter, "coefficient must be samples or a kind")
            spec = np.broadcast_to(np.asarray(spec(x, y, z), dtype=np.float64), x.shape)
        arr = np.ascontiguousarray(np.asarray(spec, dtype=np.float64).ravel())
        keep = arr
        f.kind, f.mem = _lib.FIELD_SAMPLES, _lib.MEM_HOST
        f.samples = arr.ctypes.data if arr.size else None
        f.n_samples = arr.size
    return f, keep


# ---------------------------------------------------------------------------
# results
# ---------------------------------------------------------------------------
class AssemblyResult:
    """An ``fl_result``: device outputs of one fl_assemble call (reusable)."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        self._h = C.c_void_p()
        _lib.check(_lib.lib().fl_result_create(ctx.handle, C.byref(self._h)), "fl_result_create")

    @property
    def handle(self):
        return self._h

    def sizes(self) -> _lib.Sizes:
        s = _lib.Sizes()
        _lib.check(_lib.lib().fl_result_sizes(self._h, C.byref(s)), "fl_result_sizes")
        return s

    def array(self, which: int, dtype, count: int) -> np.ndarray:
        out = np.empty(count, dtype=dtype)
        _lib.check(_lib.lib().fl_result_copy(self._h, which, out.ctypes.data if count else None,
                                             out.nbytes, _lib.MEM_HOST), "fl_result_copy")
        return out

    def device_ptr(self, which: int):
        p, nb = C.c_void_p(), C.c_int64()
        _lib.check(_lib.lib().fl_result_device_ptr(self._h, which, C.byref(p), C.byref(nb)),
                   "fl_result_device_ptr")
        return p.value, nb.value

    # typed views
    def matrix(self) -> CscMatrix:
        """A, or this shard's columns of A (rows stay global: m = all nodes)."""
        s = self.sizes()
        m = getattr(self, "_rows", s.n)
        return CscMatrix(m, s.n, self.array(_lib.A_COL_PTR, np.int32, s.n + 1),
                         self.array(_lib.A_ROW_IDX, np.int32, s.nnz),
                         self.array(_lib.A_VALUES, np.float64, s.nnz))

    def matrix_ff(self) -> CscMatrix:
        s = self.sizes()
        return CscMatrix(s.n_free, s.n_free_cols,
                         self.array(_lib.AFF_COL_PTR, np.int32, s.n_free_cols + 1),
                         self.array(_lib.AFF_ROW_IDX, np.int32, s.nnz_ff),
                         self.array(_lib.AFF_VALUES, np.float64, s.nnz_ff))

    def vector(self, which: int) -> np.ndarray:
        s = self.sizes()
        n = s.n_free_cols if which == _lib.B_F else s.n
        return self.array(which, np.float64, n)

    def face_list(self, dirichlet: bool) -> FaceList:
        """boundary_faces(mesh, 1 | 2) as produced on the GPU (mesh.hpp:222-246)."""
        s = self.sizes()
        d = getattr(self, "_dim", 2)
        n = s.n_dir_faces if dirichlet else s.n_neu_faces
        w = (_lib.DIR_FACES, _lib.DIR_FACE_ELEM, _lib.DIR_FACE_LOCAL) if dirichlet else \
            (_lib.NEU_FACES, _lib.NEU_FACE_ELEM, _lib.NEU_FACE_LOCAL)
        return FaceList(d, self.array(w[0], np.int32, n * d).reshape(n, d),
                        self.array(w[1], np.int32, n), self.array(w[2], np.int32, n))

    def partition(self) -> BoundaryPartition:
        s = self.sizes()
        return BoundaryPartition(self.array(_lib.DIR_NODES, np.int32, s.n_dir),
                                 self.array(_lib.FREE_NODES, np.int32, s.n_free),
                                 self.face_list(True), self.face_list(False))

    def __del__(self):
        if sys.is_finalizing():  # the CUDA runtime may already be gone; the OS reclaims
            return
        try:
            if self._h:
                _lib.lib().fl_result_destroy(self._h)
        except Exception:
            pass


def run(mesh: Mesh, what: int, f=None, coef=None, g_dirichlet=None, g_neumann=None,
        ctx: Optional[Context] = None, result: Optional[AssemblyResult] = None,
        device_mesh=None) -> AssemblyResult:
    """One fl_assemble call (asynchronous; sizes() synchronises).  ``device_mesh``
    overrides the mesh's cached device copy (e.g. one restricted to a column range)."""
    ctx = ctx or Context.default()
    dm = device_mesh or mesh.device(ctx)
    res = result or AssemblyResult(ctx)
    ff, k1 = _field_struct(f, mesh, "load")
    fc, k2 = _field_struct(coef, mesh, "coef")
    fd, k3 = _field_struct(g_dirichlet, mesh, "dirichlet")
    fn, k4 = _field_struct(g_neumann, mesh, "neumann")
    _lib.check(_lib.lib().fl_assemble(ctx.handle, dm.handle, C.byref(ff), C.byref(fc), C.byref(fd),
                                      C.byref(fn), what, res.handle), "fl_assemble")
    res._keep = (k1, k2, k3, k4)
    res._rows = mesh.num_nodes()
    res._dim = mesh.dim
    res._what = what
    return res


# ---------------------------------------------------------------------------
# the reference's functions
# ---------------------------------------------------------------------------
def assemble_blockwise(mesh: Mesh, symmetric_fill: bool = False, coef=None,
                       ctx: Optional[Context] = None) -> CscMatrix:
    """assembly.hpp:261.  ``symmetric_fill`` only changes the reference's triplet
    multiset; the GPU path always produces the default result."""
    if symmetric_fill:
        raise Error(ErrorCode.invalid_parameter,
                    "symmetric_fill changes the triplet multiset; only the default is provided")
    return run(mesh, _lib.OUT_STIFFNESS, coef=coef, ctx=ctx).matrix()


def assemble(mesh: Mesh, strategy=AssemblyStrategy.b200, ctx: Optional[Context] = None) -> CscMatrix:
    """assembly.hpp:302: the blockwise strategy (and the b200 tag) run on the GPU;
    the dense/triplet cross-check oracles stay in the reference."""
    strategy = AssemblyStrategy(strategy)
    if strategy in (AssemblyStrategy.blockwise, AssemblyStrategy.b200):
        return assemble_blockwise(mesh, ctx=ctx)
    raise Error(ErrorCode.invalid_parameter,
                f"strategy {strategy.name} is a CPU cross-check oracle of the reference")


def assemble_load(mesh: Mesh, f, ctx: Optional[Context] = None) -> np.ndarray:
    """system.hpp:71.  f: None | float | 'sinsin' | 'x' | 'xyz' | samples | callable(x, y, z)."""
    return run(mesh, _lib.OUT_LOAD, f=f, ctx=ctx).vector(_lib.B)


def partition_boundary(mesh: Mesh, ctx: Optional[Context] = None) -> BoundaryPartition:
    """system.hpp:50 (raises unsupported_boundary_type on Robin flags)."""
    return run(mesh, _lib.OUT_PARTITION, ctx=ctx).partition()


def apply_neumann(b, mesh: Mesh, g, ctx: Optional[Context] = None) -> np.ndarray:
    """system.hpp:123: b + (Neumann face integrals), computed on the GPU."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape[0] != mesh.num_nodes():
        raise Error(ErrorCode.shape_mismatch, "apply_neumann: vector length mismatch")
    if g is None or not np.any(mesh.bd_flags == 2):
        return b.copy()
    add = run(mesh, _lib.OUT_LOAD, f=None, g_neumann=g, ctx=ctx).vector(_lib.B)
    return b + add


def assemble_system(mesh: Mesh, f, g_dirichlet, g_neumann=None, coef=None,
                    ctx: Optional[Context] = None, result: Optional[AssemblyResult] = None
                    ) -> AssemblyResult:
    """solve_poisson's pre-solve path (solver.hpp:226-242) fused into one pass:
    partition_boundary, assemble_blockwise, assemble_load, apply_neumann,
    apply_dirichlet, submatrix(A, free, free) and b_f.  Device-resident result."""
    return run(mesh, _lib.OUT_SYSTEM, f=f, coef=coef, g_dirichlet=g_dirichlet,
               g_neumann=g_neumann, ctx=ctx, result=result)


def poisson_system(mesh: Mesh, f, g_dirichlet, g_neumann=None, coef=None,
                   ctx: Optional[Context] = None) -> PoissonSystem:
    r = assemble_system(mesh, f, g_dirichlet, g_neumann, coef, ctx)
    return PoissonSystem(r.matrix(), r.vector(_lib.B), r.vector(_lib.U0), r.vector(_lib.B_MOD),
                         r.partition(), r.matrix_ff(), r.vector(_lib.B_F))


def apply_dirichlet(a: CscMatrix, b, mesh: Mesh, g, ctx: Optional[Context] = None) -> DirichletSystem:
    """system.hpp:182-201 for any A and b: partition_boundary(mesh), u0 = g at the
    Dirichlet nodes, b - A u0 with A u0 summed in matvec's column order
    (sparse.hpp:129-141) -- on the GPU, bitwise.  g: float | 'x' | 'xyz' |
    'sinsin' | node samples | callable(x, y, z)."""
    ctx = ctx or Context.default()
    b = np.ascontiguousarray(b, dtype=np.float64)
    cp = np.ascontiguousarray(a.col_ptr, dtype=np.int32)
    ri = np.ascontiguousarray(a.row_idx, dtype=np.int32)
    va = np.ascontiguousarray(a.values, dtype=np.float64)
    fd, keep = _field_struct(g, mesh, "dirichlet")
    res = AssemblyResult(ctx)
    _lib.check(_lib.lib().fl_apply_dirichlet(ctx.handle, mesh.device(ctx).handle, int(a.m), int(a.n),
                                             cp.ctypes.data, ri.ctypes.data, va.ctypes.data, int(b.shape[0]),
                                             b.ctypes.data, _lib.MEM_HOST, C.byref(fd), res.handle),
               "fl_apply_dirichlet")
    res._rows = mesh.num_nodes()
    res._dim = mesh.dim
    return DirichletSystem(res.vector(_lib.U0), res.vector(_lib.B_MOD), res.partition())


def accumulate(idx, vals, size: int, ctx: Optional[Context] = None) -> np.ndarray:
    """sparse.hpp:186-198: out[k] = 0.0 + the vals with idx == k in their order (GPU, bitwise)."""
    ctx = ctx or Context.default()
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    if idx.shape != vals.shape:
        raise Error(ErrorCode.shape_mismatch, "accumulate: index/value lengths differ")
    out = np.zeros(max(int(size), 0), dtype=np.float64)
    _lib.check(_lib.lib().fl_accumulate(ctx.handle, int(idx.size), idx.ctypes.data if idx.size else None,
                                        vals.ctypes.data if vals.size else None, int(size),
                                        out.ctypes.data if out.size else None, _lib.MEM_HOST), "fl_accumulate")
    return out


def submatrix(a: CscMatrix, rows, cols, ctx: Optional[Context] = None) -> CscMatrix:
    """sparse.hpp:159: A(rows, cols) for strictly increasing index sets (GPU)."""
    ctx = ctx or Context.default()
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    cp = np.ascontiguousarray(a.col_ptr, dtype=np.int32)
    ri = np.ascontiguousarray(a.row_idx, dtype=np.int32)
    va = np.ascontiguousarray(a.values, dtype=np.float64)
    res = AssemblyResult(ctx)
    _lib.check(_lib.lib().fl_submatrix(ctx.handle, a.m, a.n, cp.ctypes.data, ri.ctypes.data,
                                       va.ctypes.data, rows.size, rows.ctypes.data, cols.size,
                                       cols.ctypes.data, _lib.MEM_HOST, res.handle), "fl_submatrix")
    s = res.sizes()
    return CscMatrix(int(rows.size), int(cols.size),
                     res.array(_lib.A_COL_PTR, np.int32, cols.size + 1),
                     res.array(_lib.A_ROW_IDX, np.int32, s.nnz),
                     res.array(_lib.A_VALUES, np.float64, s.nnz))


# ---------------------------------------------------------------------------
# the solve after the path
# ---------------------------------------------------------------------------
_PRECOND = {"none": 0, "jacobi": 1, "auto": 2, "auto_select": 2}


@dataclass
class CgResult:  # solver.hpp:34-39
    x: np.ndarray
    iterations: int
    relres: float
    converged: bool


@dataclass
class Solution:  # solver.hpp:179-184
    u: np.ndarray
    iterations: int
    final_relres: float
    partition: BoundaryPartition


def _cg_options(rel_tol, max_iter, preconditioner):
    o = _lib.CgOptions()
    o.rel_tol, o.max_iter = float(rel_tol), int(max_iter)
    o.preconditioner = _PRECOND[preconditioner] if isinstance(preconditioner, str) else int(preconditioner)
    return o


def matvec(a: CscMatrix, x, ctx: Optional[Context] = None) -> np.ndarray:
    """sparse.hpp:129: y = A x on the GPU, bitwise the reference's order."""
    ctx = ctx or Context.default()
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape[0] != a.n:
        raise Error(ErrorCode.shape_mismatch, "matvec: vector length mismatch")
    y = np.empty(a.m, dtype=np.float64)
    cp = np.ascontiguousarray(a.col_ptr, dtype=np.int32)
    ri = np.ascontiguousarray(a.row_idx, dtype=np.int32)
    va = np.ascontiguousarray(a.values, dtype=np.float64)
    _lib.check(_lib.lib().fl_matvec(ctx.handle, a.m, a.n, cp.ctypes.data, ri.ctypes.data, va.ctypes.data,
                                    x.ctypes.data, y.ctypes.data, _lib.MEM_HOST), "fl_matvec")
    return y


def cg_solve(a: CscMatrix, b, rel_tol: float = 1e-10, max_iter: int = 0, preconditioner="auto",
             ctx: Optional[Context] = None) -> CgResult:
    """solver.hpp:63: preconditioned CG on the GPU (x0 = 0; best iterate on the cap)."""
    ctx = ctx or Context.default()
    if a.m != a.n:
        raise Error(ErrorCode.shape_mismatch, "cg_solve: matrix not square")
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.shape[0] != a.n:
        raise Error(ErrorCode.shape_mismatch, "cg_solve: vector length mismatch")
    x = np.empty(a.n, dtype=np.float64)
    it, rr, cv = C.c_int64(), C.c_double(), C.c_int32()
    cp = np.ascontiguousarray(a.col_ptr, dtype=np.int32)
    ri = np.ascontiguousarray(a.row_idx, dtype=np.int32)
    va = np.ascontiguousarray(a.values, dtype=np.float64)
    o = _cg_options(rel_tol, max_iter, preconditioner)
    _lib.check(_lib.lib().fl_cg_solve(ctx.handle, a.n, cp.ctypes.data, ri.ctypes.data, va.ctypes.data,
                                      b.ctypes.data, _lib.MEM_HOST, C.byref(o), x.ctypes.data,
                                      C.byref(it), C.byref(rr), C.byref(cv)), "fl_cg_solve")
    return CgResult(x, it.value, rr.value, bool(cv.value))


def solve_poisson(mesh: Mesh, f, g_dirichlet, g_neumann=None, coef=None, rel_tol: float = 1e-10,
                  max_iter: int = 0, preconditioner="auto", pin_node: int = 0,
                  ctx: Optional[Context] = None) -> Solution:
    """solver.hpp:223-276, device-resident from the assembly through the CG solve
    to the nodal vector: with Dirichlet faces the free-node system (lift, A_ff,
    b_f); without them the pure-Neumann path (compatibility, pinned node,
    zero-average shift)."""
    ctx = ctx or Context.default()
    o = _cg_options(rel_tol, max_iter, preconditioner)
    u = np.empty(mesh.num_nodes(), dtype=np.float64)
    it, rr = C.c_int64(), C.c_double()
    probe = run(mesh, _lib.OUT_PARTITION, ctx=ctx)
    if probe.sizes().n_dir_faces > 0:
        if g_dirichlet is None:
            raise Error(ErrorCode.invalid_parameter,
                        "mesh has Dirichlet faces but the problem provides no g_dirichlet")
        r = assemble_system(mesh, f, g_dirichlet, g_neumann, coef, ctx)
        _lib.check(_lib.lib().fl_solve_system(ctx.handle, r.handle, C.byref(o), u.ctypes.data,
                                              _lib.MEM_HOST, C.byref(it), C.byref(rr)), "fl_solve_system")
    else:
        r = run(mesh, _lib.OUT_STIFFNESS | _lib.OUT_LOAD | _lib.OUT_PARTITION, f=f, coef=coef,
                g_neumann=g_neumann, ctx=ctx)
        _lib.check(_lib.lib().fl_solve_neumann(ctx.handle, mesh.device(ctx).handle, r.handle, int(pin_node),
                                               C.byref(o), u.ctypes.data, _lib.MEM_HOST, C.byref(it),
                                               C.byref(rr)), "fl_solve_neumann")
    return Solution(u, it.value, rr.value, r.partition())


def from_triplets(m: int, n: int, ii, jj, ss, ctx: Optional[Context] = None) -> CscMatrix:
    """sparse.hpp:61: COO with duplicates -> CSC on the
    GPU; duplicates summed in their original order, exact zeros dropped."""
    ctx = ctx or Context.default()
    ii = np.ascontiguousarray(ii, dtype=np.int32)
    jj = np.ascontiguousarray(jj, dtype=np.int32)
    ss = np.ascontiguousarray(ss, dtype=np.float64)
    if not (ii.shape == jj.shape == ss.shape):
        raise Error(ErrorCode.shape_mismatch, "triplet arrays differ in length")
    res = AssemblyResult(ctx)
    _lib.check(_lib.lib().fl_from_triplets(ctx.handle, int(m), int(n), ii.size,
                                           ii.ctypes.data if ii.size else None,
                                           jj.ctypes.data if jj.size else None,
                                           ss.ctypes.data if ss.size else None, _lib.MEM_HOST,
                                           res.handle), "fl_from_triplets")
    s = res.sizes()
    return CscMatrix(int(m), int(n), res.array(_lib.A_COL_PTR, np.int32, n + 1),
                     res.array(_lib.A_ROW_IDX, np.int32, s.nnz),
                     res.array(_lib.A_VALUES, np.float64, s.nnz))
