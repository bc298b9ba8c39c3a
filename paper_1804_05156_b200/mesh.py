"""Mesh data model and canonical meshes (mesh.hpp).

``Mesh`` mirrors ``femlite::Mesh`` (mesh.hpp:60-96): the immutable triple
(nodes, elems, bd_flags) with zero-based int32 connectivity and one int8 flag
per element face (face f opposite local vertex f).  The arrays live on the
host; ``Mesh.device(ctx)`` uploads them once to an ``fl_mesh`` (device
buffers + the cached topology plan) that every assembly call reuses.

``make_mesh`` validates on the GPU (fl_mesh_validate: index range, flag values,
positive signed measure -- mesh.hpp:148-187).  The generators and boundary
flagging are input preparation, vectorised numpy restatements
of mesh.hpp:251-405 that are checked against the reference in tests.
"""
from __future__ import annotations

import ctypes as C
import sys
import enum

import numpy as np

from . import _lib
from .context import Context
from .errors import Error, ErrorCode

# mesh.hpp:29-30
TRI_FACES = np.array([[1, 2], [2, 0], [0, 1]], dtype=np.int64)
TET_FACES = np.array([[1, 3, 2], [0, 2, 3], [0, 3, 1], [0, 1, 2]], dtype=np.int64)


class MeshShape(enum.IntEnum):  # mesh.hpp:306
    unit_square = 0
    unit_cube = 1
    lshape = 2


class Mesh:
    def __init__(self, dim: int, nodes, elems, bd_flags=None):
        self.dim = int(dim)
        self.nodes = np.ascontiguousarray(np.asarray(nodes, dtype=np.float64).reshape(-1, self.dim))
        self.elems = np.ascontiguousarray(np.asarray(elems, dtype=np.int32).reshape(-1, self.dim + 1))
        if bd_flags is None or np.size(bd_flags) == 0:
            bd_flags = np.zeros(self.elems.shape, dtype=np.int8)
        self.bd_flags = np.ascontiguousarray(np.asarray(bd_flags, dtype=np.int8).reshape(self.elems.shape))
        self._dev = {}

    # mesh.hpp:62-64
    def num_nodes(self) -> int:
        return int(self.nodes.shape[0])

    def num_elems(self) -> int:
        return int(self.elems.shape[0])

    def with_flags(self, flags) -> "Mesh":
        return Mesh(self.dim, self.nodes, self.elems, flags)

    def device(self, ctx: Context | None = None) -> "DeviceMesh":
        ctx = ctx or Context.default()
        key = id(ctx)
        if key not in self._dev:
            self._dev[key] = DeviceMesh(ctx, self)
        return self._dev[key]


class DeviceMesh:
    """An ``fl_mesh``: device copies of the arrays plus the topology plan."""

    def __init__(self, ctx: Context, mesh: Mesh):
        self.ctx = ctx
        self.dim = mesh.dim
        self.n_nodes = mesh.num_nodes()
        self.n_elems = mesh.num_elems()
        self._h = C.c_void_p()
        L = _lib.lib()
        _lib.check(L.fl_mesh_create(ctx.handle, mesh.dim, self.n_nodes, self.n_elems,
                                    mesh.nodes.ctypes.data, mesh.elems.ctypes.data,
                                    mesh.bd_flags.ctypes.data, _lib.MEM_HOST, C.byref(self._h)),
                   "fl_mesh_create")

    @classmethod
    def from_device(cls, ctx: Context, dim: int, n_nodes: int, n_elems: int, nodes_ptr: int,
                    elems_ptr: int, flags_ptr: int | None) -> "DeviceMesh":
        self = cls.__new__(cls)
        self.ctx, self.dim, self.n_nodes, self.n_elems = ctx, dim, n_nodes, n_elems
        self._h = C.c_void_p()
        _lib.check(_lib.lib().fl_mesh_create(ctx.handle, dim, n_nodes, n_elems, nodes_ptr, elems_ptr,
                                             flags_ptr, _lib.MEM_DEVICE, C.byref(self._h)),
                   "fl_mesh_create")
        return self

    @property
    def handle(self):
        return self._h

    def set_columns(self, col_begin: int, col_end: int):
        """Own CSC columns [col_begin, col_end) only (one rank's shard)."""
        _lib.check(_lib.lib().fl_mesh_set_columns(self.ctx.handle, self._h, int(col_begin),
                                                  int(col_end)), "fl_mesh_set_columns")

    def plan(self):
        _lib.check(_lib.lib().fl_mesh_plan(self.ctx.handle, self._h), "fl_mesh_plan")

    def validate(self):
        _lib.check(_lib.lib().fl_mesh_validate(self.ctx.handle, self._h), "fl_mesh_validate")

    def __del__(self):
        if sys.is_finalizing():  # the CUDA runtime may already be gone; the OS reclaims
            return
        try:
            if self._h:
                _lib.lib().fl_mesh_destroy(self._h)
        except Exception:
            pass


def make_mesh(dim: int, nodes, elems, bd_flags=None, ctx: Context | None = None) -> Mesh:
    """mesh.hpp:174-187: validate the raw arrays (on the GPU) and build a Mesh."""
    if dim not in (2, 3):
        raise Error(ErrorCode.invalid_parameter, "mesh dimension must be 2 or 3")
    nodes = np.asarray(nodes, dtype=np.float64).ravel()
    elems = np.asarray(elems, dtype=np.int32).ravel()
    if nodes.size % dim:
        raise Error(ErrorCode.shape_mismatch, "node array length not divisible by dim")
    if elems.size % (dim + 1):
        raise Error(ErrorCode.shape_mismatch, "elem array length not divisible by dim+1")
    if bd_flags is not None and np.size(bd_flags) and np.size(bd_flags) != elems.size:
        raise Error(ErrorCode.shape_mismatch, "bd_flags shape differs from elems")
    m = Mesh(dim, nodes, elems, bd_flags)
    m.device(ctx).validate()
    return m


# ---------------------------------------------------------------------------
# generators (mesh.hpp:310-405), vectorised
# ---------------------------------------------------------------------------
def _unit_square(n: int):
    h = 1.0 / n
    j, i = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    nodes = np.stack([i.ravel() * h, j.ravel() * h], axis=1)
    jj, ii = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    v00 = (jj * (n + 1) + ii).ravel()
    v10, v01, v11 = v00 + 1, v00 + n + 1, v00 + n + 2
    elems = np.empty((n * n, 2, 3), dtype=np.int32)
    elems[:, 0] = np.stack([v00, v10, v11], axis=1)
    elems[:, 1] = np.stack([v00, v11, v01], axis=1)
    return nodes, elems.reshape(-1, 3)


_KUHN_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
_KUHN_ODD = [False, True, True, False, False, True]


def _unit_cube(n: int):
    h = 1.0 / n
    k, j, i = np.meshgrid(np.arange(n + 1), np.arange(n + 1), np.arange(n + 1), indexing="ij")
    nodes = np.stack([i.ravel() * h, j.ravel() * h, k.ravel() * h], axis=1)
    kk, jj, ii = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    base = [ii.ravel().astype(np.int64), jj.ravel().astype(np.int64), kk.ravel().astype(np.int64)]

    def nid(c):
        return (c[2] * (n + 1) + c[1]) * (n + 1) + c[0]

    elems = np.empty((n * n * n, 6, 4), dtype=np.int32)
    for p, perm in enumerate(_KUHN_PERMS):
        c = [base[0].copy(), base[1].copy(), base[2].copy()]
        tet = [nid(c)]
        for s in range(3):
            c[perm[s]] = c[perm[s]] + 1
            tet.append(nid(c))
        if _KUHN_ODD[p]:
            tet[2], tet[3] = tet[3], tet[2]
        elems[:, p] = np.stack(tet, axis=1)
    return nodes, elems.reshape(-1, 4)


def _lshape(n: int):
    h = 1.0 / n
    m = 2 * n
    ci = np.arange(m)
    cj, cii = np.meshgrid(ci, ci, indexing="ij")
    kept = ~((cii >= n) & (cj < n))  # cell (i, j) kept; array indexed [j, i]
    used = np.zeros((m + 1, m + 1), dtype=bool)
    used[:-1, :-1] |= kept
    used[:-1, 1:] |= kept
    used[1:, :-1] |= kept
    used[1:, 1:] |= kept
    remap = -np.ones((m + 1, m + 1), dtype=np.int64)
    remap[used] = np.arange(int(used.sum()))
    gj, gi = np.nonzero(used)  # row-major: j outer, i inner -- mesh.hpp:383-393 order
    nodes = np.stack([-1.0 + gi * h, -1.0 + gj * h], axis=1)
    kj, ki = np.nonzero(kept)
    v00, v10 = remap[kj, ki], remap[kj, ki + 1]
    v01, v11 = remap[kj + 1, ki], remap[kj + 1, ki + 1]
    elems = np.empty((kj.size, 2, 3), dtype=np.int32)
    elems[:, 0] = np.stack([v00, v10, v11], axis=1)
    elems[:, 1] = np.stack([v00, v11, v01], axis=1)
    return nodes, elems.reshape(-1, 3)


def generate_mesh(shape, n: int) -> Mesh:
    """mesh.hpp:410-419: canonical meshes, all flags zero."""
    if n < 1:
        raise Error(ErrorCode.invalid_parameter, "subdivision count must be >= 1")
    shape = MeshShape(shape)
    if shape == MeshShape.unit_square:
        nodes, elems = _unit_square(n)
        return Mesh(2, nodes, elems)
    if shape == MeshShape.unit_cube:
        nodes, elems = _unit_cube(n)
        return Mesh(3, nodes, elems)
    nodes, elems = _lshape(n)
    return Mesh(2, nodes, elems)


# ---------------------------------------------------------------------------
# boundary flagging (mesh.hpp:251-304)
# ---------------------------------------------------------------------------
def face_vertices(mesh: Mesh) -> np.ndarray:
    """[NT, d+1, d]: vertices of face f of every element (kTriFaces/kTetFaces order)."""
    table = TRI_FACES if mesh.dim == 2 else TET_FACES
    return mesh.elems[:, table]


def boundary_face_mask(mesh: Mesh) -> np.ndarray:
    """[NT, d+1] bool: faces that belong to exactly one element (sorted-key match)."""
    fv = np.sort(face_vertices(mesh).astype(np.int64), axis=2).reshape(-1, mesh.dim)
    n = max(mesh.num_nodes(), 1)
    if mesh.dim == 2:
        key = fv[:, 0] * n + fv[:, 1]
        _, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
    elif n ** 3 < 2 ** 62:
        key = (fv[:, 0] * n + fv[:, 1]) * n + fv[:, 2]
        _, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
    else:
        _, inv, cnt = np.unique(fv, axis=0, return_inverse=True, return_counts=True)
    return (cnt[inv.ravel()] == 1).reshape(mesh.num_elems(), mesh.dim + 1)


def set_boundary_flags(mesh: Mesh, classifier) -> Mesh:
    """Flag every true boundary face with classifier(centroid) (vectorised: the
    classifier receives coordinate arrays x, y, z of the face centroids)."""
    mask = boundary_face_mask(mesh)
    return mesh.with_flags(_classify(mesh, mask, classifier))


def _classify(mesh: Mesh, mask: np.ndarray, classifier) -> np.ndarray:
    d = mesh.dim
    flags = np.zeros(mask.shape, dtype=np.int8)
    t, lf = np.nonzero(mask)
    if t.size == 0:
        return flags
    table = TRI_FACES if d == 2 else TET_FACES
    verts = mesh.elems[t[:, None], table[lf]]  # [M, d]
    cen = []
    for c in range(d):  # mesh.hpp:288-294: sum over face vertices from 0.0, then / d
        acc = np.zeros(t.size)
        for k in range(d):
            acc = acc + mesh.nodes[verts[:, k], c]
        cen.append(acc / d)
    z = cen[2] if d == 3 else np.zeros(t.size)
    vals = np.asarray(classifier(cen[0], cen[1], z), dtype=np.int64)
    vals = np.broadcast_to(vals, t.shape)
    if np.any((vals < 0) | (vals > 3)):
        raise Error(ErrorCode.invalid_flag_value, "classifier returned a flag outside {0..3}")
    flags[t, lf] = vals.astype(np.int8)
    return flags


def generated_boundary_mask(mesh: Mesh, shape, n: int, chunk: int = 1 << 22) -> np.ndarray:
    """Boundary faces of an (unpermuted or permuted) generated mesh without a
    global sort: a face of these structured meshes is on the boundary iff all
    its vertices lie on one boundary segment.  Per-node segment bitmasks, AND
    over the face's vertices.  Equal to boundary_face_mask (tested)."""
    x = mesh.nodes[:, 0]
    y = mesh.nodes[:, 1]
    shape = MeshShape(shape)
    bits = np.zeros(mesh.num_nodes(), dtype=np.uint8)
    if shape in (MeshShape.unit_square, MeshShape.unit_cube):
        segs = []
        for c in range(mesh.dim):
            xc = mesh.nodes[:, c]
            segs += [xc == 0.0, xc == 1.0]
    else:
        segs = [x == -1.0, x == 1.0, y == -1.0, y == 1.0, (x == 0.0) & (y <= 0.0), (y == 0.0) & (x >= 0.0)]
    for k, sgm in enumerate(segs):
        bits |= (sgm.astype(np.uint8) << np.uint8(k))
    table = TRI_FACES if mesh.dim == 2 else TET_FACES
    out = np.empty((mesh.num_elems(), mesh.dim + 1), dtype=bool)
    for s0 in range(0, mesh.num_elems(), chunk):
        e = mesh.elems[s0:s0 + chunk]
        acc = np.full((e.shape[0], mesh.dim + 1), 0xFF, dtype=np.uint8)
        for k in range(mesh.dim):
            acc &= bits[e[:, table[:, k]]]
        out[s0:s0 + chunk] = acc != 0
    return out


def flag_generated(mesh: Mesh, shape, n: int, classifier) -> Mesh:
    return mesh.with_flags(_classify(mesh, generated_boundary_mask(mesh, shape, n), classifier))


# presets.hpp:36-45 classifiers (vectorised) + the L-shape one of config 2
TOL = 1e-10


def classifier_dirichlet(x, y, z):
    return np.ones_like(x, dtype=np.int64)


def classifier_neumann(x, y, z):
    return np.full(x.shape, 2, dtype=np.int64)


def classifier_mixed(x, y, z):
    return np.where(np.abs(y) < TOL, 2, 1)


def classifier_lshape(x, y, z):
    re = ((np.abs(x) < TOL) & (y < 0.0)) | ((np.abs(y) < TOL) & (x > 0.0))
    return np.where(re, 2, 1)
