"""set_boundary_flags on the GPU (mesh.hpp:251-304).

The face matching (which faces belong to exactly one element) and the
centroids run on the device (fl_boundary_faces); the classifier -- the
reference's arbitrary callable -- runs on the host on the boundary faces'
centroids only; fl_mesh_set_boundary_flags writes the device mesh's flags, so
an assembly on the same device mesh follows without another upload.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .context import Context
from .errors import Error, ErrorCode
from .mesh import DeviceMesh, Mesh


def boundary_faces(mesh: Mesh, ctx: Optional[Context] = None, device_mesh: Optional[DeviceMesh] = None):
    """-> (faces int32[M, 2] of (t, local face) ascending, centroids float64[M, 3])."""
    ctx = ctx or Context.default()
    dm = device_mesh or DeviceMesh(ctx, mesh)
    L = _lib.lib()
    n = C.c_int64()
    _lib.check(L.fl_boundary_faces(ctx.handle, dm.handle, C.byref(n)), "fl_boundary_faces")
    faces = np.empty((n.value, 2), dtype=np.int32)
    cen = np.empty((n.value, 3), dtype=np.float64)
    if n.value:
        _lib.check(L.fl_boundary_faces_copy(ctx.handle, dm.handle, faces.ctypes.data, cen.ctypes.data,
                                            _lib.MEM_HOST), "fl_boundary_faces_copy")
    return faces, cen


def set_boundary_flags(mesh: Mesh, classifier, ctx: Optional[Context] = None) -> Mesh:
    """mesh.hpp:251: flag every true boundary face with classifier(centroid), 0
    elsewhere.  ``classifier`` is an int (every boundary face gets it) or a
    vectorised callable classifier(x, y, z) -> int array over the boundary
    faces' centroids.  Returns the flagged Mesh; its device copy (with the
    flags already written on the GPU) is cached for the next assembly."""
    ctx = ctx or Context.default()
    dm = DeviceMesh(ctx, Mesh(mesh.dim, mesh.nodes, mesh.elems))
    faces, cen = boundary_faces(mesh, ctx, dm)
    L = _lib.lib()
    if callable(classifier):
        vals = np.asarray(classifier(cen[:, 0], cen[:, 1], cen[:, 2]), dtype=np.int64)
        vals = np.broadcast_to(vals, (faces.shape[0],))
        if np.any((vals < 0) | (vals > 3)):
            raise Error(ErrorCode.invalid_flag_value, "classifier returned a flag outside {0..3}")
        v8 = np.ascontiguousarray(vals, dtype=np.int8)
        _lib.check(L.fl_mesh_set_boundary_flags(ctx.handle, dm.handle,
                                                v8.ctypes.data if v8.size else None, 0, _lib.MEM_HOST),
                   "fl_mesh_set_boundary_flags")
    else:
        fill = int(classifier)
        if fill < 0 or fill > 3:
            raise Error(ErrorCode.invalid_flag_value, "classifier returned a flag outside {0..3}")
        v8 = np.full(faces.shape[0], fill, dtype=np.int8)
        _lib.check(L.fl_mesh_set_boundary_flags(ctx.handle, dm.handle, None, fill, _lib.MEM_HOST),
                   "fl_mesh_set_boundary_flags")
    flags = np.zeros((mesh.num_elems(), mesh.dim + 1), dtype=np.int8)
    flags[faces[:, 0], faces[:, 1]] = v8
    out = mesh.with_flags(flags)
    out._dev = {id(ctx): dm}
    return out
