"""The reference's text writers on the GPU.

    write_matrix_market(a, out)   matrix_market.hpp:15-24
    write_mesh(mesh, out)         mesh_io.hpp:125-142
    format_real(v) / format_reals detail::format_real, mesh_io.hpp:56-60 ("%.17g")

The text is formatted on the device (exact "%.17g", csrc/fl_text.cu) and is
byte-identical to the reference's output; `out` may be a path, a binary file
object, or None (the bytes are returned).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .context import Context
from .errors import Error, ErrorCode
from .mesh import Mesh


class Text:
    """A device-resident text (fl_text)."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        h = C.c_void_p()
        _lib.check(_lib.lib().fl_text_create(ctx.handle, C.byref(h)), "fl_text_create")
        self._h = h

    @property
    def handle(self):
        return self._h

    def size(self) -> int:
        n = C.c_int64()
        _lib.check(_lib.lib().fl_text_size(self._h, C.byref(n)), "fl_text_size")
        return n.value

    def bytes(self) -> bytes:
        n = self.size()
        buf = np.empty(max(n, 1), dtype=np.uint8)
        _lib.check(_lib.lib().fl_text_copy(self._h, buf.ctypes.data, n, _lib.MEM_HOST), "fl_text_copy")
        return buf[:n].tobytes()

    def __del__(self):
        try:
            if self._h:
                _lib.lib().fl_text_destroy(self._h)
                self._h = None
        except Exception:
            pass


def _emit(data: bytes, out):
    if out is None:
        return data
    if isinstance(out, str):
        try:
            with open(out, "wb") as f:
                f.write(data)
        except OSError as e:  # write_matrix_market(a, path): io_error
            raise Error(ErrorCode.io_error, f"cannot open '{out}' for writing") from e
        return None
    out.write(data)
    return None


def write_matrix_market(a, out=None, ctx: Optional[Context] = None, text: Optional[Text] = None):
    """matrix_market.hpp:15-24 for a CscMatrix (host arrays)."""
    ctx = ctx or Context.default()
    t = text or Text(ctx)
    cp = np.ascontiguousarray(a.col_ptr, dtype=np.int32)
    ri = np.ascontiguousarray(a.row_idx, dtype=np.int32)
    va = np.ascontiguousarray(a.values, dtype=np.float64)
    if cp.size != a.n + 1 or ri.size != va.size or int(cp[-1]) != va.size:
        raise Error(ErrorCode.shape_mismatch, "CSC arrays inconsistent")
    _lib.check(_lib.lib().fl_write_matrix_market(ctx.handle, int(a.m), int(a.n), cp.ctypes.data,
                                                 ri.ctypes.data if ri.size else None,
                                                 va.ctypes.data if va.size else None,
                                                 _lib.MEM_HOST, t.handle), "fl_write_matrix_market")
    return _emit(t.bytes(), out)


def write_result_matrix_market(result, out=None, free_block: bool = False, text: Optional[Text] = None):
    """Write A (or A(free, free)) of an AssemblyResult straight from device memory."""
    ctx = result.ctx
    t = text or Text(ctx)
    s = result.sizes()
    if free_block:
        cp, ri, va, m = _lib.AFF_COL_PTR, _lib.AFF_ROW_IDX, _lib.AFF_VALUES, s.n_free
        n = s.n_free_cols
    else:
        cp, ri, va, m = _lib.A_COL_PTR, _lib.A_ROW_IDX, _lib.A_VALUES, getattr(result, "_rows", s.n)
        n = s.n
    _lib.check(_lib.lib().fl_write_matrix_market(ctx.handle, int(m), int(n), result.device_ptr(cp)[0],
                                                 result.device_ptr(ri)[0], result.device_ptr(va)[0],
                                                 _lib.MEM_DEVICE, t.handle), "fl_write_matrix_market")
    return _emit(t.bytes(), out)


def write_mesh(mesh: Mesh, out=None, ctx: Optional[Context] = None, text: Optional[Text] = None):
    """mesh_io.hpp:125-142 of a mesh (its device copy)."""
    ctx = ctx or Context.default()
    t = text or Text(ctx)
    _lib.check(_lib.lib().fl_write_mesh(ctx.handle, mesh.device(ctx).handle, t.handle), "fl_write_mesh")
    return _emit(t.bytes(), out)


def format_reals(values, exact: bool = False, ctx: Optional[Context] = None) -> list:
    """detail::format_real ("%.17g") of every value, formatted on the device.
    exact=True forces the big-integer rounding path for every value (test hook)."""
    ctx = ctx or Context.default()
    v = np.ascontiguousarray(values, dtype=np.float64).ravel()
    t = Text(ctx)
    _lib.check(_lib.lib().fl_format_reals(ctx.handle, v.size, v.ctypes.data if v.size else None,
                                          _lib.MEM_HOST, 1 if exact else 0, t.handle), "fl_format_reals")
    data = t.bytes()
    return data.decode().split("\n")[:-1] if data else []


def format_real(v: float, ctx: Optional[Context] = None) -> str:
    return format_reals([v], ctx=ctx)[0]
