"""Per-device context (fl_ctx): CUDA device, stream, launch counter."""
from __future__ import annotations

import ctypes as C
import sys

from . import _lib


class Context:
    """Owns an ``fl_ctx``.  One per device; ``Context.default()`` is shared."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        _lib.check(_lib.lib().fl_create(device, C.byref(self._h)), "fl_create")
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = cls(device)
        return cls._default[device]

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: int | None):
        """Run on an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)."""
        _lib.check(_lib.lib().fl_set_stream(self._h, C.c_void_p(stream_ptr or 0)), "fl_set_stream")

    def synchronize(self):
        _lib.check(_lib.lib().fl_synchronize(self._h), "fl_synchronize")

    def launch_count(self) -> int:
        return int(_lib.lib().fl_launch_count(self._h))

    def last_timings(self):
        buf = (C.c_double * 4)()
        _lib.check(_lib.lib().fl_last_timings(self._h, buf), "fl_last_timings")
        return list(buf)

    def last_kernel_timings(self):
        """[element records, column kernel, placement] ms of the last assembly (FL_PROFILE=1)."""
        buf = (C.c_double * 3)()
        _lib.check(_lib.lib().fl_last_kernel_timings(self._h, buf), "fl_last_kernel_timings")
        return list(buf)

    def close(self):
        if self._h:
            _lib.lib().fl_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        if sys.is_finalizing():  # the CUDA runtime may already be gone; the OS reclaims
            return
        try:
            self.close()
        except Exception:
            pass
