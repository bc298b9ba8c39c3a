"""Error codes and exception type of the reference (error.hpp:10-37)."""
from __future__ import annotations

import enum


class ErrorCode(enum.IntEnum):
    index_out_of_range = 0
    shape_mismatch = 1
    non_positive_volume = 2
    invalid_flag_value = 3
    degenerate_element = 4
    invalid_parameter = 5
    parse_error = 6
    io_error = 7
    unknown_rule = 8
    unsorted_index_set = 9
    too_large_for_dense = 10
    not_positive_definite = 11
    max_iter_exceeded = 12
    no_dirichlet_boundary = 13
    unsupported_boundary_type = 14


class Error(RuntimeError):
    """femlite::Error: carries the reference's ErrorCode (None for ABI/CUDA
    failures, which additionally carry the raw ``status``)."""

    def __init__(self, code, what: str = "", status: int | None = None):
        super().__init__(what)
        self._code = code
        self.status = status if status is not None else (int(code) + 1 if code is not None else None)

    def code(self):
        return self._code
