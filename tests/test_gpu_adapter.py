"""GPU: the reference's own C++ API vs the B200 path through the C++ adapter.

oracle/_ref/adapter_check (built by oracle/Makefile from oracle/adapter_check.cpp
with the unmodified femlite headers) calls femlite::assemble_blockwise,
assemble_load, partition_boundary, apply_neumann, apply_dirichlet, submatrix and
the adapter's femlite_b200:: equivalents (include/femlite_b200_adapter.hpp ->
C-ABI -> libfemlite_b200.so) on the same meshes and compares them bitwise.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


@pytest.mark.skipif(not os.path.exists(BIN), reason="adapter_check not built (needs the reference headers)")
def test_reference_api_vs_adapter_bitwise():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
