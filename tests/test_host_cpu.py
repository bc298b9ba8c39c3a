"""CPU tests of the product's host side (no GPU needed).

* the C-ABI library loads and exports every entry point include/*.h declares;
* the host mirrors of the reference's mesh API (generators, boundary flags)
  reproduce the reference's arrays (golden fixtures) bitwise;
* the host-side field sampling of the ABI (fl_host_sample) equals the oracle's
  restatement of the reference's load-point rule;
* the multi-GPU shard arithmetic (column ranges, offsets, stitching).
"""
from __future__ import annotations

import ctypes as C
import glob
import os
import re

import numpy as np
import pytest

from oracle import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = sorted(glob.glob(os.path.join(ROOT, "include", "*.h")))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _declared_symbols():
    syms = set()
    for h in HEADERS:
        txt = open(h).read()
        syms |= set(re.findall(r"FL_API\s+[\w\s\*]+?\b(fl_\w+)\s*\(", txt))
    return syms


def test_headers_declare_abi():
    syms = _declared_symbols()
    assert {"fl_create", "fl_mesh_create", "fl_assemble", "fl_result_sizes", "fl_result_copy",
            "fl_mesh_set_columns", "fl_submatrix"} <= syms


def test_library_exports_every_declared_symbol():
    from paper_1804_05156_b200 import _lib
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in sorted(_declared_symbols()) if not hasattr(lib, s)]
    assert not missing, missing
    # the ctypes signature table covers the same set
    assert _declared_symbols() <= set(_lib.SIGNATURES), \
        sorted(_declared_symbols() - set(_lib.SIGNATURES))


def test_abi_version_matches_header():
    from paper_1804_05156_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "femlite_b200.h")).read()
    v = int(re.search(r"#define FL_ABI_VERSION (\d+)", hdr).group(1))
    assert _lib.lib().fl_abi_version() == v


def test_sizes_struct_layout_matches_header():
    from paper_1804_05156_b200 import _lib
    assert C.sizeof(_lib.Sizes) == 6 * 4 + 2 * 8


@pytest.mark.parametrize("tag,shape,n,cls", [
    ("square1", 0, 1, "dirichlet"), ("square4_mixed", 0, 4, "mixed"), ("square8", 0, 8, "dirichlet"),
    ("lshape4", 2, 4, "lshape"), ("cube2", 1, 2, "dirichlet"), ("cube3_mixed", 1, 3, "mixed"),
])
def test_generators_and_flags_match_reference(tag, shape, n, cls):
    from paper_1804_05156_b200 import mesh as M
    g = np.load(os.path.join(GOLDEN, tag + ".npz"))
    m = M.generate_mesh(M.MeshShape(shape), n)
    assert m.dim == int(g["dim"])
    assert m.nodes.reshape(-1).tobytes() == g["nodes"].reshape(-1).tobytes()
    np.testing.assert_array_equal(m.elems.reshape(-1), g["elems"].reshape(-1))
    classifier = {"dirichlet": M.classifier_dirichlet, "mixed": M.classifier_mixed,
                  "lshape": M.classifier_lshape}[cls]
    fm = M.set_boundary_flags(m, classifier)
    np.testing.assert_array_equal(fm.bd_flags.reshape(-1), g["flags"].reshape(-1))
    # the vectorised large-mesh flagging path agrees as well
    gm = M.flag_generated(m, M.MeshShape(shape), n, classifier)
    np.testing.assert_array_equal(gm.bd_flags.reshape(-1), g["flags"].reshape(-1))


@pytest.mark.parametrize("tag", ["square8_jit", "lshape4_jit", "cube3_mixed_jit"])
@pytest.mark.parametrize("kind", [po.FIELD_CONST, po.FIELD_SINSIN, po.FIELD_XYZ])
def test_host_sample_matches_oracle_load_points(tag, kind):
    from paper_1804_05156_b200 import configs
    from paper_1804_05156_b200.mesh import Mesh
    g = np.load(os.path.join(GOLDEN, tag + ".npz"))
    d = int(g["dim"])
    m = Mesh(d, g["nodes"], g["elems"])
    got = configs.host_samples(m, rule=0, kind=kind, value=1.25)
    want = po.sample_load_points(d, g["nodes"], g["elems"], kind, 1.25)
    assert np.asarray(got).tobytes() == np.asarray(want).tobytes()


def test_configs_are_deterministic():
    from paper_1804_05156_b200 import configs
    a = configs.build("C2", n=12)
    b = configs.build("C2", n=12)
    assert a.mesh.nodes.tobytes() == b.mesh.nodes.tobytes()
    np.testing.assert_array_equal(a.mesh.elems, b.mesh.elems)
    np.testing.assert_array_equal(a.mesh.bd_flags, b.mesh.bd_flags)
    c = configs.build("C5", n=3)
    assert c.mesh.dim == 3 and c.mesh.num_elems() == 6 * 27


# ---- shard arithmetic ---------------------------------------------------------------
@pytest.mark.parametrize("n,w", [(0, 1), (1, 3), (10, 3), (4225, 8), (7, 7)])
def test_column_ranges_partition(n, w):
    from paper_1804_05156_b200.shard import column_ranges
    rs = column_ranges(n, w)
    assert len(rs) == w and rs[0][0] == 0 and rs[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    sizes = [b - a for a, b in rs]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("tag", ["square8_jit", "cube3_mixed_jit"])
@pytest.mark.parametrize("w", [1, 2, 3, 5])
def test_stitch_shards_reproduces_reference(tag, w):
    from paper_1804_05156_b200.shard import column_ranges, exclusive_offsets, stitch_csc
    g = np.load(os.path.join(GOLDEN, tag + ".npz"))
    d, nodes, elems = int(g["dim"]), g["nodes"], g["elems"]
    n = nodes.shape[0]
    parts, counts = [], []
    for c0, c1 in column_ranges(n, w):
        sub = po.assemble_columns(d, nodes, elems, np.arange(c0, c1, dtype=np.int32))
        parts.append((sub.col_ptr, sub.row_idx, sub.values))
        counts.append([c1 - c0, 0, sub.nnz, 0])
    full = stitch_csc(n, parts)
    np.testing.assert_array_equal(full.col_ptr, g["a_col_ptr"])
    np.testing.assert_array_equal(full.row_idx, g["a_row_idx"])
    assert full.values.tobytes() == g["a_values"].tobytes()
    off = exclusive_offsets(np.asarray(counts))
    assert off[-1, 2] == g["a_col_ptr"][-1]
    for r, (c0, _) in enumerate(column_ranges(n, w)):
        assert off[r, 2] == g["a_col_ptr"][c0]


def test_stitch_rejects_unshifted_shard():
    from paper_1804_05156_b200.shard import stitch_csc
    with pytest.raises(ValueError):
        stitch_csc(3, [(np.array([1, 2]), np.array([0]), np.array([1.0]))])


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include/femlite"),
                    reason="reference headers absent")
def test_adapter_header_compiles_against_reference():
    import subprocess
    r = subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                        "-I/root/reference/proj/include", f"-I{ROOT}/include",
                        os.path.join(ROOT, "oracle", "adapter_check.cpp")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
