"""Benchmark of SURVEY.md §8(f) row 3: from_triplets on the GPU (host COO in,
CSC out: includes H2D/D2H) vs the reference's from_triplets (oracle/_ref)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1804_05156_b200 as fl  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 50_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000
rng = np.random.default_rng(0)
ii = rng.integers(0, n, count).astype(np.int32)
jj = rng.integers(0, n, count).astype(np.int32)
ss = rng.standard_normal(count)
ctx = fl.Context.default()
fl.from_triplets(n, n, ii[:1000], jj[:1000], ss[:1000], ctx=ctx)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    a = fl.from_triplets(n, n, ii, jj, ss, ctx=ctx)
    ts.append(time.perf_counter() - t0)
sec = float(np.median(ts))
line = {"metric": "from_triplets triplets/s (GPU, host COO in, host CSC out)", "count": count, "n": n,
        "nnz": int(a.col_ptr[-1]), "ms": sec * 1e3, "value": count / sec, "unit": "triplets/s"}
if po.have_ref():
    c2 = min(count, 5_000_000)
    t0 = time.perf_counter()
    r = po.from_triplets(n, n, ii[:c2], jj[:c2], ss[:c2], which="ref")
    rs = time.perf_counter() - t0
    g = fl.from_triplets(n, n, ii[:c2], jj[:c2], ss[:c2], ctx=ctx)
    line["cpu_baseline"] = {"value": c2 / rs, "unit": "triplets/s", "cores": 1, "kind": "reference",
                            "sample": f"first {c2} triplets, femlite from_triplets, 1 thread"}
    line["bitwise_equal_on_sample"] = bool(np.array_equal(g.col_ptr, r.col_ptr) and
                                           np.array_equal(g.row_idx, r.row_idx) and
                                           g.values.tobytes() == r.values.tobytes())
print(json.dumps(line))
