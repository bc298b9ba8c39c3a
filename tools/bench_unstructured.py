"""Assembly throughput on an unstructured Delaunay tetrahedralisation (scipy),
per column-kernel choice, with the valence histogram (the fast kernels take
columns of <= 32 incidences in 3-D)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from scipy.spatial import Delaunay  # noqa: E402

import paper_1804_05156_b200 as fl  # noqa: E402
from paper_1804_05156_b200 import _lib  # noqa: E402
from paper_1804_05156_b200.mesh import Mesh  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests"))
from meshes import fix_orientation  # noqa: E402

npts = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
rng = np.random.default_rng(0)
pts = rng.random((npts, 3))
t0 = time.time()
el = Delaunay(pts).simplices.astype(np.int32)
X = pts[el]
vol = np.abs(np.einsum("ij,ij->i", np.cross(X[:, 1] - X[:, 0], X[:, 2] - X[:, 0]), X[:, 3] - X[:, 0])) / 6
el = fix_orientation(3, pts, el[vol > 1e-12])
m = fl.set_boundary_flags(Mesh(3, pts, el), fl.classifier_dirichlet)
val = np.bincount(m.elems.ravel(), minlength=m.num_nodes())
ctx = fl.Context.default()
out = {"n_nodes": m.num_nodes(), "n_elems": m.num_elems(), "build_s": time.time() - t0,
       "valence_mean": float(val.mean()), "valence_max": int(val.max()),
       "frac_nodes_over_32": float((val > 32).mean())}
for k in ["0", "1", "2"]:
    os.environ["FL_KERNEL"] = k
    r = fl.AssemblyResult(ctx)
    for _ in range(2):
        fl.assemble_system(m, 1.0, 0.0, ctx=ctx, result=r)
        r.sizes()
    ts = []
    for _ in range(5):
        t1 = time.perf_counter()
        fl.assemble_system(m, 1.0, 0.0, ctx=ctx, result=r)
        r.sizes()
        ts.append(time.perf_counter() - t1)
    out[f"ms_kernel_{k}"] = 1e3 * float(np.median(ts))
print(json.dumps(out))
