"""One assemble_system step on a random Delaunay tetrahedralisation (ncu target)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
from scipy.spatial import Delaunay  # noqa: E402

import paper_1804_05156_b200 as fl  # noqa: E402
from meshes import fix_orientation  # noqa: E402
from paper_1804_05156_b200.mesh import Mesh  # noqa: E402

npts = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
pts = np.random.default_rng(0).random((npts, 3))
el = Delaunay(pts).simplices.astype(np.int32)
X = pts[el]
vol = np.abs(np.einsum("ij,ij->i", np.cross(X[:, 1] - X[:, 0], X[:, 2] - X[:, 0]), X[:, 3] - X[:, 0])) / 6
m = fl.set_boundary_flags(Mesh(3, pts, fix_orientation(3, pts, el[vol > 1e-12])), fl.classifier_dirichlet)
ctx = fl.Context.default()
r = fl.AssemblyResult(ctx)
for _ in range(2):
    fl.assemble_system(m, 1.0, 0.0, ctx=ctx, result=r)
    r.sizes()
print("ok", m.num_elems())
