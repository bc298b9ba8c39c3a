"""Test meshes: the reference's acceptance meshes (acceptance.cpp:90-96), the
config recipes at small n, and edge cases (single elements, high-valence
nodes that exercise the chunked column path, jittered 3-D)."""
from __future__ import annotations

import numpy as np

from paper_1804_05156_b200 import configs
from paper_1804_05156_b200.mesh import (Mesh, MeshShape, classifier_dirichlet, classifier_lshape,
                                        classifier_mixed, flag_generated, generate_mesh,
                                        set_boundary_flags)


def _signed(dim, nodes, elems):
    X = nodes[elems]
    if dim == 2:
        e2 = X[:, 0] - X[:, 2]
        e3 = X[:, 1] - X[:, 0]
        return 0.5 * (-e3[:, 0] * e2[:, 1] + e3[:, 1] * e2[:, 0])
    a, b, c = X[:, 1] - X[:, 0], X[:, 2] - X[:, 0], X[:, 3] - X[:, 0]
    return np.einsum("ij,ij->i", np.cross(a, b), c)


def fix_orientation(dim, nodes, elems):
    """mesh.hpp:199-218: swap the last two vertices of negatively oriented elements."""
    elems = elems.copy()
    neg = _signed(dim, nodes, elems) < 0
    elems[neg, dim - 1], elems[neg, dim] = elems[neg, dim].copy(), elems[neg, dim - 1].copy()
    return elems


def fan2d(k=40):
    """Centre node with k incident triangles (> 32: chunked column path)."""
    ang = 2 * np.pi * np.arange(k) / k
    nodes = np.vstack([[0.0, 0.0], np.stack([np.cos(ang), np.sin(ang)], 1)])
    elems = np.array([[0, 1 + i, 1 + (i + 1) % k] for i in range(k)], dtype=np.int32)
    m = Mesh(2, nodes, fix_orientation(2, nodes, elems))
    return set_boundary_flags(m, classifier_dirichlet)


def bipyramid3d(k=20):
    """Centre node with 2k incident tetrahedra (> 32)."""
    ang = 2 * np.pi * np.arange(k) / k
    ring = np.stack([np.cos(ang), np.sin(ang), np.zeros(k)], 1)
    nodes = np.vstack([[0, 0, 0], ring, [0, 0, 1.0], [0, 0, -1.0]])
    top, bot = k + 1, k + 2
    el = []
    for i in range(k):
        a, b = 1 + i, 1 + (i + 1) % k
        el.append([0, a, b, top])
        el.append([0, b, a, bot])
    elems = np.array(el, dtype=np.int32)
    m = Mesh(3, nodes, fix_orientation(3, nodes, elems))
    return set_boundary_flags(m, classifier_dirichlet)


def jitter3d(n=4, seed=7):
    m = flag_generated(generate_mesh(MeshShape.unit_cube, n), MeshShape.unit_cube, n,
                       classifier_dirichlet)
    interior = np.all((m.nodes > 0) & (m.nodes < 1), axis=1)
    rng = np.random.default_rng(seed)
    nodes = m.nodes.copy()
    nodes[interior] += rng.uniform(-0.15 / n, 0.15 / n, size=(int(interior.sum()), 3))
    assert np.all(_signed(3, nodes, m.elems) > 0)
    return Mesh(3, nodes, m.elems, m.bd_flags)


def single_triangle():
    return set_boundary_flags(Mesh(2, [0, 0, 1, 0, 0, 1], [0, 1, 2]), classifier_dirichlet)


def single_tet():
    return set_boundary_flags(Mesh(3, [0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1], [0, 1, 2, 3]),
                              classifier_dirichlet)


def catalog():
    """name -> Mesh (flagged).  Small enough for the reference in seconds."""
    out = {}
    for n in (1, 2, 4, 8, 16, 33):
        out[f"square{n}"] = flag_generated(generate_mesh(MeshShape.unit_square, n),
                                           MeshShape.unit_square, n, classifier_dirichlet)
    for n in (1, 2, 4, 8):
        out[f"lshape{n}"] = flag_generated(generate_mesh(MeshShape.lshape, n), MeshShape.lshape,
                                           n, classifier_lshape)
    for n in (1, 2, 4, 5):
        out[f"cube{n}"] = flag_generated(generate_mesh(MeshShape.unit_cube, n),
                                         MeshShape.unit_cube, n, classifier_dirichlet)
    out["square8_mixed"] = flag_generated(generate_mesh(MeshShape.unit_square, 8),
                                          MeshShape.unit_square, 8, classifier_mixed)
    out["cube3_mixed"] = flag_generated(generate_mesh(MeshShape.unit_cube, 3),
                                        MeshShape.unit_cube, 3, classifier_mixed)
    out["C1_n16"] = configs.build("C1", n=16).mesh
    out["C2_n16"] = configs.build("C2", n=16).mesh
    out["C3_n24"] = configs.build("C3", n=24).mesh
    out["C4_n6"] = configs.build("C4", n=6).mesh
    out["C5_n6"] = configs.build("C5", n=6).mesh
    out["fan40"] = fan2d(40)
    out["bipyramid20"] = bipyramid3d(20)
    out["jitter3d"] = jitter3d(4)
    out["triangle"] = single_triangle()
    out["tet"] = single_tet()
    return out
