"""The five BASELINE.json configurations as seeded synthetic meshes.

Recipes follow SURVEY.md §8(d); all inputs are generated here (no dataset is
involved).  Randomness uses a counter-based splitmix64 so the same seed gives
the same mesh on any host:

  C1  unit_square:128, all boundary faces Dirichlet (flag 1), f = 1, g = 0
  C2  lshape:512, outer faces flag 1, re-entrant faces flag 2, interior nodes
      jittered by U(-0.2h, 0.2h) per coordinate, f = sin(pi x) sin(pi y), g = 0
  C3  unit_square:4096, flags 1, node ids AND element order permuted, f = 1
  C4  unit_cube:128 (Kuhn), flags 1, f = 1
  C5  unit_cube:256 (Kuhn), node ids permuted, coefficient
      a = 1 + 0.5 sin(2 pi x1) at element barycentres, f = 1

``scale`` shrinks n for parity tests with the same recipe.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import (Mesh, MeshShape, classifier_dirichlet, classifier_lshape, flag_generated,
                   generate_mesh)

DEFAULT_SEED = 20261019
MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Counter-based splitmix64 (Steele et al.) on uint64 arrays."""
    z = (x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uniform01(seed: int, counter: np.ndarray) -> np.ndarray:
    """U[0,1) doubles from (seed, counter): top 53 bits of splitmix64."""
    with np.errstate(over="ignore"):
        x = splitmix64(np.uint64(seed) * np.uint64(0x100000001B3) + counter.astype(np.uint64))
    return (x >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def permutation(seed: int, n: int) -> np.ndarray:
    """A seeded permutation of range(n) (stable argsort of splitmix64 keys)."""
    with np.errstate(over="ignore"):
        keys = splitmix64(np.uint64(seed) * np.uint64(0x9E3779B1) + np.arange(n, dtype=np.uint64))
    return np.argsort(keys, kind="stable").astype(np.int64)


def permute_nodes(mesh: Mesh, seed: int) -> Mesh:
    """Node k -> pi[k]: nodes moved, element entries mapped."""
    pi = permutation(seed, mesh.num_nodes())
    nodes = np.empty_like(mesh.nodes)
    nodes[pi] = mesh.nodes
    elems = pi[mesh.elems].astype(np.int32)
    return Mesh(mesh.dim, nodes, elems, mesh.bd_flags)


def permute_elements(mesh: Mesh, seed: int) -> Mesh:
    """Element order sigma: elem rows and their flag rows move together."""
    sigma = permutation(seed, mesh.num_elems())
    return Mesh(mesh.dim, mesh.nodes, mesh.elems[sigma], mesh.bd_flags[sigma])


def jitter_interior(mesh: Mesh, h: float, seed: int, amp: float = 0.2) -> Mesh:
    """x += U(-amp h, amp h), then y += U(...), for nodes on no flag-1/2 face,
    counters (2k, 2k+1) for node k; asserts positive orientation afterwards."""
    nv = mesh.dim + 1
    on_face = np.zeros(mesh.num_nodes(), dtype=bool)
    t, lf = np.nonzero(mesh.bd_flags > 0)
    for k in range(nv):
        sel = lf != k
        on_face[mesh.elems[t[sel], k]] = True
    interior = np.nonzero(~on_face)[0]
    nodes = mesh.nodes.copy()
    ux = uniform01(seed, 2 * interior.astype(np.uint64))
    uy = uniform01(seed, 2 * interior.astype(np.uint64) + np.uint64(1))
    nodes[interior, 0] = nodes[interior, 0] + (-amp * h + (2.0 * amp * h) * ux)
    nodes[interior, 1] = nodes[interior, 1] + (-amp * h + (2.0 * amp * h) * uy)
    out = Mesh(mesh.dim, nodes, mesh.elems, mesh.bd_flags)
    X = out.nodes[out.elems]
    e2 = X[:, 0] - X[:, 2]
    e3 = X[:, 1] - X[:, 0]
    area = 0.5 * (-e3[:, 0] * e2[:, 1] + e3[:, 1] * e2[:, 0])
    assert np.all(area > 0.0), "jitter produced a non-positive element"
    return out


@dataclass
class Config:
    name: str
    mesh: Mesh
    f: object                      # load source (api field spec)
    coef: object = None            # element coefficient (None = reference operator)
    g_dirichlet: object = 0.0
    g_neumann: object = None
    description: str = ""
    meta: dict = field(default_factory=dict)


FULL_N = {"C1": 128, "C2": 512, "C3": 4096, "C4": 128, "C5": 256}


def build(name: str, n: int | None = None, seed: int = DEFAULT_SEED, f_mode: str = "kind") -> Config:
    """Build config `name` at its full size (n=None) or at subdivision n.

    f_mode: 'kind' (device-evaluated built-in field) or 'samples' (host-sampled
    values, bitwise with the reference's f; only matters for C2's sin*sin)."""
    n = n or FULL_N[name]
    if name in ("C1", "C3"):
        m = generate_mesh(MeshShape.unit_square, n)
        m = flag_generated(m, MeshShape.unit_square, n, classifier_dirichlet)
        if name == "C3":
            m = permute_elements(permute_nodes(m, seed), seed + 1)
        return Config(name, m, 1.0, description=f"unit_square:{n}" + (" permuted" if name == "C3" else ""),
                      meta={"n": n, "seed": seed})
    if name == "C2":
        m = generate_mesh(MeshShape.lshape, n)
        m = flag_generated(m, MeshShape.lshape, n, classifier_lshape)
        m = jitter_interior(m, 1.0 / n, seed)
        f = "sinsin"
        if f_mode == "samples":
            f = host_samples(m, rule=0, kind=2)
        return Config(name, m, f, description=f"lshape:{n} jittered", meta={"n": n, "seed": seed})
    if name in ("C4", "C5"):
        m = generate_mesh(MeshShape.unit_cube, n)
        m = flag_generated(m, MeshShape.unit_cube, n, classifier_dirichlet)
        coef = None
        if name == "C5":
            m = permute_nodes(m, seed)
            coef = "coef_c5"
        return Config(name, m, 1.0, coef=coef,
                      description=f"unit_cube:{n}" + (" permuted+coef" if name == "C5" else ""),
                      meta={"n": n, "seed": seed})
    raise ValueError(name)


def host_samples(mesh: Mesh, rule: int, kind: int, value: float = 0.0) -> np.ndarray:
    """fl_host_sample: a built-in field at the rule's points, evaluated on the host
    with glibc sin (bitwise the reference's std::function evaluation)."""
    from . import _lib
    nv = mesh.dim + 1
    count = {0: mesh.num_elems() * nv, 1: mesh.num_elems(), 2: mesh.num_nodes(),
             3: mesh.num_elems() * nv}[rule]
    out = np.empty(count, dtype=np.float64)
    _lib.check(_lib.lib().fl_host_sample(mesh.dim, mesh.num_nodes(), mesh.num_elems(),
                                         mesh.nodes.ctypes.data, mesh.elems.ctypes.data, rule, kind,
                                         value, out.ctypes.data), "fl_host_sample")
    return out


def algorithmic_bytes(dim: int, n_nodes: int, n_elems: int, nnz: int) -> int:
    """B_SL: elems + nodes + col_ptr + (row_idx, values) + b."""
    return 4 * (dim + 1) * n_elems + 8 * dim * n_nodes + 4 * (n_nodes + 1) + 12 * nnz + 8 * n_nodes


def system_bytes(dim: int, n_nodes: int, n_elems: int, nnz: int, n_free: int, nnz_ff: int) -> int:
    """B_sys: B_SL + flags + node lists + (u0, b_mod) + A_ff + b_f."""
    return (algorithmic_bytes(dim, n_nodes, n_elems, nnz) + (dim + 1) * n_elems + 4 * n_nodes
            + 16 * n_nodes + 4 * (n_free + 1) + 12 * nnz_ff + 8 * n_free)
