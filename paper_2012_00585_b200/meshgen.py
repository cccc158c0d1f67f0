"""Synthetic meshes for the BASELINE configs (numpy, vectorised).

The reference has only 2D quads (mesh.cpp:62-85); the 3D conventions below are ours and
are fixed here:
  * quad4  n x n: the reference's generate_structured numbering — vertex (i row, j col) is
           i*(n+1)+j, element (i,j) = [v0, v0+1, v0+n+2, v0+n+1] (CCW), row-major elements.
  * hex8   n^3: node (x,y,z) = (z*(n+1)+y)*(n+1)+x, lexicographic elements, local order
           000,100,110,010,001,101,111,011 (xyz bits).
  * tet4   Kuhn split of the n^3 hex grid: every cube cut along its (0,0,0)-(1,1,1)
           diagonal into 6 tets, one per axis permutation (conforming), 6 tets per cube in a
           fixed permutation order, cubes lexicographic.
  * hex27  n^3 Q2 elements on the (2n+1)^3 lexicographic node grid, local nodes
           lexicographic over the 3x3x3 sub-grid (x fastest).
  * permutations: perm = stable argsort of splitmix64(seed*2^32 + i) — a seeded uniform
           random permutation that numpy computes without a sequential Fisher-Yates loop.
"""
from __future__ import annotations

import numpy as np

_M1 = np.uint64(0x9E3779B97F4A7C15)
_M2 = np.uint64(0xBF58476D1CE4E5B9)
_M3 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + _M1
        z = (z ^ (z >> np.uint64(30))) * _M2
        z = (z ^ (z >> np.uint64(27))) * _M3
        return z ^ (z >> np.uint64(31))


def hash_permutation(n: int, seed: int) -> np.ndarray:
    keys = splitmix64((np.uint64(seed) << np.uint64(32)) + np.arange(n, dtype=np.uint64))
    return np.argsort(keys, kind="stable").astype(np.int64)


def quad4_structured(n: int):
    nv = n + 1
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    v0 = (i * nv + j).reshape(-1)
    conn = np.stack([v0, v0 + 1, v0 + nv + 1, v0 + nv], axis=1).astype(np.int64)
    return conn, nv * nv


def hex8_box(nx: int, ny: int, nz: int):
    """nx x ny x nz hex8 elements; node (x,y,z) = (z*(ny+1)+y)*(nx+1)+x."""
    ax, ay = nx + 1, ny + 1
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    base = ((z * ay + y) * ax + x).reshape(-1).astype(np.int64)
    ex, ey, ez = 1, ax, ax * ay
    offs = np.array([0, ex, ex + ey, ey, ez, ez + ex, ez + ex + ey, ez + ey], dtype=np.int64)
    return base[:, None] + offs[None, :], ax * ay * (nz + 1)


def hex8_structured(n: int):
    return hex8_box(n, n, n)


_KUHN_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def tet4_kuhn(n: int):
    nv = n + 1
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    base = ((z * nv + y) * nv + x).reshape(-1).astype(np.int64)
    step = np.array([1, nv, nv * nv], dtype=np.int64)
    tets = []
    for p in _KUHN_PERMS:
        o1 = step[p[0]]
        o2 = o1 + step[p[1]]
        o3 = o2 + step[p[2]]
        tets.append(np.stack([base, base + o1, base + o2, base + o3], axis=1))
    conn = np.stack(tets, axis=1).reshape(-1, 4)  # cube-major, 6 tets per cube
    return conn.astype(np.int64), nv ** 3


def hex27_structured(n: int):
    nv = 2 * n + 1
    z, y, x = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    base = ((2 * z * nv + 2 * y) * nv + 2 * x).reshape(-1).astype(np.int64)
    lz, ly, lx = np.meshgrid(np.arange(3), np.arange(3), np.arange(3), indexing="ij")
    offs = ((lz * nv + ly) * nv + lx).reshape(-1).astype(np.int64)
    return base[:, None] + offs[None, :], nv ** 3


def permute_elements(conn: np.ndarray, seed: int) -> np.ndarray:
    return conn[hash_permutation(conn.shape[0], seed)]


def permute_nodes(conn: np.ndarray, n_nodes: int, seed: int) -> np.ndarray:
    perm = hash_permutation(n_nodes, seed)
    return perm[conn]


def element_dofs(conn: np.ndarray, d: int) -> np.ndarray:
    """ElementDofs::flat for every element: node v carries DOFs v*d..v*d+d-1 (dof_map.hpp:59)."""
    if d == 1:
        return np.ascontiguousarray(conn, dtype=np.int64)
    k = np.arange(d, dtype=np.int64)
    return (conn[:, :, None] * d + k[None, None, :]).reshape(conn.shape[0], -1)


SEED_K = 42
SEED_PERM = 7

CONFIGS = {
    1: dict(mesh="quad4", n=256, d=1, perm=None, name="quad4 256^2 d=1 lexicographic (CSR)"),
    2: dict(mesh="hex8", n=64, d=3, perm="elements", name="hex8 64^3 d=3 elements permuted (CSR+CRAC)"),
    3: dict(mesh="tet4", n=128, d=1, perm="nodes", name="tet4 Kuhn 128^3x6 d=1 nodes permuted (CSR+CRAC)"),
    4: dict(mesh="hex27", n=48, d=3, perm=None, name="hex27 48^3 d=3 (CRAC vs CSR)"),
    5: dict(mesh="hex8", n=256, d=3, perm=None, name="hex8 256^3 d=3 row-partitioned"),
}

_GEN = {"quad4": quad4_structured, "hex8": hex8_structured, "tet4": tet4_kuhn,
        "hex27": hex27_structured}


def make_mesh(mesh: str, n: int, perm=None, seed: int = SEED_PERM):
    conn, n_nodes = _GEN[mesh](n)
    if perm == "elements":
        conn = permute_elements(conn, seed)
    elif perm == "nodes":
        conn = permute_nodes(conn, n_nodes, seed)
    return conn, n_nodes


def config_mesh(cfg: int, n: int | None = None):
    """(conn, n_nodes, d) of BASELINE config `cfg`, optionally at a smaller size n."""
    c = CONFIGS[cfg]
    conn, n_nodes = make_mesh(c["mesh"], c["n"] if n is None else n, c["perm"])
    return conn, n_nodes, c["d"]


def closed_form_nnz(mesh: str, n: int, d: int) -> int:
    """Exact NNZ of the structured patterns."""
    if mesh == "quad4":
        return d * d * (3 * n + 1) ** 2
    if mesh == "hex8":
        return d * d * (3 * n + 1) ** 3
    if mesh == "hex27":
        return d * d * (8 * n + 1) ** 3
    if mesh == "tet4":
        N = n + 1
        return d * d * (N ** 3 + 2 * (3 * (N - 1) * N * N + 3 * (N - 1) ** 2 * N + (N - 1) ** 3))
    raise ValueError(mesh)


def collapse_elements(conn, rng, frac: float = 0.3):
    """Degenerate elements (a local node repeated: a quad collapsed to a triangle, a hex to a
    wedge) for a random `frac` of the elements. scatter_element adds every (i, j) pair, so a
    repeated node's slots receive several contributions per element, in (i, j) order
    (assembly.hpp:77-92)."""
    conn = np.array(conn, copy=True)
    npe = conn.shape[1]
    for e in np.flatnonzero(rng.random(conn.shape[0]) < frac):
        a, b = rng.choice(npe, size=2, replace=False)
        conn[e, a] = conn[e, b]
    return conn
