"""Tetrahedral mesh container, beam generator and vertex graph (host setup).

Mirrors tetsim.mesh (mesh.py:48-181, 293-315): the element order is part of
the contract -- assembly derives its deterministic fill order from it -- so
`generate_beam` reproduces the reference's node and element numbering
exactly (node id = i + nx*(j + ny*k); cells k-major; the six tets of a cell
in itertools.permutations order, odd permutations with nodes 1,2 swapped).
It is vectorised instead of looping per cell (the reference spends seconds in
Python loops at 100k nodes); mesh generation is setup, not the hot path.
"""

from __future__ import annotations

import enum
import itertools
from dataclasses import dataclass, field, replace

import numpy as np

__all__ = [
    "ElementKind",
    "Mesh",
    "Graph",
    "MeshError",
    "generate_beam",
    "vertex_adjacency",
]


class MeshError(ValueError):
    """Invalid mesh data (bad indices, degenerate elements, ...)."""


class ElementKind(enum.Enum):
    TETRA4 = "tetra4"


@dataclass(frozen=True)
class Mesh:
    """Immutable tetrahedral mesh (reference mesh.py:48-114).

    nodes        (n, 3) float64 positions
    elements     (m, 4) int64 node ids; list order defines the fill order
    fixed_nodes  sorted unique pinned node ids
    """

    nodes: np.ndarray
    elements: np.ndarray
    element_kind: ElementKind = ElementKind.TETRA4
    fixed_nodes: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))

    def __post_init__(self):
        nodes = np.ascontiguousarray(np.asarray(self.nodes, dtype=np.float64))
        elements = np.ascontiguousarray(np.asarray(self.elements, dtype=np.int64))
        fixed = np.asarray(self.fixed_nodes, dtype=np.int64)
        if nodes.ndim != 2 or nodes.shape[1] != 3:
            raise MeshError(f"nodes must be (n, 3), got {nodes.shape}")
        if elements.size and (elements.ndim != 2 or elements.shape[1] != 4):
            raise MeshError(f"elements must be (m, 4), got {elements.shape}")
        elements = elements.reshape(-1, 4)
        if elements.size and (elements.min() < 0 or elements.max() >= len(nodes)):
            raise MeshError("element index out of range")
        fixed = np.unique(fixed)
        if fixed.size and (fixed[0] < 0 or fixed[-1] >= len(nodes)):
            raise MeshError("fixed node index out of range")
        object.__setattr__(self, "nodes", nodes)
        object.__setattr__(self, "elements", elements)
        object.__setattr__(self, "fixed_nodes", fixed)
        vol = self.signed_volumes()
        if vol.size and np.any(vol == 0.0):
            bad = int(np.flatnonzero(vol == 0.0)[0])
            raise MeshError(f"element {bad} is degenerate (zero rest volume)")
        for a in (self.nodes, self.elements, self.fixed_nodes):
            a.setflags(write=False)

    @property
    def node_count(self) -> int:
        return len(self.nodes)

    @property
    def element_count(self) -> int:
        return len(self.elements)

    @property
    def ndof(self) -> int:
        return 3 * len(self.nodes)

    def signed_volumes(self) -> np.ndarray:
        """det([p1-p0, p2-p0, p3-p0]) / 6 per element (same LAPACK call as the reference)."""
        if not len(self.elements):
            return np.empty(0)
        p = self.nodes[self.elements]
        return np.linalg.det(p[:, 1:] - p[:, :1]) / 6.0

    def with_fixed_nodes(self, fixed_nodes) -> "Mesh":
        return replace(self, fixed_nodes=np.asarray(fixed_nodes, dtype=np.int64))

    def fixed_dofs(self) -> np.ndarray:
        return (3 * self.fixed_nodes[:, None] + np.arange(3)).ravel()


@dataclass(frozen=True)
class Graph:
    """Undirected vertex graph, CSR adjacency with sorted neighbour lists."""

    n: int
    indptr: np.ndarray
    indices: np.ndarray

    def __post_init__(self):
        self.indptr.setflags(write=False)
        self.indices.setflags(write=False)

    def neighbors(self, v: int) -> np.ndarray:
        return self.indices[self.indptr[v]: self.indptr[v + 1]]

    def degree(self, v: int) -> int:
        return int(self.indptr[v + 1] - self.indptr[v])


def _parity(perm) -> int:
    inv = sum(1 for i in range(3) for j in range(i + 1, 3) if perm[i] > perm[j])
    return -1 if inv % 2 else 1


def generate_beam(nx: int, ny: int, nz: int, spacing: float) -> Mesh:
    """Regular nx*ny*nz-node beam, each cell split into 6 tets on its main diagonal."""
    if nx < 2 or ny < 2 or nz < 2:
        raise MeshError(f"beam dimensions must be >= 2, got ({nx}, {ny}, {nz})")
    if not spacing > 0.0:
        raise MeshError(f"spacing must be positive, got {spacing}")
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    nodes = spacing * np.stack([i, j, k], axis=-1).reshape(-1, 3).astype(np.float64)

    ck, cj, ci = np.meshgrid(np.arange(nz - 1), np.arange(ny - 1), np.arange(nx - 1), indexing="ij")
    corner = np.stack([ci.ravel(), cj.ravel(), ck.ravel()], axis=1).astype(np.int64)  # k-major cells
    stride = np.array([1, nx, nx * ny], dtype=np.int64)
    base = corner @ stride
    tets = np.empty((len(corner), 6, 4), dtype=np.int64)
    for s, perm in enumerate(itertools.permutations(range(3))):
        step = np.zeros(3, dtype=np.int64)
        ids = [base]
        for axis in perm:
            step[axis] += 1
            ids.append(base + int(step @ stride))
        if _parity(perm) < 0:
            ids[1], ids[2] = ids[2], ids[1]
        tets[:, s, :] = np.stack(ids, axis=1)
    return Mesh(nodes=nodes, elements=tets.reshape(-1, 4))


def vertex_adjacency(mesh: Mesh) -> Graph:
    """Vertex graph: edge (i, j) iff i and j share an element; sorted, no self loops."""
    n = mesh.node_count
    el = mesh.elements
    if not len(el):
        return Graph(n=n, indptr=np.zeros(n + 1, dtype=np.int64), indices=np.empty(0, dtype=np.int64))
    a, b = np.nonzero(~np.eye(4, dtype=bool))
    src = el[:, a].ravel()
    dst = el[:, b].ravel()
    codes = np.unique(src * n + dst)
    src, dst = codes // n, codes % n
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
    return Graph(n=n, indptr=indptr, indices=dst.astype(np.int64))
