"""Seeded 2D triangle curl-curl systems: the reference's own sparse regime
(input generation, not the hot path).

The reference meshes and assembles 2D problems only (``mesh.py``, ``fem.py``).
This module restates, vectorised, the pieces its tests and the paper use for
the uniform family: the unit square as two triangles (``uniform_tri_mesh(0)``,
mesh.py:163-182), red refinement with the reference's vertex / edge / cell
numbering (``refine``, mesh.py:201-257; ``mesh_from_cells``, mesh.py:108-160),
the vertical-stripes coefficient (``assign_mu_stripes``, mesh.py:408-413),
Whitney triangle elements (``tri_element_matrices``, fem.py:53-84) and the
assembly with tangential Dirichlet elimination (``assemble`` /
``build_gradient``, fem.py:111-195).  Every floating-point operation follows
the reference's order, so the systems are bit-identical to the reference's
(tests/test_tri2d.py checks this against the reference-generated fixtures).

In 2D the harmonic-extension components stay small (3-8 DoFs), P is sparse
and the hierarchy has many levels: the regime where the north star's kernel
design (CSR SpMV, sparse P / P^T, short wavefront sweeps) is the hot path.
``stripes_system(L)`` at L = 9 (785,408 DoFs) is bench.py's ``--config 2d-L9``.
"""

from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np
import scipy.sparse as sp

__all__ = ["TriMesh", "uniform_tri_mesh0", "refine", "refinement_chain", "assemble_tri", "stripes_system",
           "tri_chain"]


def _csr(a, shape=None):
    """The reference's csr() normal form (sparse.py:58-65)."""
    m = sp.csr_matrix(a, shape=shape, dtype=np.float64)
    m.sum_duplicates()
    m.sort_indices()
    m.eliminate_zeros()
    return m


@dataclass
class TriMesh:
    """Mesh2D (mesh.py:33-66) for triangles: CCW cells, edges tail < head in
    lexicographic order, cell_edges / cell_edge_signs per local side
    (0,1), (1,2), (2,0), boundary flags."""

    vertices: np.ndarray
    cells: np.ndarray
    edges: np.ndarray
    cell_edges: np.ndarray
    cell_edge_signs: np.ndarray
    boundary_edge: np.ndarray
    boundary_vertex: np.ndarray

    @property
    def nv(self):
        return len(self.vertices)

    @property
    def nc(self):
        return len(self.cells)

    @property
    def ne(self):
        return len(self.edges)

    def cell_centroids(self):
        return self.vertices[self.cells].mean(axis=1)


def _from_cells(vertices, cells):
    """mesh_from_cells (mesh.py:108-160), vectorised (cells are CCW by construction)."""
    nv = len(vertices)
    a = cells
    t = np.stack([a[:, 0], a[:, 1], a[:, 2]], axis=1)
    h = np.stack([a[:, 1], a[:, 2], a[:, 0]], axis=1)
    lo, hi = np.minimum(t, h), np.maximum(t, h)
    key = lo.astype(np.int64) * nv + hi
    uniq, inv, cnt = np.unique(key.ravel(), return_inverse=True, return_counts=True)
    edges = np.stack([uniq // nv, uniq % nv], axis=1).astype(np.int64)
    cell_edges = inv.reshape(-1, 3).astype(np.int64)
    signs = np.where(t < h, 1, -1).astype(np.int64)
    boundary_edge = cnt == 1
    boundary_vertex = np.zeros(nv, dtype=bool)
    boundary_vertex[edges[boundary_edge].ravel()] = True
    return TriMesh(vertices, cells, edges, cell_edges, signs, boundary_edge, boundary_vertex)


def uniform_tri_mesh0():
    """uniform_tri_mesh(0) (mesh.py:163-182): the unit square, two triangles."""
    xs = np.linspace(0.0, 1.0, 2)
    X, Y = np.meshgrid(xs, xs)
    vertices = np.column_stack([X.ravel(), Y.ravel()])
    return _from_cells(vertices, np.array([(0, 1, 3), (0, 3, 2)], dtype=np.int64))


def refine(mesh):
    """Red refinement (mesh.py:201-257): fine vertices = coarse vertices then
    edge midpoints in edge order; children of cell c in the reference's order;
    coarse_edge_children[E] = (half at the tail, half at the head)."""
    nv, ne = mesh.nv, mesh.ne
    mid = 0.5 * (mesh.vertices[mesh.edges[:, 0]] + mesh.vertices[mesh.edges[:, 1]])
    fv = np.vstack([mesh.vertices, mid])
    v0, v1, v2 = mesh.cells[:, 0], mesh.cells[:, 1], mesh.cells[:, 2]
    m01, m12, m20 = nv + mesh.cell_edges[:, 0], nv + mesh.cell_edges[:, 1], nv + mesh.cell_edges[:, 2]
    kids = np.stack([np.stack([v0, m01, m20], 1), np.stack([m01, v1, m12], 1), np.stack([m20, m12, v2], 1),
                     np.stack([m01, m12, m20], 1)], axis=1).reshape(-1, 3)
    fine = _from_cells(fv, kids)
    nvf = fine.nv
    fkey = fine.edges[:, 0] * nvf + fine.edges[:, 1]
    m = nv + np.arange(ne)
    t, h = mesh.edges[:, 0], mesh.edges[:, 1]
    k0 = np.minimum(t, m) * nvf + np.maximum(t, m)
    k1 = np.minimum(h, m) * nvf + np.maximum(h, m)
    children = np.stack([np.searchsorted(fkey, k0), np.searchsorted(fkey, k1)], axis=1).astype(np.int64)
    return fine, SimpleNamespace(coarse_edge_children=children)


def refinement_chain(base, nrefine):
    meshes, rmaps = [base], []
    for _ in range(nrefine):
        fine, rmap = refine(meshes[-1])
        meshes.append(fine)
        rmaps.append(rmap)
    return meshes, rmaps


def stripes_mu(mesh, fine_level, hi=10.0, lo=0.1):
    """assign_mu_stripes (mesh.py:408-413)."""
    ncols = 2 ** fine_level
    col = np.clip((mesh.cell_centroids()[:, 0] * ncols).astype(int), 0, ncols - 1)
    return np.where(col % 2 == 0, hi, lo)


def _tri_elements(V):
    """tri_element_matrices (fem.py:53-84) for all cells at once; V: (nc, 3, 2)."""
    p0, p1, p2 = V[:, 0], V[:, 1], V[:, 2]
    d1, d2 = p1 - p0, p2 - p0
    area = 0.5 * (d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0])
    if np.any(area <= 0):
        raise ValueError("triangle is degenerate or clockwise")
    g = np.empty((len(V), 3, 2))
    g[:, 0, 0], g[:, 0, 1] = p1[:, 1] - p2[:, 1], p2[:, 0] - p1[:, 0]
    g[:, 1, 0], g[:, 1, 1] = p2[:, 1] - p0[:, 1], p0[:, 0] - p2[:, 0]
    g[:, 2, 0], g[:, 2, 1] = p0[:, 1] - p1[:, 1], p1[:, 0] - p0[:, 0]
    g /= (2.0 * area)[:, None, None]
    S = np.broadcast_to((1.0 / area)[:, None, None], (len(V), 3, 3))
    gram = np.matmul(g, g.transpose(0, 2, 1))
    I2 = (area / 12.0)[:, None, None] * (np.ones((3, 3)) + np.eye(3))
    sides = [(0, 1), (1, 2), (2, 0)]
    M = np.empty((len(V), 3, 3))
    for a, (i, j) in enumerate(sides):
        for b, (k, l) in enumerate(sides):
            M[:, a, b] = (gram[:, j, l] * I2[:, i, k] - gram[:, j, k] * I2[:, i, l]
                          - gram[:, i, l] * I2[:, j, k] + gram[:, i, k] * I2[:, j, l])
    return S, M


def assemble_tri(mesh, mu, beta):
    """assemble(mesh, mu, beta) (fem.py:143-195) with build_gradient
    (fem.py:111-140): returns the reference's CurlCurlSystem fields."""
    if beta < 0:
        raise ValueError("shift must be nonnegative")
    S, M = _tri_elements(mesh.vertices[mesh.cells])
    signs = mesh.cell_edge_signs.astype(np.float64)
    D = signs[:, :, None] * signs[:, None, :]
    S = S * D / mu[:, None, None]
    M = M * D
    ge = mesh.cell_edges
    rows = np.repeat(ge, 3, axis=1).ravel()
    cols = np.tile(ge, (1, 3)).ravel()
    shape = (mesh.ne, mesh.ne)
    As_full = _csr((S.ravel(), (rows, cols)), shape=shape)
    Am_full = _csr((M.ravel(), (rows, cols)), shape=shape)
    free_e, free_v = ~mesh.boundary_edge, ~mesh.boundary_vertex
    free_edges = np.full(mesh.ne, -1, dtype=np.int64)
    free_edges[free_e] = np.arange(free_e.sum())
    free_nodes = np.full(mesh.nv, -1, dtype=np.int64)
    free_nodes[free_v] = np.arange(free_v.sum())
    e = np.flatnonzero(free_e)
    tail, head = mesh.edges[e, 0], mesh.edges[e, 1]
    r = free_edges[e]
    hv, tv = free_nodes[head] >= 0, free_nodes[tail] >= 0
    # per edge: the head entry first, then the tail entry (fem.py:126-134)
    order_r = np.stack([r, r], 1).ravel()
    order_c = np.stack([free_nodes[head], free_nodes[tail]], 1).ravel()
    order_v = np.stack([np.ones(len(e)), -np.ones(len(e))], 1).ravel()
    keep_g = np.stack([hv, tv], 1).ravel()
    G = _csr((order_v[keep_g], (order_r[keep_g], order_c[keep_g])), shape=(int(free_e.sum()), int(free_v.sum())))
    keep = np.flatnonzero(free_edges >= 0)
    As = _csr(As_full[keep][:, keep])
    Am = _csr(Am_full[keep][:, keep])
    As = _csr(0.5 * (As + As.T))
    Am = _csr(0.5 * (Am + Am.T))
    A = _csr(As + beta * Am) if beta > 0 else As.copy()
    A = _csr(0.5 * (A + A.T))
    return SimpleNamespace(A=A, As=As, Am=Am, G=G, beta=float(beta), free_edges=free_edges, free_nodes=free_nodes,
                           n=A.shape[0])


def tri_chain(L, stripes=False, beta=0.01):
    """(meshes, rmaps, system) of the reference tests' tri_chain / tri_setup:
    uniform_tri_mesh(0) refined L times, stripes or constant mu, beta = 0.01."""
    meshes, rmaps = refinement_chain(uniform_tri_mesh0(), L)
    m = meshes[-1]
    mu = stripes_mu(m, L) if stripes else np.ones(m.nc)
    return meshes, rmaps, assemble_tri(m, mu, beta)


def stripes_system(L, beta=0.01):
    """The supplementary 2D benchmark family: stripes mu (10 / 0.1 per grid
    column) on the L-times refined square, beta = 0.01."""
    return tri_chain(L, stripes=True, beta=beta)[2]
