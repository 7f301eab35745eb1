"""Seeded 3D Kuhn-cube curl-curl systems (input generation, not the hot path).

The reference package only meshes 2D domains (``mesh.py``/``fem.py``); every
BASELINE configuration is a unit cube split into n^3 hexahedra x 6 Kuhn
tetrahedra.  This module produces those systems with the reference's own
conventions so the oracle and the GPU path see identical
arrays:

* vertices of the (n+1)^3 grid, lexicographic numbering v = (k(n+1)+j)(n+1)+i;
* six tets per hex, cube-major / permutation-minor, vertex order
  v0 -> v0+e_a -> v0+e_a+e_b -> v0+e_x+e_y+e_z;
* edges stored tail < head, numbered by lexicographic (tail, head) sort
  (as ``mesh_from_cells``, reference mesh.py:128-141);
* Whitney element matrices with unit tangential-integral DoFs, the 3D
  analogue of ``tri_element_matrices`` (reference fem.py:53-84);
* tangential Dirichlet elimination and the discrete gradient exactly as
  ``build_gradient``/``assemble`` (reference fem.py:111-195): edge rows and
  vertex columns on the boundary are removed, G[e, head] = +1,
  G[e, tail] = -1, and A = csr(0.5 (A + A^T)) with A = As + beta Am.

The stiffness weight is mu^{-1} per tet (BASELINE states mu^{-1} directly;
the reference multiplies the element stiffness by 1/mu, fem.py:173).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

__all__ = ["KuhnSystem", "kuhn_mesh", "kuhn_chain", "assemble_kuhn", "config_system", "config_chain",
           "CONFIGS", "rhs", "assemble_kuhn_gpu", "config_system_gpu"]


def _canon(a, shape=None):
    """Canonical CSR (sorted, duplicates summed, exact zeros dropped) — the same
    normal form as the reference's ``csr()`` (sparse.py:58-65)."""
    m = sp.csr_matrix(a, shape=shape, dtype=np.float64)
    m.sum_duplicates()
    m.sort_indices()
    m.eliminate_zeros()
    return m


@dataclass
class KuhnMesh:
    n: int
    vertices: np.ndarray        # (nv, 3)
    tets: np.ndarray            # (nt, 4)
    edges: np.ndarray           # (ne, 2) tail < head
    tet_edges: np.ndarray       # (nt, 6)
    tet_edge_signs: np.ndarray  # (nt, 6)
    boundary_edge: np.ndarray
    boundary_vertex: np.ndarray

    @property
    def nv(self):
        return len(self.vertices)

    @property
    def ne(self):
        return len(self.edges)

    @property
    def nc(self):
        return len(self.tets)

    def tet_centroids(self):
        return self.vertices[self.tets].mean(axis=1)


@dataclass
class KuhnSystem:
    """Same fields as the reference's ``CurlCurlSystem`` (fem.py:30-50)."""

    A: sp.csr_matrix
    As: sp.csr_matrix
    Am: sp.csr_matrix
    G: sp.csr_matrix
    beta: float
    free_edges: np.ndarray
    free_nodes: np.ndarray
    mesh: KuhnMesh = None

    @property
    def n(self):
        return self.A.shape[0]


_LOCAL_EDGES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))


def kuhn_mesh(n, order=None):
    """Unit cube, n^3 hexes, 6 Kuhn tets each (conforming, nested under 2x).

    ``order`` (optional) numbers the vertices: ``order[lex]`` is the number of
    the grid vertex with lexicographic index lex (default: the identity).  Tets
    stay cube-major / permutation-minor over the grid; edges are numbered by
    the (tail, head) sort of the renumbered vertices."""
    if n < 1:
        raise ValueError("n must be >= 1")
    N = n + 1
    idx = np.arange(N ** 3, dtype=np.int64)
    if order is None:
        order = idx
    order = np.asarray(order, dtype=np.int64)
    if order.shape != idx.shape or not np.array_equal(np.sort(order), idx):
        raise ValueError("order must be a permutation of the grid vertices")
    lex_of = np.empty_like(order)
    lex_of[order] = idx                       # vertex number -> lexicographic index
    gi, gj, gk = lex_of % N, (lex_of // N) % N, lex_of // (N * N)
    vertices = np.stack([gi, gj, gk], axis=1).astype(np.float64) / n
    step = np.array([1, N, N * N], dtype=np.int64)
    ck, cj, ci = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    v0 = ((ck * N + cj) * N + ci).ravel()
    far = v0 + step.sum()
    tets = []
    for a, b, _ in itertools.permutations(range(3)):
        tets.append(np.stack([v0, v0 + step[a], v0 + step[a] + step[b], far], axis=1))
    # cube-major / permutation-minor order
    tets = order[np.stack(tets, axis=1).reshape(-1, 4)]

    loc = np.array(_LOCAL_EDGES)
    ends = tets[:, loc]                      # (nt, 6, 2)
    lo, hi = ends.min(axis=2), ends.max(axis=2)
    keys = lo * (N ** 3) + hi
    uniq, inv = np.unique(keys.ravel(), return_inverse=True)
    edges = np.stack([uniq // (N ** 3), uniq % (N ** 3)], axis=1)
    tet_edges = inv.reshape(-1, 6)
    tet_edge_signs = np.where(ends[:, :, 0] < ends[:, :, 1], 1, -1)

    g = np.stack([gi, gj, gk], axis=1)
    on_face = (g == 0) | (g == n)                         # (nv, 3)
    boundary_vertex = on_face.any(axis=1)
    t, h = edges[:, 0], edges[:, 1]
    same_low = (g[t] == g[h]) & (g[t] == 0)
    same_high = (g[t] == g[h]) & (g[t] == n)
    boundary_edge = (same_low | same_high).any(axis=1)
    return KuhnMesh(n, vertices, tets, edges, tet_edges, tet_edge_signs,
                    boundary_edge, boundary_vertex)


def _tet_element(coords):
    """Whitney stiffness/mass (6x6) of one tet; local edge (i,j) basis
    W_ij = l_i grad l_j - l_j grad l_i with unit tangential integral i->j."""
    M4 = np.column_stack([np.ones(4), coords])
    inv = np.linalg.inv(M4)                  # columns: lambda coefficients
    grads = inv[1:, :].T                      # (4, 3) grad lambda_i
    vol = abs(np.linalg.det(M4)) / 6.0
    curls = np.array([2.0 * np.cross(grads[i], grads[j]) for i, j in _LOCAL_EDGES])
    S = vol * curls @ curls.T
    gram = grads @ grads.T
    I2 = vol / 20.0 * (np.ones((4, 4)) + np.eye(4))
    M = np.empty((6, 6))
    for a, (i, j) in enumerate(_LOCAL_EDGES):
        for b, (k, l) in enumerate(_LOCAL_EDGES):
            M[a, b] = (gram[j, l] * I2[i, k] - gram[j, k] * I2[i, l]
                       - gram[i, l] * I2[j, k] + gram[i, k] * I2[j, l])
    return S, M


def assemble_kuhn(mesh, muinv, beta):
    """Assemble A = As(mu^{-1}) + beta Am on the free edges (fem.py:143-195 in 3D)."""
    muinv = np.asarray(muinv, dtype=np.float64)
    if muinv.shape != (mesh.nc,):
        raise ValueError("coefficient field does not match the mesh")
    if np.any(muinv <= 0):
        raise ValueError("coefficient values must be positive")
    if beta < 0:
        raise ValueError("shift must be nonnegative")
    nper = 6
    # all tets of one permutation type are translates: 6 element matrix pairs
    S6, M6 = [], []
    for p in range(nper):
        S, M = _tet_element(mesh.vertices[mesh.tets[p]])
        S6.append(S)
        M6.append(M)
    S6, M6 = np.array(S6), np.array(M6)
    ptype = np.arange(mesh.nc) % nper
    signs = mesh.tet_edge_signs.astype(np.float64)
    D = signs[:, :, None] * signs[:, None, :]
    Se = S6[ptype] * D * muinv[:, None, None]
    Me = M6[ptype] * D
    ge = mesh.tet_edges
    rows = np.repeat(ge, 6, axis=1).ravel()
    cols = np.tile(ge, (1, 6)).ravel()
    shape = (mesh.ne, mesh.ne)
    As_full = _canon((Se.ravel(), (rows, cols)), shape=shape)
    Am_full = _canon((Me.ravel(), (rows, cols)), shape=shape)

    free_e = ~mesh.boundary_edge
    free_v = ~mesh.boundary_vertex
    free_edges = np.full(mesh.ne, -1, dtype=np.int64)
    free_edges[free_e] = np.arange(int(free_e.sum()))
    free_nodes = np.full(mesh.nv, -1, dtype=np.int64)
    free_nodes[free_v] = np.arange(int(free_v.sum()))
    fe = np.flatnonzero(free_e)
    t, h = mesh.edges[fe, 0], mesh.edges[fe, 1]
    r = free_edges[fe]
    hv, tv = free_nodes[h], free_nodes[t]
    gr = np.concatenate([r[hv >= 0], r[tv >= 0]])
    gc = np.concatenate([hv[hv >= 0], tv[tv >= 0]])
    gv = np.concatenate([np.ones(int((hv >= 0).sum())), -np.ones(int((tv >= 0).sum()))])
    G = _canon((gv, (gr, gc)), shape=(int(free_e.sum()), int(free_v.sum())))

    keep = fe
    As = _canon(As_full[keep][:, keep])
    Am = _canon(Am_full[keep][:, keep])
    As = _canon(0.5 * (As + As.T))
    Am = _canon(0.5 * (Am + Am.T))
    A = _canon(As + beta * Am) if beta > 0 else As.copy()
    A = _canon(0.5 * (A + A.T))
    return KuhnSystem(A, As, Am, G, float(beta), free_edges, free_nodes, mesh)


# --------------------------------------------------------------- coefficient fields

def _checkerboard(mesh, k, lo, hi):
    """k^3 checkerboard of sub-cubes; (I+J+K) even -> lo, odd -> hi (per tet centroid)."""
    c = mesh.tet_centroids()
    cell = np.clip((c * k).astype(np.int64), 0, k - 1)
    par = cell.sum(axis=1) % 2
    return np.where(par == 0, lo, hi)


def _block_loguniform(mesh, block, seed, lo_exp=-3.0, hi_exp=3.0):
    """mu^{-1} constant on block^3-hex blocks, 10^U(lo,hi), block-lexicographic draw."""
    nb = mesh.n // block
    rng = np.random.default_rng(seed)
    vals = 10.0 ** rng.uniform(lo_exp, hi_exp, nb ** 3)
    c = mesh.tet_centroids()
    cell = np.clip((c * nb).astype(np.int64), 0, nb - 1)
    return vals[(cell[:, 2] * nb + cell[:, 1]) * nb + cell[:, 0]]


def _inclusions(mesh, count, seed, rmin=0.03, rmax=0.08, inside=1e-6, background=1.0):
    rng = np.random.default_rng(seed)
    radii = rng.uniform(rmin, rmax, count)
    centres = rng.uniform(0.0, 1.0, (count, 3))
    c = mesh.tet_centroids()
    out = np.full(mesh.nc, background)
    for r, x in zip(radii, centres):
        out[np.sum((c - x) ** 2, axis=1) <= r * r] = inside
    return out


# name -> (n, beta, coefficient builder, route); BASELINE.json configs[0..4]
CONFIGS = {
    "c1": dict(n=8, beta=1e-2, field=lambda m: np.ones(m.nc), route="alg"),
    "c2": dict(n=32, beta=1e-3, field=lambda m: _checkerboard(m, 4, 1.0, 1e6), route="alg"),
    "c3": dict(n=64, beta=1e-3, field=lambda m: _block_loguniform(m, 8, seed=0), route="ref"),
    "c4": dict(n=128, beta=1e-4, field=lambda m: _inclusions(m, 64, seed=0), route="alg"),
    "c5": dict(n=256, beta=1e-3, field=lambda m: _checkerboard(m, 8, 1.0, 1e6), route="alg"),
}


@dataclass
class KuhnRefinement:
    """Duck-typed ``RefinementMap`` (reference mesh.py:187-193): the two fine
    children (tail side, head side) of every coarse edge."""

    coarse_edge_children: np.ndarray


def kuhn_chain(n_base, nrefine):
    """Nested Kuhn meshes n_base -> 2 n_base -> ... (``nrefine`` refinements)
    numbered like the reference's ``refine`` (mesh.py:201-257): the fine mesh
    keeps the coarse vertices first, in coarse order, followed by the midpoint
    of every coarse edge in coarse edge order (every fine vertex is a coarse
    vertex or the midpoint of exactly one Kuhn edge, since all diagonals point
    the same way).  Returns (meshes coarse -> fine, refinement maps)."""
    mesh = kuhn_mesh(n_base)
    meshes, rmaps = [mesh], []
    n = n_base
    for _ in range(nrefine):
        N = n + 1
        lex = np.arange(N ** 3, dtype=np.int64)
        cur_lex_of = np.empty(N ** 3, dtype=np.int64)
        cur_lex_of[_vertex_numbers(mesh)] = lex
        g = np.stack([cur_lex_of % N, (cur_lex_of // N) % N, cur_lex_of // (N * N)], axis=1)  # by vertex number
        t, h = mesh.edges[:, 0], mesh.edges[:, 1]
        fine_g = np.vstack([2 * g, g[t] + g[h]])           # fine grid coords of fine vertex numbers
        n2, N2 = 2 * n, 2 * n + 1
        if len(fine_g) != N2 ** 3:
            raise AssertionError("Kuhn refinement does not cover the fine grid")
        flex = (fine_g[:, 2] * N2 + fine_g[:, 1]) * N2 + fine_g[:, 0]
        order = np.empty(N2 ** 3, dtype=np.int64)
        order[flex] = np.arange(N2 ** 3, dtype=np.int64)
        fine = kuhn_mesh(n2, order)
        keys = {(int(a), int(b)): e for e, (a, b) in enumerate(fine.edges)}
        mid = mesh.nv + np.arange(mesh.ne)
        kids = np.empty((mesh.ne, 2), dtype=np.int64)
        for e in range(mesh.ne):
            m = int(mid[e])
            kids[e, 0] = keys[(min(int(t[e]), m), max(int(t[e]), m))]
            kids[e, 1] = keys[(min(int(h[e]), m), max(int(h[e]), m))]
        meshes.append(fine)
        rmaps.append(KuhnRefinement(kids))
        mesh, n = fine, n2
    return meshes, rmaps


def _vertex_numbers(mesh):
    """order[lex] of a KuhnMesh, recovered from its vertex coordinates."""
    N = mesh.n + 1
    g = np.rint(mesh.vertices * mesh.n).astype(np.int64)
    lex = (g[:, 2] * N + g[:, 1]) * N + g[:, 0]
    order = np.empty(N ** 3, dtype=np.int64)
    order[lex] = np.arange(N ** 3, dtype=np.int64)
    return order


def config_chain(name, n_fine=None, n_base=None):
    """A config on a nested chain (the "ref" route): (system, meshes, rmaps).
    Defaults: BASELINE's chain for the config (c3: 8 -> 16 -> 32 -> 64)."""
    cfg = CONFIGS[name]
    n_fine = cfg["n"] if n_fine is None else n_fine
    n_base = 8 if n_base is None else n_base
    nref = 0
    while n_base * 2 ** nref < n_fine:
        nref += 1
    if n_base * 2 ** nref != n_fine:
        raise ValueError("n_fine must be n_base * 2^k")
    meshes, rmaps = kuhn_chain(n_base, nref)
    fine = meshes[-1]
    return assemble_kuhn(fine, cfg["field"](fine), cfg["beta"]), meshes, rmaps


def config_system(name, n=None):
    """Build the system of a BASELINE config (optionally at another size n)."""
    cfg = CONFIGS[name]
    mesh = kuhn_mesh(cfg["n"] if n is None else n)
    return assemble_kuhn(mesh, cfg["field"](mesh), cfg["beta"])


# --------------------------------------------------------------- GPU assembly

class _KuhnCells:
    """The cells of ``kuhn_mesh(n)`` (lexicographic numbering) without its edge
    table: enough for the coefficient fields (``n``, ``nc``, ``tet_centroids``),
    with the centroids computed from the same float coordinates in the same
    order, hence bit-identical to ``KuhnMesh.tet_centroids``."""

    def __init__(self, n):
        self.n = int(n)

    @property
    def nc(self):
        return 6 * self.n ** 3

    def tet_corners(self):
        n = self.n
        ck, cj, ci = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
        g0 = np.stack([ci.ravel(), cj.ravel(), ck.ravel()], axis=1)         # hex lower corners, cube-major
        eye = np.eye(3, dtype=np.int64)
        corners = []
        for a, b, _ in itertools.permutations(range(3)):
            corners.append(np.stack([g0, g0 + eye[a], g0 + eye[a] + eye[b], g0 + 1], axis=1))
        return np.stack(corners, axis=1).reshape(-1, 4, 3)                  # (nt, 4, 3) grid coords

    def tet_centroids(self):
        return (self.tet_corners().astype(np.float64) / self.n).mean(axis=1)


def _element_matrices(n):
    """S, M of the six tet shapes of hex 0, exactly as assemble_kuhn computes them."""
    N = n + 1
    lex = np.arange(N ** 3, dtype=np.int64)
    g = np.stack([lex % N, (lex // N) % N, lex // (N * N)], axis=1)
    verts = g.astype(np.float64) / n
    step = np.array([1, N, N * N], dtype=np.int64)
    S6, M6 = [], []
    for a, b, _ in itertools.permutations(range(3)):
        tet = np.array([0, step[a], step[a] + step[b], step.sum()])
        S, M = _tet_element(verts[tet])
        S6.append(S)
        M6.append(M)
    return np.ascontiguousarray(S6, np.float64), np.ascontiguousarray(M6, np.float64)


def assemble_kuhn_gpu(n, muinv, beta, device=0):
    """``assemble_kuhn(kuhn_mesh(n), muinv, beta)`` on the GPU (csrc/kuhn.cu):
    same pattern, G and index maps; an entry of A can differ from the host
    assembly in the last bit (duplicates are summed in tet order here, in the
    order of scipy's unstable sort there).  ``As``/``Am`` are not returned."""
    import ctypes as C

    from .multilevel import _Device
    from . import _lib

    muinv = np.ascontiguousarray(muinv, dtype=np.float64)
    if muinv.shape != (6 * n ** 3,):
        raise ValueError("coefficient field does not match the mesh")
    if np.any(muinv <= 0):
        raise ValueError("coefficient values must be positive")
    if beta < 0:
        raise ValueError("shift must be nonnegative")
    S6, M6 = _element_matrices(n)
    dev = _Device(device)
    sizes = np.zeros(6, np.int64)
    dev.check(dev.lib.hcamg_kuhn_assemble(dev.h, int(n), _lib.ptr(muinv), C.c_double(beta), _lib.ptr(S6),
                                          _lib.ptr(M6), _lib.ptr(sizes)))
    nfe, nnz_a, nfv, nnz_g, ne, nv = (int(x) for x in sizes)
    ap, ai, av = np.empty(nfe + 1, np.int64), np.empty(nnz_a, np.int32), np.empty(nnz_a, np.float64)
    gp, gi, gv = np.empty(nfe + 1, np.int64), np.empty(nnz_g, np.int32), np.empty(nnz_g, np.float64)
    fe, fv = np.empty(ne, np.int64), np.empty(nv, np.int64)
    dev.check(dev.lib.hcamg_kuhn_export(dev.h, _lib.ptr(ap), _lib.ptr(ai), _lib.ptr(av), _lib.ptr(gp), _lib.ptr(gi),
                                        _lib.ptr(gv), _lib.ptr(fe), _lib.ptr(fv)))
    A = sp.csr_matrix((av, ai, ap), shape=(nfe, nfe))
    G = sp.csr_matrix((gv, gi, gp), shape=(nfe, nfv))
    return KuhnSystem(A, None, None, G, float(beta), fe, fv, None)


def config_system_gpu(name, n=None, device=0):
    """``config_system`` with the assembly on the GPU ("alg" configs, lexicographic numbering)."""
    cfg = CONFIGS[name]
    n = cfg["n"] if n is None else n
    return assemble_kuhn_gpu(n, cfg["field"](_KuhnCells(n)), cfg["beta"], device=device)


def rhs(n, seed=0):
    """Seeded uniform[-1,1] right-hand side (seed recorded as 0 by default)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)
