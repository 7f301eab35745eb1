"""CPU oracle for the AMG-PCG hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy/scipy, the reference algorithm of
arXiv 2602.23613's ``hcurl_amg`` package for the path named by
BASELINE.json's north star: ``build_hierarchy`` ("alg" and "ref" routes),
``vcycle``, ``pcg``, ``amg_solve`` and ``operator_complexity``.  It is the
checker the GPU product is compared against; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import it.  The product path (``paper_2602_23613_b200``) never calls it.

The floating-point parts use the very same scipy/numpy/LAPACK primitives as
the reference (the reference's arithmetic lives in scipy 1.18.1 sparsetools,
scipy.sparse.csgraph and numpy 2.3.5 / scipy-openblas 0.3.30), so on the same
inputs this restatement is bit-identical to the reference; the combinatorial
parts (strong adjacency, greedy C/F, matching) are reorganised (vectorised
masks, a lazy max-heap instead of an O(N) argmax per pick) but keep the
reference's exact tie-break semantics.  Pinning: ``tests/test_oracle_golden.py``
checks every function against fixtures produced by the reference itself
(``tests/golden/make_golden.py``, run in the build container where
``/root/reference`` is importable).

Citations are ``file:line`` in ``/root/reference/pkg/src/hcurl_amg``.
Known deliberate divergence: the reference factors components / coarsest
matrices above 4096 DoFs with a pure-Python up-looking sparse Cholesky
(sparse.py:212-273); this oracle always uses the dense LAPACK path (the same
factorization, different roundoff) — the survey's "raised cutoff" run.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components, reverse_cuthill_mckee

PIVOT_RTOL = 1e-13                  # sparse.py:30
INV_SQRT2 = 1.0 / np.sqrt(2.0)      # splitting.py:47 (0x3FE6A09E667F3BCC)


class NotPositiveDefiniteError(RuntimeError):
    """Cholesky breakdown with the failing pivot (sparse.py:50-55)."""

    def __init__(self, pivot, message=None):
        self.pivot = int(pivot)
        super().__init__(message or f"matrix is not positive definite (pivot {pivot})")


# ----------------------------------------------------------------------------- sparse core

def canon(a, shape=None):
    """Canonical CSR: sorted, duplicates summed, exact zeros dropped (sparse.py:58-65)."""
    m = sp.csr_matrix(a, shape=shape, dtype=np.float64)
    m.sum_duplicates()
    m.sort_indices()
    m.eliminate_zeros()
    return m


def max_abs(M):
    return float(np.abs(M.data).max()) if M.nnz else 0.0


def symmetric_part(M):
    """canon(0.5 (M + M^T)) — used by nodal_dual and galerkin (splitting.py:133, sparse.py:122)."""
    return canon(0.5 * (M + M.T))


def galerkin(P, A):
    """P^T A P symmetrised (sparse.py:113-122).  For a HybridP (large
    component, see harmonic_interp) the Schur form is used:
    P^T A P = P_s^T A P_s - W'^T A_GG^{-1} W' = sym(P_s^T A P_s) - sym(W'^T Z)
    with W' = A[rows, :] P_s the block's right-hand side (exact in exact
    arithmetic; the dropped residual term Z^T (W' - A_GG Z) is ~1e-15 of A_c,
    measured at n = 8 and 16 against the reference's P^T (A P))."""
    if A.shape[0] != A.shape[1] or A.shape[0] != P.shape[0]:
        raise ValueError(f"dimension mismatch: P {P.shape}, A {A.shape}")
    if isinstance(P, HybridP):
        S = symmetric_part(P.Ps.T @ (A @ P.Ps)).toarray()
        D = np.asarray(P.Wg.T @ P.Z)                      # (cols x cols)
        D = 0.5 * (D + D.T)
        S[np.ix_(P.cols, P.cols)] -= D
        return canon(S)
    return symmetric_part(P.T @ (A @ P))


def _pivot_loop(Ad, floor):
    """Column Cholesky naming the first failing pivot (sparse.py:172-185)."""
    n = Ad.shape[0]
    L = np.zeros_like(Ad)
    for j in range(n):
        d = Ad[j, j] - L[j, :j] @ L[j, :j]
        if not np.isfinite(d) or d <= floor:
            raise NotPositiveDefiniteError(j)
        L[j, j] = np.sqrt(d)
        if j + 1 < n:
            L[j + 1:, j] = (Ad[j + 1:, j] - L[j + 1:, :j] @ L[j, :j]) / L[j, j]
    return L


def dense_chol(Ad):
    """LAPACK lower Cholesky + relative pivot floor (sparse.py:188-209)."""
    if Ad.shape[0] == 0:
        return np.zeros((0, 0))
    dg = np.diag(Ad)
    scale = float(np.abs(dg).max()) if len(dg) else 0.0
    try:
        L = np.linalg.cholesky(Ad)
    except np.linalg.LinAlgError:
        _pivot_loop(Ad, PIVOT_RTOL * scale)
        raise
    piv = np.diag(L) ** 2
    if piv.min() <= PIVOT_RTOL * scale:
        raise NotPositiveDefiniteError(int(np.argmin(piv)),
                                       f"pivot {piv.min():.3e} below the breakdown floor "
                                       "(near-singular block)")
    return L


@dataclass
class Factor:
    """Permuted dense Cholesky of the coarsest operator (sparse.py:146-165, 276-301)."""

    perm: np.ndarray
    L: np.ndarray

    @property
    def n(self):
        return self.L.shape[0]


def factor_coarsest(A):
    if A.shape[0] != A.shape[1]:
        raise ValueError("matrix must be square")
    asym, scale = max_abs(canon(A - A.T)), max_abs(A)
    if scale > 0 and asym > 1e-12 * scale:
        raise ValueError(f"matrix not symmetric: asymmetry {asym:.3e}")
    n = A.shape[0]
    if n == 0:
        return Factor(np.zeros(0, dtype=np.int64), np.zeros((0, 0)))
    perm = np.asarray(reverse_cuthill_mckee(A, symmetric_mode=True), dtype=np.int64)
    L = dense_chol(A[perm][:, perm].tocsr().toarray())
    # the reference stores csr(L) and densifies it again: same values
    return Factor(perm, canon(L).toarray())


def solve_coarsest(f, b):
    """sparse.py:304-321 (dense path)."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape[0] != f.n:
        raise ValueError(f"dimension mismatch: factor {f.n}, rhs {b.shape}")
    if f.n == 0:
        return b.copy()
    y = scipy.linalg.solve_triangular(f.L, b[f.perm], lower=True)
    xp = scipy.linalg.solve_triangular(f.L.T, y, lower=False)
    x = np.empty_like(xp)
    x[f.perm] = xp
    return x


# ----------------------------------------------------------------------------- splitting

@dataclass(frozen=True)
class Pair:
    """ExteriorPair (splitting.py:50-57)."""

    dof1: int
    dof2: int
    sign1: int
    sign2: int
    tail: int
    mid: int
    head: int


@dataclass
class Split:
    """Splitting (splitting.py:60-85)."""

    pairs: list
    interior_dofs: np.ndarray
    n: int
    dof_edges: np.ndarray = None
    pair_mesh_edges: np.ndarray = None
    coarse_nodes: np.ndarray = None

    @property
    def n_pairs(self):
        return len(self.pairs)


def augment(G):
    """augment_gradient (splitting.py:100-125) -> (Gtilde, boundary column ids)."""
    G = canon(G)
    per_row = np.diff(G.indptr)
    if np.any(per_row > 2):
        raise ValueError(f"row {int(np.argmax(per_row > 2))} has more than 2 nonzeros")
    if G.nnz and np.any(np.abs(G.data) != 1.0):
        raise ValueError("gradient entries must be +-1")
    lone = np.flatnonzero(per_row == 1)
    m = G.shape[1]
    if lone.size == 0:
        return G, np.zeros(0, dtype=np.int64)
    extra = canon((-G.data[G.indptr[lone]], (lone, np.arange(lone.size))),
                  shape=(G.shape[0], lone.size))
    return canon(sp.hstack([G, extra])), (m + np.arange(lone.size)).astype(np.int64)


def nodal_dual(A, Gt):
    """G~^T (A G~), symmetrised (splitting.py:128-133)."""
    if A.shape[1] != Gt.shape[0]:
        raise ValueError(f"dimension mismatch: A {A.shape}, Gtilde {Gt.shape}")
    return symmetric_part(Gt.T @ (A @ Gt))


def _rows_of(M):
    return np.repeat(np.arange(M.shape[0]), np.diff(M.indptr))


def strong_lists(An, theta):
    """Strong mask per stored entry (splitting.py:136-155), vectorised.

    Entry (i, j), j != i, is strong iff |a_ij| >= theta * max_{k != i} |a_ik|.
    Returns (strong CSR pattern, its transpose = strong_to lists).
    """
    rows = _rows_of(An)
    off = An.indices != rows
    mag = np.where(off, np.abs(An.data), -np.inf)
    rmax = np.full(An.shape[0], -np.inf)
    np.maximum.at(rmax, rows, mag)
    mask = off & (np.abs(An.data) >= theta * rmax[rows])
    S = sp.csr_matrix((np.ones(int(mask.sum())), (rows[mask], An.indices[mask])),
                      shape=An.shape)
    S.sort_indices()
    ST = S.T.tocsr()
    ST.sort_indices()
    return S, ST


def neighbours(An):
    """Stored off-diagonal pattern per row (splitting.py:158-165)."""
    rows = _rows_of(An)
    keep = An.indices != rows
    cnt = np.bincount(rows[keep], minlength=An.shape[0])
    ptr = np.concatenate([[0], np.cumsum(cnt)])
    return ptr, An.indices[keep].astype(np.int64)


UNASSIGNED, COARSE, FINE = 0, 1, 2


def greedy_cf(An, c_init=(), f_init=(), theta=0.25):
    """classical_cf (splitting.py:171-211) with a lazy max-heap.

    The reference picks argmax(measure over unassigned), lowest index on ties;
    a heap keyed (-measure, index) with stale-entry skipping yields the same
    sequence of picks because measures only ever grow.
    """
    n = An.shape[0]
    c_init = np.asarray(list(c_init), dtype=np.int64)
    f_init = np.asarray(list(f_init), dtype=np.int64)
    if len(np.intersect1d(c_init, f_init)) > 0:
        raise ValueError("initial coarse and fine sets overlap")
    state = np.zeros(n, dtype=np.int8)
    state[c_init] = COARSE
    state[f_init] = FINE
    S, ST = strong_lists(An, theta)
    nptr, nidx = neighbours(An)
    # measure[i] = number of strong neighbours of i already fine
    measure = np.asarray(S @ (state == FINE).astype(np.float64)).astype(np.int64)
    heap = [(-int(measure[i]), int(i)) for i in np.flatnonzero(state == UNASSIGNED)]
    heapq.heapify(heap)
    st_ptr, st_idx = ST.indptr, ST.indices
    while heap:
        negm, i = heapq.heappop(heap)
        if state[i] != UNASSIGNED or -negm != measure[i]:
            continue
        state[i] = COARSE
        for j in nidx[nptr[i]:nptr[i + 1]]:
            if state[j] != UNASSIGNED:
                continue
            state[j] = FINE
            for k in st_idx[st_ptr[j]:st_ptr[j + 1]]:
                measure[k] += 1
                if state[k] == UNASSIGNED:
                    heapq.heappush(heap, (-int(measure[k]), int(k)))
    return np.flatnonzero(state == COARSE), np.flatnonzero(state == FINE)


def nodal_split(A, Gt, bcols, theta=0.25):
    """nodal_cf (splitting.py:214-229) -> (c_G, F, A_nodal)."""
    An = nodal_dual(A, Gt)
    bcols = np.asarray(bcols, dtype=np.int64)
    nptr, nidx = neighbours(An)
    touched = np.concatenate([nidx[nptr[b]:nptr[b + 1]] for b in bcols]) if len(bcols) else np.zeros(0, np.int64)
    f_init = np.setdiff1d(np.unique(touched), bcols)
    C, F = greedy_cf(An, c_init=bcols, f_init=f_init, theta=theta)
    return np.setdiff1d(C, bcols), F, An


def edge_table(Gt):
    """(min node, max node) -> (row, value at min, value at max) over two-entry
    rows, later rows winning (splitting.py:232-243)."""
    table = {}
    two = np.flatnonzero(np.diff(Gt.indptr) == 2)
    lo = Gt.indptr[two]
    for r, a, b, va, vb in zip(two.tolist(), Gt.indices[lo].tolist(), Gt.indices[lo + 1].tolist(),
                               Gt.data[lo].tolist(), Gt.data[lo + 1].tolist()):
        table[(a, b)] = (r, va, vb)
    return table


def algebraic_split(A, G, theta=0.25, dof_edges=None):
    """build_algebraic_splitting (splitting.py:246-298).

    The reference scans, for each coarse i (ascending), every coarse j > i at
    nodal distance two and every common nodal neighbour k (both ascending),
    accepting the first k whose path edges (i,k), (k,j) exist in G~, are
    distinct and still available and whose mid node is unused.  Only triples
    whose two path edges exist can be accepted, so the same ordered candidate
    list is generated from the edge graph instead: k over the edge-neighbours
    of i, j over the edge-neighbours of k, filtered by the nodal-graph
    adjacency k in N(i) & N(j), then sorted by (j, k).  Same triples, same
    order, same acceptance rule; O(edge degree^2) per node instead of
    O(nodal degree^2), which matters on dense coarse levels.
    """
    Gt, bcols = augment(G)
    c_G, _, An = nodal_split(A, Gt, bcols, theta)
    coarse = np.union1d(c_G, bcols)
    nn = An.shape[0]
    in_b = np.zeros(nn, dtype=bool)
    in_b[bcols] = True
    is_c = np.zeros(nn, dtype=bool)
    is_c[coarse] = True
    nptr, nidx = neighbours(An)
    table = edge_table(Gt)           # (min, max) -> (last row, value at min, value at max)
    eadj = [[] for _ in range(nn)]
    for (u, v) in table:
        eadj[u].append(v)
        eadj[v].append(u)
    eadj = [sorted(set(e)) for e in eadj]

    def adjacent(u, v):
        row = nidx[nptr[u]:nptr[u + 1]]
        pos = np.searchsorted(row, v)
        return pos < row.size and row[pos] == v

    free = np.ones(A.shape[0], dtype=bool)
    used_mid = np.zeros(nn, dtype=bool)
    pairs = []
    for i in coarse.tolist():
        cand = set()
        for k in eadj[i]:
            if not adjacent(i, k):
                continue
            for j in eadj[k]:
                if j > i and is_c[j] and not (in_b[i] and in_b[j]) and adjacent(j, k):
                    cand.add((j, k))
        last_j = -1
        for j, k in sorted(cand):
            if j == last_j or used_mid[k]:
                continue
            e1 = table[(i, k) if i < k else (k, i)]
            e2 = table[(k, j) if k < j else (j, k)]
            if e1[0] == e2[0] or not (free[e1[0]] and free[e2[0]]):
                continue
            g1 = e1[1] if k < i else e1[2]      # Gtilde[dof1, k]
            g2 = e2[1] if k < j else e2[2]      # Gtilde[dof2, k]
            pairs.append(Pair(e1[0], e2[0], int(np.sign(g1)), int(-np.sign(g2)), i, k, j))
            free[e1[0]] = free[e2[0]] = False
            used_mid[k] = True
            last_j = j
    return Split(pairs, np.flatnonzero(free), A.shape[0], dof_edges=dof_edges, coarse_nodes=c_G)


def refinement_split(coarse_mesh, fine_mesh, rmap, edge_to_dof, n):
    """build_refinement_splitting (splitting.py:301-330)."""
    free = np.ones(n, dtype=bool)
    dof_edges = np.full(n, -1, dtype=np.int64)
    live = np.flatnonzero(edge_to_dof >= 0)
    dof_edges[edge_to_dof[live]] = live
    pairs, owners = [], []
    fe = np.asarray(fine_mesh.edges)
    for E in range(coarse_mesh.ne):
        c1, c2 = (int(c) for c in rmap.coarse_edge_children[E])
        d1, d2 = int(edge_to_dof[c1]), int(edge_to_dof[c2])
        if d1 < 0 or d2 < 0:
            continue
        t, h = (int(v) for v in coarse_mesh.edges[E])
        mid = int(np.intersect1d(fe[c1], fe[c2])[0])
        pairs.append(Pair(d1, d2, 1 if fe[c1][1] == mid else -1, 1 if fe[c2][0] == mid else -1,
                          t, mid, h))
        owners.append(E)
        free[d1] = free[d2] = False
    return Split(pairs, np.flatnonzero(free), n, dof_edges=dof_edges,
                 pair_mesh_edges=np.array(owners, dtype=np.int64))


def restriction(split):
    """R of realize_RS (splitting.py:333-347, 363-372)."""
    npair = split.n_pairs
    rows = np.repeat(np.arange(npair), 2)
    cols = np.array([d for p in split.pairs for d in (p.dof1, p.dof2)], dtype=np.int64)
    vals = np.array([s * INV_SQRT2 for p in split.pairs for s in (p.sign1, p.sign2)])
    return canon((vals, (rows, cols)), shape=(npair, split.n))


def dump(split):
    """dump_splitting text (splitting.py:375-380): parity-fixture format."""
    out = [f"n {split.n}"]
    out += [f"{p.tail} {p.mid} {p.head} {p.dof1} {p.sign1} {p.dof2} {p.sign2}" for p in split.pairs]
    return "\n".join(out) + "\n"


# ----------------------------------------------------------------------------- transfer

def components(A_II):
    """Connected components as sorted index arrays (transfer.py:49-52)."""
    ncomp, lab = connected_components(A_II, directed=False)
    order = np.argsort(lab, kind="stable")
    cuts = np.searchsorted(lab[order], np.arange(ncomp + 1))
    return [order[cuts[c]:cuts[c + 1]] for c in range(ncomp)]


def coarse_grad(R, G, mode, coarse_nodes=None):
    """coarse_gradient (transfer.py:55-74) -> (Gc, kept columns)."""
    RG = canon(R @ G)
    cnt = np.diff(RG.tocsc().indptr)
    if mode == "refinement":
        cols = np.flatnonzero(cnt > 0)
    elif mode == "algebraic":
        if coarse_nodes is None:
            raise ValueError("algebraic mode needs the coarse nodal set")
        cols = np.asarray(sorted(coarse_nodes), dtype=np.int64)
        cols = cols[cnt[cols] > 0]
    else:
        raise ValueError(f"unknown mode {mode!r}")
    Gc = canon(RG[:, cols]) if len(cols) else sp.csr_matrix((RG.shape[0], 0))
    return Gc, cols


# ----------------------------------------------------------------------------- large components

DENSE_COMPONENT_CUTOFF = 4096   # transfer.py:35
ENVELOPE_NB = 1024


@dataclass
class EnvelopeFactor:
    """Lower Cholesky factor of P A P^T (P = reverse Cuthill-McKee, the order the
    reference's cholesky() applies above its dense cutoff, sparse.py:276-301)
    kept in NB-row block rows restricted to the block envelope: block row I
    holds columns [j0[I] NB, (I + 1) NB).  Cholesky fill never leaves the
    envelope, so this is the reference's factorisation (its up-looking sparse
    loop, sparse.py:212-273, with the same pivot floor), computed with LAPACK
    / BLAS-3 on dense tiles instead of per-entry Python.  ``inv[I]`` is the
    inverse of the diagonal block (triangular solves become GEMMs)."""

    perm: np.ndarray
    nb: int
    j0: np.ndarray
    rows: list            # block row I: (rows_I, (I - j0[I] + 1) nb) array
    inv: list             # inverse of the diagonal block of block row I

    @property
    def n(self):
        return len(self.perm)

    def block(self, I, J):
        nb = self.nb
        c = (J - self.j0[I]) * nb
        return self.rows[I][:, c:c + nb]


def envelope_cholesky(Acc, nb=None):
    """RCM + blocked left-looking Cholesky inside the block envelope (see
    EnvelopeFactor); raises NotPositiveDefiniteError with the failing pivot in
    the factored order, as the reference's sparse path does."""
    nb = nb or ENVELOPE_NB
    A = canon(Acc)
    n = A.shape[0]
    perm = np.asarray(reverse_cuthill_mckee(A, symmetric_mode=True), dtype=np.int64)
    Ap = A[perm][:, perm].tocsr()
    Ap.sort_indices()
    T = -(-n // nb)
    first = np.minimum(Ap.indices[Ap.indptr[:-1]], np.arange(n))  # first column per row (sorted rows)
    j0 = np.array([first[I * nb:(I + 1) * nb].min() // nb for I in range(T)], dtype=np.int64)
    scale = float(np.abs(A.diagonal()).max()) if n else 0.0
    floor = PIVOT_RTOL * scale
    potrf, trtri = scipy.linalg.lapack.dpotrf, scipy.linalg.lapack.dtrtri
    rows, inv = [], []
    for I in range(T):
        r0, r1 = I * nb, min(n, (I + 1) * nb)
        c0 = j0[I] * nb
        R = np.zeros((r1 - r0, (I - j0[I] + 1) * nb))
        blk = Ap[r0:r1]
        rr = np.repeat(np.arange(r1 - r0), np.diff(blk.indptr))
        keep = blk.indices <= rr + r0
        R[rr[keep], blk.indices[keep] - c0] = blk.data[keep]
        for J in range(j0[I], I + 1):
            cJ = (J - j0[I]) * nb
            k0 = max(j0[I], j0[J]) * nb                     # common columns of block rows I and J
            X = R[:, cJ:cJ + nb]
            if k0 < J * nb:
                RJ = rows[J] if J < I else R
                X[:, :RJ.shape[0]] -= R[:, k0 - c0:J * nb - c0] @ RJ[:, k0 - j0[J] * nb:J * nb - j0[J] * nb].T
            if J < I:
                R[:, cJ:cJ + nb] = X @ inv[J].T                  # L_IJ = A_IJ L_JJ^{-T}
            else:
                m = r1 - r0
                D = np.tril(X[:, :m])
                D = D + np.tril(D, -1).T
                LII, info = potrf(D, lower=1, clean=1)
                if info != 0:
                    _pivot_loop(D, floor)                     # names the failing pivot
                    raise NotPositiveDefiniteError(r0 + info - 1)
                piv = np.diag(LII) ** 2
                if piv.min() <= floor:
                    raise NotPositiveDefiniteError(r0 + int(np.argmin(piv)))
                R[:, cJ:cJ + m] = LII
                R[:, cJ + m:] = 0.0
                Li, info = trtri(np.ascontiguousarray(LII), lower=1)
                inv.append(np.tril(Li))
        rows.append(R)
    return EnvelopeFactor(perm, nb, j0, rows, inv)


def envelope_solve(F, Bp, active=None):
    """Solve (L L^T) Z = Bp in place for a dense right-hand side already in the
    factored row order.  ``active[I]``: number of leading columns that can be
    nonzero in block row I of the forward solve (columns sorted by their first
    nonzero row: the staircase of L^{-1} Bp)."""
    nb, T = F.nb, len(F.rows)
    m = Bp.shape[1]
    act = np.full(T, m, dtype=np.int64) if active is None else active
    for I in range(T):                                    # Y = L^{-1} Bp
        r0, r1 = I * nb, min(F.n, (I + 1) * nb)
        a = int(act[I])
        if a == 0:
            continue
        c0 = F.j0[I] * nb
        X = Bp[r0:r1, :a]
        if c0 < r0:
            X -= F.rows[I][:, :r0 - c0] @ Bp[c0:r0, :a]
        Bp[r0:r1, :a] = F.inv[I] @ X
    for I in range(T - 1, -1, -1):                        # Z = L^{-T} Y
        r0, r1 = I * nb, min(F.n, (I + 1) * nb)
        X = Bp[r0:r1]
        for K in range(I + 1, T):
            if F.j0[K] <= I:
                k0, k1 = K * nb, min(F.n, (K + 1) * nb)
                X -= F.block(K, I)[:, :r1 - r0].T @ Bp[k0:k1]
        Bp[r0:r1] = F.inv[I].T @ X
    return Bp


class HybridP:
    """P = P_s - S Z: a sparse part plus one dense block (rows x cols of P),
    the interpolation of a component too large for a CSR P (SURVEY.md F3:
    35 GB of dense rows at config 2).  Supports ``P @ e`` and ``P.T @ r``,
    the two products the V-cycle uses (multilevel.py:183)."""

    def __init__(self, Ps, Z, rows, cols):
        self.Ps, self.Z, self.rows, self.cols = Ps, Z, rows, cols
        self.shape = Ps.shape

    @property
    def nnz(self):
        return self.Ps.nnz + self.Z.size

    def __matmul__(self, e):
        y = self.Ps @ e
        y[self.rows] -= self.Z @ e[self.cols]
        return y

    @property
    def T(self):
        outer = self

        class _T:
            shape = (outer.shape[1], outer.shape[0])

            def __matmul__(self, r):
                out = outer.Ps.T @ r
                out[outer.cols] -= outer.Z.T @ r[outer.rows]
                return out
        return _T()


@dataclass
class Transfer:
    P: sp.csr_matrix
    R: sp.csr_matrix
    Gc: sp.csr_matrix
    cols: np.ndarray
    Z_blocks: list = field(default_factory=list)   # (interior rows, keep cols, Z) per component


def _alt_component_solve(Acc, rhs):
    """Reproducibility-floor solver: LU of the reversed-order block (another
    valid fp64 algorithm).  Used only to MEASURE how far
    two correct fp64 implementations drift apart, never as the oracle."""
    rev = np.arange(Acc.shape[0])[::-1]
    lu = scipy.linalg.lu_factor(Acc[np.ix_(rev, rev)])
    Z = np.empty_like(rhs)
    Z[rev] = scipy.linalg.lu_solve(lu, rhs[rev])
    return Z


def harmonic_interp(A, split, mode="refinement", G=None, floor_solver=False, large="dense"):
    """sparse_ideal_interp (transfer.py:77-122): P = R^T - S_I A_II^{-1} S_I^T A R^T.

    ``large="dense"`` (default, the pinned path): every component is solved
    with dense LAPACK.  ``large="envelope"``: a component above the reference's
    4096-DoF cutoff is factored by RCM + envelope Cholesky (the reference's own
    route there, sparse.py:276-301) and kept as the dense block of a
    HybridP instead of entering the CSR P (config 2: 4.4e9 entries).  Used by
    bench.py's CPU reference arm; at that size the reference itself cannot run,
    so this path is checked against the dense path at n = 16 only."""
    R = restriction(split)
    Rt = canon(R.T)
    inner = split.interior_dofs
    blocks = []
    if len(inner) == 0 or split.n_pairs == 0:
        P = Rt
    else:
        Ai = A[inner, :]
        W = canon(Ai @ Rt)
        A_II = canon(Ai[:, inner])
        ri, ci, vi = [], [], []
        hybrid = None
        for comp in components(A_II):
            Wc = W[comp, :].tocsc()
            keep = np.flatnonzero(np.diff(Wc.indptr) > 0)
            if keep.size == 0:
                continue
            if large == "envelope" and len(comp) > DENSE_COMPONENT_CUTOFF and hybrid is None:
                F = envelope_cholesky(A_II[comp][:, comp])
                Wp = Wc[:, keep].tocsr()[F.perm]
                first = np.full(len(keep), len(comp), dtype=np.int64)   # first (factored) row per column
                coo = Wp.tocoo()
                np.minimum.at(first, coo.col, coo.row)
                colperm = np.argsort(first, kind="stable")
                active = np.searchsorted(first[colperm], (np.arange(len(F.rows)) + 1) * F.nb)
                Z = np.asarray(Wp[:, colperm].todense())
                envelope_solve(F, Z, active)
                hybrid = (inner[comp[F.perm]], keep[colperm], Z, Wp[:, colperm].tocsr())
                continue
            Acc = A_II[comp][:, comp].toarray()
            rhs = np.asarray(Wc[:, keep].todense())
            if floor_solver:
                Z = _alt_component_solve(Acc, rhs)
            else:
                Z = scipy.linalg.cho_solve((dense_chol(Acc), True), rhs)
            blocks.append((inner[comp], keep, Z))
            nzr, nzc = np.nonzero(Z)
            ri.append(inner[comp[nzr]])
            ci.append(keep[nzc])
            vi.append(-Z[nzr, nzc])
        if ri:
            corr = canon((np.concatenate(vi), (np.concatenate(ri), np.concatenate(ci))),
                         shape=(split.n, split.n_pairs))
        else:
            corr = sp.csr_matrix((split.n, split.n_pairs))
        P = canon(Rt + corr)
        if hybrid is not None:
            rows, cols, Z, Wg = hybrid
            P = HybridP(P, Z, rows, cols)
            P.Wg = Wg          # the block's right-hand side W' (rows x cols), for the Galerkin product
    if G is not None:
        Gc, cols = coarse_grad(R, G, mode, split.coarse_nodes)
    else:
        Gc, cols = sp.csr_matrix((split.n_pairs, 0)), np.zeros(0, dtype=np.int64)
    return Transfer(P, R, Gc, cols, blocks)


# ----------------------------------------------------------------------------- smoother

@dataclass
class Patches:
    """PatchSet (smoothers.py:26-40)."""

    patches: list
    factors: list
    update_rows: list
    update_blocks: list


def vertex_patches(A, Gl):
    """build_patches (smoothers.py:60-95)."""
    n = A.shape[0]
    Gc = Gl.tocsc()
    pl = []
    seen = np.zeros(n, dtype=bool)
    for v in range(Gc.shape[1]):
        r = Gc.indices[Gc.indptr[v]:Gc.indptr[v + 1]]
        if r.size:
            p = np.unique(r)
            pl.append(p)
            seen[p] = True
    pl += [np.array([d]) for d in np.flatnonzero(~seen)]
    Ac = A.tocsc()
    facs, rows_l, blocks = [], [], []
    for pid, p in enumerate(pl):
        cols = Ac[:, p]
        rows = np.unique(cols.indices)
        blk = np.asarray(cols[rows, :].todense())
        try:
            facs.append(dense_chol(blk[np.searchsorted(rows, p), :]))
        except NotPositiveDefiniteError as err:
            raise NotPositiveDefiniteError(err.pivot, f"singular patch block {pid}") from err
        rows_l.append(rows)
        blocks.append(blk)
    return Patches(pl, facs, rows_l, blocks)


def l1_diag(A):
    """build_l1_jacobi (smoothers.py:50-52)."""
    return np.asarray(abs(A).sum(axis=1)).ravel()


_potrs = scipy.linalg.lapack.get_lapack_funcs("potrs", (np.zeros(1),))


def _sweep(ps, x, r, order):
    # scipy.linalg.cho_solve((L, True), b) is LAPACK dpotrs(L, b, lower=1)
    # after argument checks; calling dpotrs directly is bit-identical and
    # drops most of the per-patch Python overhead (smoothers.py:98-103)
    for p in order:
        idx = ps.patches[p]
        d, info = _potrs(ps.factors[p], r[idx], lower=1)
        x[idx] += d
        r[ps.update_rows[p]] -= ps.update_blocks[p] @ d


def _jacobi(A, l1, x, r):
    d = r / l1
    x += d
    r -= A @ d


def smooth(A, ps, l1, x, b, direction="forward"):
    """OSS-l1 (smoothers.py:112-137)."""
    if A.shape[0] != len(b) or len(x) != len(b):
        raise ValueError("shape mismatch")
    x = np.array(x, dtype=np.float64)
    r = b - A @ x
    m = len(ps.patches)
    if direction == "forward":
        _sweep(ps, x, r, range(m))
        _jacobi(A, l1, x, r)
    elif direction == "backward":
        _jacobi(A, l1, x, r)
        _sweep(ps, x, r, range(m - 1, -1, -1))
    elif direction == "symmetric":
        _sweep(ps, x, r, range(m))
        _jacobi(A, l1, x, r)
        _jacobi(A, l1, x, r)
        _sweep(ps, x, r, range(m - 1, -1, -1))
    else:
        raise ValueError(f"unknown direction {direction!r}")
    return x


# ----------------------------------------------------------------------------- multilevel

@dataclass
class OLevel:
    A: sp.csr_matrix
    G: sp.csr_matrix
    P: sp.csr_matrix = None
    patches: Patches = None
    l1: np.ndarray = None
    coarse_factor: Factor = None
    splitting: Split = None
    transfer: Transfer = None

    @property
    def n(self):
        return self.A.shape[0]


@dataclass
class OHierarchy:
    levels: list
    method: str
    stalled: bool = False
    notes: list = field(default_factory=list)

    @property
    def depth(self):
        return len(self.levels)


@dataclass
class OReport:
    iterations: int
    residual_history: np.ndarray
    converged: bool
    operator_complexity: float
    note: str = ""


def sign_gradient(Gc):
    """_normalized_gradient (multilevel.py:71-75)."""
    G = canon(Gc)
    G.data = np.sign(G.data)
    return canon(G)


def hierarchy(system, method, meshes=None, rmaps=None, max_levels=20, min_coarse=32,
              theta=0.25, smoother=True, floor_solver=False, large="dense", log=None):
    """build_hierarchy (multilevel.py:78-164) for the "alg" and "ref" routes.

    ``smoother=False`` skips the patch factorisation (used when only the
    setup integers/operators are compared at sizes where it is slow).
    ``floor_solver=True`` swaps the component Cholesky for a reversed-order
    LU to measure the fp64 reproducibility floor of P, A_c and x.
    """
    if method in ("geo", "ref") and (meshes is None or rmaps is None):
        raise ValueError(f"method {method!r} requires the nested mesh chain")
    if method not in ("ref", "alg"):
        raise ValueError(f"unknown method {method!r}")
    A, G = system.A, system.G
    levels, notes, stalled = [], [], False
    pos = len(meshes) - 1 if meshes is not None else 0
    e2d = system.free_edges
    dof_edges = None
    if e2d is not None:
        dof_edges = np.full(system.n, -1, dtype=np.int64)
        live = np.flatnonzero(e2d >= 0)
        dof_edges[e2d[live]] = live
    import time as _time
    t_last = [_time.perf_counter()]

    def mark(what):
        if log is not None:
            now = _time.perf_counter()
            log(f"oracle setup: {what} {now - t_last[0]:.1f} s")
            t_last[0] = now

    while True:
        n = A.shape[0]
        if n <= min_coarse or len(levels) + 1 >= max_levels:
            break
        if method == "ref":
            if pos == 0:
                stalled = True
                notes.append(f"mesh chain exhausted at {n} DoFs")
                break
            split = refinement_split(meshes[pos - 1], meshes[pos], rmaps[pos - 1], e2d, n)
            if split.n_pairs == 0:
                stalled = True
                notes.append("refinement splitting produced no pairs")
                break
            tr = harmonic_interp(A, split, "refinement", G, floor_solver, large)
            nxt = np.full(meshes[pos - 1].ne, -1, dtype=np.int64)
            nxt[split.pair_mesh_edges] = np.arange(split.n_pairs)
        else:
            split = algebraic_split(A, G, theta, dof_edges if not levels else None)
            mark(f"level {len(levels)} splitting (n={n})")
            if split.n_pairs == 0 or split.n_pairs >= n:
                if split.n_pairs == 0:
                    stalled = True
                    notes.append("algebraic coarsening found no pairs")
                break
            tr = harmonic_interp(A, split, "algebraic", G, floor_solver, large)
            mark(f"level {len(levels)} interpolation")
            nxt = None
        P = tr.P
        if P.shape[1] == 0 or P.shape[1] >= n:
            stalled = True
            notes.append(f"no size reduction ({n} -> {P.shape[1]})")
            break
        levels.append(OLevel(A, G, P, vertex_patches(A, G) if smoother else None, l1_diag(A),
                             splitting=split, transfer=tr))
        mark(f"level {len(levels) - 1} patches")
        A = galerkin(P, A)
        mark(f"level {len(levels) - 1} galerkin")
        G = sign_gradient(tr.Gc)
        e2d = nxt
        pos -= 1
    levels.append(OLevel(A, G, coarse_factor=factor_coarsest(A)))
    mark("coarsest factor")
    return OHierarchy(levels, method, stalled, notes)


def _cycle(levels, ell, b):
    """multilevel.py:177-184."""
    lv = levels[ell]
    if lv.P is None:
        return solve_coarsest(lv.coarse_factor, b)
    x = smooth(lv.A, lv.patches, lv.l1, np.zeros_like(b), b, "forward")
    r = b - lv.A @ x
    x = x + lv.P @ _cycle(levels, ell + 1, lv.P.T @ r)
    return smooth(lv.A, lv.patches, lv.l1, x, b, "backward")


def vcycle(h, b, x=None):
    """multilevel.py:187-196."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape[0] != h.levels[0].n:
        raise ValueError("rhs does not match the finest level")
    if x is None:
        return _cycle(h.levels, 0, b)
    x = np.asarray(x, dtype=np.float64)
    return x + _cycle(h.levels, 0, b - h.levels[0].A @ x)


def operator_complexity(h):
    """multilevel.py:199-201."""
    return float(sum(lv.A.nnz for lv in h.levels)) / float(h.levels[0].A.nnz)


def amg_solve(h, b, x0=None, tol=1e-8, maxit=500):
    """multilevel.py:204-235."""
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    A = h.levels[0].A
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return np.zeros_like(b), OReport(0, np.zeros(0), True, operator_complexity(h))
    hist = []
    rel = np.linalg.norm(b - A @ x) / bn
    done = rel <= tol
    note, growth, it = "", 0, 0
    while not done and it < maxit:
        x = vcycle(h, b, x)
        prev, rel = rel, np.linalg.norm(b - A @ x) / bn
        hist.append(rel)
        it += 1
        if rel <= tol:
            done = True
            break
        growth = growth + 1 if rel > prev else 0
        if growth >= 5:
            note = "diverged: residual grew over 5 consecutive iterations"
            break
    return x, OReport(it, np.array(hist), done, operator_complexity(h), note)


def pcg(A, b, precond, x0=None, tol=1e-8, maxit=500, oc=1.0):
    """multilevel.py:238-281."""
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    bn = np.linalg.norm(b)
    if bn == 0.0:
        return np.zeros_like(b), OReport(0, np.zeros(0), True, oc)
    r = b - A @ x
    rel = np.linalg.norm(r) / bn
    if rel <= tol:
        return x, OReport(0, np.zeros(0), True, oc)
    z = precond(r)
    p = z.copy()
    rz = r @ z
    hist, it, done = [], 0, False
    while it < maxit:
        Ap = A @ p
        pAp = p @ Ap
        if pAp <= 0.0:
            raise RuntimeError(f"PCG breakdown: p^T A p = {pAp:.3e} (non-SPD operator)")
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        it += 1
        rel = np.linalg.norm(r) / bn
        hist.append(rel)
        if rel <= tol:
            done = True
            break
        z = precond(r)
        rz_new = r @ z
        if rz_new <= 0.0:
            raise RuntimeError("PCG breakdown: preconditioner is not SPD")
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, OReport(it, np.array(hist), done, oc)
