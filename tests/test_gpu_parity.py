"""GPU path (through the C-ABI) vs the CPU oracle on the golden cases.

Integer outputs are compared bit-exactly: C/F split (c_G), the pair list, the
interior set, patch lists, and the sparsity patterns of every A_l, P_l, G_l.
Floating point: level-0 A and every G exactly; P, A_c, V-cycle output and
PCG solution normwise within max(1e-10, 10 x floor), where the floor is
MEASURED per case as the distance between the oracle and the same oracle
with its component Cholesky swapped for a reversed-order LU (two valid fp64
algorithms).  On the 1e6-contrast checkerboard the
floor is 2.5e-5, on the 100-contrast stripes 3e-10, elsewhere <= 4e-12.
PCG iteration counts must agree within +-1 (they agree exactly in practice).
"""

import numpy as np
import pytest

from oracle import amg_oracle as O
from tests.cases import CASES, load

import paper_2602_23613_b200 as P

pytestmark = pytest.mark.gpu



def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)) if np.size(b) else 0.0


def same_pattern(a, b):
    a, b = a.tocsr(), b.tocsr()
    return (a.shape == b.shape and a.nnz == b.nnz and np.array_equal(a.indptr, b.indptr)
            and np.array_equal(a.indices, b.indices))


@pytest.fixture(scope="module", params=CASES)
def pair(request):
    c = load(request.param)
    ho = O.hierarchy(c.system, c.meta["method"], meshes=c.meshes, rmaps=c.rmaps)
    hf = O.hierarchy(c.system, c.meta["method"], meshes=c.meshes, rmaps=c.rmaps, floor_solver=True)
    b = c.z["pcg_b"]
    xo, ro = O.pcg(c.system.A, b, precond=lambda r: O.vcycle(ho, r), tol=1e-8)
    xf, rf = O.pcg(c.system.A, b, precond=lambda r: O.vcycle(hf, r), tol=1e-8)
    c.hist_tol = 1e-6
    if ro.iterations == rf.iterations:
        c.hist_tol = max(1e-6, 10.0 * float(np.max(np.abs(rf.residual_history - ro.residual_history)
                                                   / ro.residual_history)))
    floor = max([rel(f.P.data, o.P.data) for f, o in zip(hf.levels[:-1], ho.levels[:-1])]
                + [np.linalg.norm(xf - xo) / np.linalg.norm(xo)])
    c.tol = max(1e-10, 10.0 * floor)
    hg = P.build_hierarchy(c.system, c.meta["method"], meshes=c.meshes, rmaps=c.rmaps)
    return request.param, c, ho, hg


def test_hierarchy_integers_bit_exact(pair):
    name, c, ho, hg = pair
    assert hg.depth == ho.depth and hg.stalled == ho.stalled and hg.notes == ho.notes
    for ell, (lg, lo) in enumerate(zip(hg.levels, ho.levels)):
        assert lg.n == lo.n
        assert same_pattern(lg.A, lo.A), f"A_{ell} pattern"
        assert same_pattern(lg.G, lo.G) and np.array_equal(lg.G.data, lo.G.data), f"G_{ell}"
        if lo.P is None:
            assert lg.P is None
            continue
        so, sg = lo.splitting, lg.splitting
        assert [tuple(p) for p in sg.pairs] == [(p.dof1, p.dof2, p.sign1, p.sign2, p.tail, p.mid, p.head)
                                               for p in so.pairs]
        assert np.array_equal(sg.interior_dofs, so.interior_dofs)
        if so.coarse_nodes is not None:
            assert np.array_equal(sg.coarse_nodes, so.coarse_nodes)
        if so.pair_mesh_edges is not None:
            assert np.array_equal(sg.pair_mesh_edges, so.pair_mesh_edges)
        assert same_pattern(lg.P, lo.P), f"P_{ell} pattern"
        assert len(lg.patches.patches) == len(lo.patches.patches)
        assert all(np.array_equal(a, b) for a, b in zip(lg.patches.patches, lo.patches.patches))


def test_splitting_text_matches_reference_dump(pair):
    """The GPU splittings written in the reference's text format
    (splitting.py:375-380) hash to the reference's own dumps."""
    import hashlib

    from paper_2602_23613_b200.formats import dump_splitting
    name, c, ho, hg = pair
    for ell, ref in enumerate(c.meta["levels"]):
        if "dump_sha" in ref:
            text = dump_splitting(hg.levels[ell].splitting)
            assert hashlib.sha256(text.encode()).hexdigest() == ref["dump_sha"], f"level {ell}"


def test_hierarchy_values(pair):
    name, c, ho, hg = pair
    tol = c.tol
    assert np.array_equal(hg.levels[0].A.data, ho.levels[0].A.data)
    for lg, lo in zip(hg.levels, ho.levels):
        assert rel(lg.A.data, lo.A.data) <= max(tol, 1e-12)
        if lo.P is not None:
            assert rel(lg.P.data, lo.P.data) <= tol
            assert rel(lg.l1.d, lo.l1) <= max(tol, 1e-12)
    assert P.operator_complexity(hg) == O.operator_complexity(ho)


def test_galerkin_bit_consistency(pair):
    """tests/test_multilevel.py:51-62: re-forming P^T A P with scipy from the
    exported operators reproduces A_{l+1} bit for bit (the GPU SpGEMM sums in
    scipy's order without FMA)."""
    name, c, ho, hg = pair
    for ell in range(hg.depth - 1):
        lv, nx = hg.levels[ell], hg.levels[ell + 1]
        M = lv.P.T @ (lv.A @ lv.P)
        rebuilt = P.csr(0.5 * (M + M.T))
        assert same_pattern(rebuilt, nx.A)
        assert np.array_equal(rebuilt.data, nx.A.data)


def test_solves(pair):
    name, c, ho, hg = pair
    tol = c.tol
    b = c.z["pcg_b"]
    assert rel(P.vcycle(hg, b), O.vcycle(ho, b)) <= tol
    xo, ro = O.pcg(c.system.A, b, precond=lambda r: O.vcycle(ho, r), tol=1e-8)
    xg, rg = P.pcg(c.system.A, b, precond=lambda r: P.vcycle(hg, r), tol=1e-8)
    assert rg.converged and abs(rg.iterations - ro.iterations) <= 1
    assert np.linalg.norm(xg - xo) <= tol * np.linalg.norm(xo)
    # true residual: the recurrence residual reaches tol; the true one is bounded by
    # the oracle's own gap (kappa(A) * eps; large on the 1e6-contrast case)
    true_o = np.linalg.norm(c.system.A @ xo - b)
    assert np.linalg.norm(c.system.A @ xg - b) <= max(1.01e-8 * np.linalg.norm(b), 10 * true_o)
    if rg.iterations == ro.iterations:
        assert np.allclose(rg.residual_history, ro.residual_history, rtol=max(c.hist_tol, 10 * tol), atol=0)
    xa, ra = P.amg_solve(hg, c.z["amg_b"], x0=c.z["amg_x0"], tol=1e-8, maxit=200)
    if c.meta["amg_iters"] >= 200:
        # the reference's stand-alone AMG stagnates on the 1e6-contrast fields (no
        # convergence in 200 cycles); whether and when its divergence guard fires
        # is roundoff-driven there
        assert not ra.converged
        return
    assert abs(ra.iterations - c.meta["amg_iters"]) <= 1
    assert np.linalg.norm(xa - c.z["amg_x"]) <= tol * np.linalg.norm(c.z["amg_x"])


def test_pcg_deterministic(pair):
    name, c, ho, hg = pair
    b = c.z["pcg_b"]
    x1, r1 = P.pcg(c.system.A, b, precond=lambda r: P.vcycle(hg, r), tol=1e-8)
    x2, r2 = P.pcg(c.system.A, b, precond=lambda r: P.vcycle(hg, r), tol=1e-8)
    assert np.array_equal(x1, x2) and np.array_equal(r1.residual_history, r2.residual_history)
