"""The reference's smoother contracts (pkg/tests/test_smoothers.py) run on the
device OSS-l1 legs through the drop-in ``smoothers`` module, plus the
CholeskyFactor fields and the coarsest-level solve (sparse.py:146-165,
276-321)."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2602_23613_b200 as P
from oracle import amg_oracle as O
from paper_2602_23613_b200.smoothers import build_l1_jacobi, build_patches, smooth
from paper_2602_23613_b200.sparse import cholesky, csr, solve
from tests.cases import api_system

pytestmark = pytest.mark.gpu


def tri_system(L=2):
    return api_system(f"tri{L}")[2]


def test_l1_values():
    s = tri_system()
    l1 = build_l1_jacobi(s.A)
    assert np.all(l1.d >= s.A.diagonal() - 1e-15)
    assert np.allclose(build_l1_jacobi(csr([[2.0, -1.0], [-1.0, 2.0]])).d, [3.0, 3.0])


def test_patches_cover_and_match_incidence():
    s = tri_system(1)
    ps = build_patches(s.A, s.G)
    covered = np.zeros(s.n, dtype=bool)
    for p in ps.patches:
        covered[p] = True
    assert covered.all()
    Gc = s.G.tocsc()
    for v in range(Gc.shape[1]):
        rows = Gc.indices[Gc.indptr[v]:Gc.indptr[v + 1]]
        assert len(ps.patches[v]) == len(np.unique(rows))


def test_patches_match_oracle_fields():
    s = tri_system(2)
    ps = build_patches(s.A, s.G)
    po = O.vertex_patches(s.A, s.G)
    assert all(np.array_equal(a, b) for a, b in zip(ps.patches, po.patches))
    for a, b in zip(ps.update_rows, po.update_rows):
        assert np.array_equal(a, b)
    for a, b in zip(ps.update_blocks, po.update_blocks):
        assert np.array_equal(a, b)
    for a, b in zip(ps.factors, po.factors):
        assert np.allclose(a, b, rtol=1e-13, atol=0)


def test_single_column_gradient_single_patch():
    A = csr(np.diag([2.0, 3.0, 4.0]))
    G = csr(np.array([[1.0], [-1.0], [0.0]]))
    ps = build_patches(A, G)
    assert ps.patches[0].tolist() == [0, 1]
    assert any(p.tolist() == [2] for p in ps.patches)


def test_fixed_point_invariance():
    s = tri_system()
    rng = np.random.default_rng(0)
    x_star = rng.standard_normal(s.n)
    b = s.A @ x_star
    ps = build_patches(s.A, s.G)
    l1 = build_l1_jacobi(s.A)
    for direction in ("forward", "backward", "symmetric"):
        x = smooth(s.A, ps, l1, x_star, b, direction)
        assert np.max(np.abs(x - x_star)) <= 1e-12 * max(1.0, np.abs(x_star).max())


def test_single_patch_covering_everything_solves():
    A = csr(np.array([[4.0, 1.0], [1.0, 3.0]]))
    G = csr(np.array([[1.0, -1.0], [-1.0, 1.0]]))
    ps = build_patches(A, G)
    b = np.array([1.0, 2.0])
    x = smooth(A, ps, build_l1_jacobi(A), np.zeros(2), b, "forward")
    assert np.linalg.norm(A @ x - b) <= 1e-13


def a_norm(A, e):
    return float(np.sqrt(e @ (A @ e)))


def test_energy_monotonicity():
    s = tri_system(2)
    ps = build_patches(s.A, s.G)
    l1 = build_l1_jacobi(s.A)
    rng = np.random.default_rng(1)
    x_star = rng.standard_normal(s.n)
    b = s.A @ x_star
    for direction in ("forward", "backward", "symmetric"):
        for _ in range(5):
            x0 = rng.standard_normal(s.n)
            before = a_norm(s.A, x0 - x_star)
            after = a_norm(s.A, smooth(s.A, ps, l1, x0, b, direction) - x_star)
            assert after < before, f"{direction}: {after} !< {before}"


def test_symmetric_error_propagator_is_a_selfadjoint():
    s = tri_system(1)
    ps = build_patches(s.A, s.G)
    l1 = build_l1_jacobi(s.A)

    def apply_E(e):
        return -smooth(s.A, ps, l1, -e, np.zeros(s.n), "symmetric")

    rng = np.random.default_rng(2)
    for _ in range(5):
        e1, e2 = rng.standard_normal((2, s.n))
        lhs = apply_E(e1) @ (s.A @ e2)
        rhs = e1 @ (s.A @ apply_E(e2))
        assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs), 1.0)


def test_forward_backward_are_mutually_adjoint():
    s = tri_system(1)
    ps = build_patches(s.A, s.G)
    l1 = build_l1_jacobi(s.A)

    def apply_dir(e, direction):
        return -smooth(s.A, ps, l1, -e, np.zeros(s.n), direction)

    rng = np.random.default_rng(3)
    for _ in range(5):
        e1, e2 = rng.standard_normal((2, s.n))
        lhs = apply_dir(e1, "forward") @ (s.A @ e2)
        rhs = e1 @ (s.A @ apply_dir(e2, "backward"))
        assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs), 1.0)


def test_smooth_matches_oracle_all_legs():
    s = tri_system(3)
    ps = build_patches(s.A, s.G)
    po = O.vertex_patches(s.A, s.G)
    l1o = O.l1_diag(s.A)
    rng = np.random.default_rng(4)
    x0, b = rng.standard_normal((2, s.n))
    for sweep in ("auto", "leg", "grid", "wave", "flow", "fwave"):
        ps._dev.set_option("sweep", P.multilevel.SWEEP_MODES[sweep])
        for d in ("forward", "backward", "symmetric"):
            xg = smooth(s.A, ps, None, x0, b, d)
            xo = O.smooth(s.A, po, l1o, x0, b, d)
            assert np.max(np.abs(xg - xo)) <= 1e-10 * np.max(np.abs(xo)), (sweep, d)


def test_smooth_shape_check():
    s = tri_system(1)
    ps = build_patches(s.A, s.G)
    l1 = build_l1_jacobi(s.A)
    with pytest.raises(ValueError):
        smooth(s.A, ps, l1, np.zeros(3), np.zeros(s.n))
    with pytest.raises(ValueError):
        smooth(s.A, ps, l1, np.zeros(s.n), np.zeros(s.n), "sideways")


# ---------------------------------------------------------------- CholeskyFactor / solve

def test_cholesky_factor_fields():
    s = tri_system(2)
    f = cholesky(s.A)
    fo = O.factor_coarsest(s.A)
    assert sorted(f.ordering) == list(range(s.n))
    L = f.factor.toarray()
    Ap = s.A[f.ordering][:, f.ordering].toarray()
    assert np.allclose(L, np.tril(L)) and np.all(np.diag(L) > 0)
    assert np.max(np.abs(L @ L.T - Ap)) <= 1e-13 * np.max(np.abs(Ap))
    if np.array_equal(f.ordering, fo.perm):  # reverse Cuthill-McKee (scipy breaks degree ties unstably)
        assert np.allclose(L, fo.L, rtol=1e-12, atol=1e-14 * np.max(np.abs(fo.L)))
    b = np.random.default_rng(5).standard_normal(s.n)
    x = solve(f, b)
    assert np.linalg.norm(s.A @ x - b) <= 1e-11 * np.linalg.norm(b)
    B = np.random.default_rng(6).standard_normal((s.n, 3))
    X = solve(f, B)
    assert np.linalg.norm(s.A @ X - B) <= 1e-11 * np.linalg.norm(B)


def test_coarse_factor_solve_on_multilevel_hierarchy():
    """solve() on the coarse factor of a hierarchy with depth
    > 1 must apply the coarsest inverse, not a V-cycle on level 0."""
    meshes, rmaps, system = api_system("tri3")
    h = P.build_hierarchy(system, "alg")
    assert h.depth > 1
    Lc = h.levels[-1]
    cf = Lc.coarse_factor
    assert cf.n == Lc.n
    b = np.random.default_rng(7).standard_normal(Lc.n)
    x = solve(cf, b)
    assert x.shape == (Lc.n,)
    assert np.linalg.norm(Lc.A @ x - b) <= 1e-10 * np.linalg.norm(b)
    with pytest.raises(ValueError):
        solve(cf, np.zeros(Lc.n + 1))
    Ap = Lc.A[cf.ordering][:, cf.ordering].toarray()
    L = cf.factor.toarray()
    assert np.max(np.abs(L @ L.T - Ap)) <= 1e-12 * np.max(np.abs(Ap))


def test_user_hierarchy_with_device_coarse_factor():
    """A coarse factor taken from a device hierarchy can be attached to a
    user-assembled one (tests/test_multilevel.py:125-134 style)."""
    meshes, rmaps, system = api_system("tri3")
    h = P.build_hierarchy(system, "alg")
    lv = [P.Level(A=l.A, G=l.G, P=l.P) for l in h.levels[:-1]]
    lv.append(P.Level(A=h.levels[-1].A, G=h.levels[-1].G, coarse_factor=h.levels[-1].coarse_factor))
    h2 = P.Hierarchy(lv, "alg")
    b = np.random.default_rng(8).standard_normal(system.n)
    assert np.max(np.abs(P.vcycle(h2, b) - P.vcycle(h, b))) <= 1e-12 * np.max(np.abs(P.vcycle(h, b)))


def test_pcg_device_zero_rhs_without_report():
    """b = 0 with a nonzero x0 returns x = 0 even when the
    caller skips the report; errors are then read with hcamg_solve_status."""
    import ctypes as C

    import torch

    from paper_2602_23613_b200 import _lib
    meshes, rmaps, system = api_system("tri3")
    h = P.build_hierarchy(system, "alg")
    dev = h._dev
    n = system.n
    b = torch.zeros(n, dtype=torch.float64, device="cuda")
    x0 = torch.ones(n, dtype=torch.float64, device="cuda")
    x = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    dev.check(dev.lib.hcamg_pcg_device(dev.h, C.c_void_p(b.data_ptr()), C.c_void_p(x0.data_ptr()), 1e-8, 100,
                                       C.c_void_p(x.data_ptr()), None))
    rep = _lib.Report()
    dev.check(dev.lib.hcamg_solve_status(dev.h, C.byref(rep)))
    assert rep.zero_rhs == 1 and rep.iterations == 0
    assert float(x.abs().max()) == 0.0
