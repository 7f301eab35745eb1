"""BASELINE configs[1] at full size (Kuhn n = 32, 220,256 DoFs, 1e6 checkerboard):
the reference cannot build this hierarchy, so parity is checked
through size-independent properties -- the level-0 integers against the
reference-generated fixture (tests/test_split_large.py holds the split itself),
the component solve's backward error, the V-cycle's symmetry, PCG convergence
and bit-identical repeated solves."""

import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import _lib, kuhn

pytestmark = pytest.mark.gpu

FIX = os.path.join(os.path.dirname(__file__), "golden", "split_c2_n32.npz")


@pytest.fixture(scope="module")
def c2():
    s = kuhn.config_system("c2")
    return s, P.build_hierarchy(s, "alg")


def test_levels_and_level0_integers(c2):
    s, h = c2
    assert [lv.n for lv in h.levels] == [220256, 26236] and h.stalled
    # the dense block goes through the factor, on the TMA-streamed sweep kernel
    info = h.levels[0]._info
    assert info.factor_bytes > 0 and info.factor_tma == 1
    sp = h.levels[0].splitting
    z = np.load(FIX)
    assert len(sp.pairs) == 26236 and len(sp.interior_dofs) == 167784
    assert np.array_equal(np.array([tuple(p) for p in sp.pairs], dtype=np.int64), z["pairs"])
    assert np.array_equal(sp.interior_dofs, z["interior"])
    assert np.array_equal(sp.coarse_nodes, z["cG"])


def test_component_solve_backward_error(c2):
    s, h = c2
    dev = h._dev
    nG = int(h.levels[0]._info.max_component)
    rows = np.zeros(nG, np.int64)
    dev.check(dev.lib.hcamg_export_dense(dev.h, 0, 1, _lib.ptr(rows)))
    Agg = s.A[rows][:, rows].tocsr()
    v = np.random.default_rng(1).uniform(-1, 1, nG)
    out = np.zeros(nG)
    dev.check(dev.lib.hcamg_component_solve(dev.h, 0, _lib.ptr(v), _lib.ptr(out)))
    res = np.linalg.norm(Agg @ out - v) / (spla.norm(Agg, 1) * np.linalg.norm(out))
    assert res <= 1e-14, res


def test_vcycle_symmetric(c2):
    s, h = c2
    rng = np.random.default_rng(2)
    x, y = rng.uniform(-1, 1, s.n), rng.uniform(-1, 1, s.n)
    bx, by = P.vcycle(h, x), P.vcycle(h, y)
    # symmetric in exact arithmetic; roundoff through A_GG^{-1} (kappa ~ 1e12 on
    # this field) leaves ~1e-7..1e-6 relative, depending on where the residual
    # is re-formed: measured 4.8e-7 with the grid leg, 7.1e-7 with per-wave
    # launches, 2.3e-6 with the dataflow leg (which re-forms b - A x after the
    # down sweep; its smoother alone is adjoint to 2.9e-8, tools/sym_check.py)
    assert abs(bx @ y - x @ by) <= 1e-5 * np.linalg.norm(bx) * np.linalg.norm(y)
    assert bx @ x > 0 and by @ y > 0


def test_pcg_converges_and_is_deterministic(c2):
    s, h = c2
    b = kuhn.rhs(s.n, seed=0)
    x1, r1 = P.pcg(s.A, b, precond=lambda r: P.vcycle(h, r), tol=1e-8)
    x2, r2 = P.pcg(s.A, b, precond=lambda r: P.vcycle(h, r), tol=1e-8)
    assert r1.converged and r1.iterations <= 15 and r1.residual_history[-1] <= 1e-8
    assert np.array_equal(x1, x2) and r1.iterations == r2.iterations
    # the true residual sits at the conditioning floor the reference itself
    # shows on this field (4.6e-5 at n = 8, 1.3e-4 at n = 12)
    assert np.linalg.norm(s.A @ x1 - b) / np.linalg.norm(b) <= 5e-3
