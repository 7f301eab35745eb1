"""Coarsest solve through the packed lower triangle of the symmetric inverse
(csrc/symv.cu): x = A_c^{-1} b must match a dense solve and the full-matrix row
GEMV to roundoff, be bit-identical run to run, and handle odd widths, sizes
below one CTA's column span and the largest size it accepts (26,624 rows; the
config-2 coarsest level has 26,236)."""

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg  # noqa: F401

import paper_2602_23613_b200 as P

pytestmark = pytest.mark.gpu


def _spd(n, seed=11):
    rng = np.random.default_rng(seed)
    main = 2.5 + rng.uniform(0, 1, n)
    off = -np.ones(n - 1)
    return sp.csr_matrix(sp.diags([off, main, off], [-1, 0, 1]))


@pytest.mark.parametrize("n", [1, 2, 511, 512, 513, 4097, 26624])
def test_symv_coarse_solve(monkeypatch, n):
    monkeypatch.setenv("HCAMG_COARSE_GEMV_MIN", "0")
    A = _spd(n)
    b = np.random.default_rng(2).uniform(-1, 1, n)
    x = P.vcycle(P.Hierarchy([P.Level(A=A)], "alg"), b)
    xr = sp.linalg.spsolve(A.tocsc(), b)
    assert np.linalg.norm(x - xr) <= 1e-12 * np.linalg.norm(xr)
    h = P.Hierarchy([P.Level(A=A)], "alg")
    assert np.array_equal(P.vcycle(h, b), x) and np.array_equal(P.vcycle(h, b), x)
    monkeypatch.setenv("HCAMG_COARSE_SYMV", "0")
    xf = P.vcycle(P.Hierarchy([P.Level(A=A)], "alg"), b)
    assert np.linalg.norm(x - xf) <= 1e-13 * np.linalg.norm(xf)
