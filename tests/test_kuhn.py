"""3D Kuhn-cube input generator (SURVEY.md §A.2 / §A.4 sanity values)."""

import numpy as np

from paper_2602_23613_b200 import kuhn


def test_counts_and_exact_sequence():
    for n in (2, 3, 4):
        m = kuhn.kuhn_mesh(n)
        assert m.ne == 3 * n * (n + 1) ** 2 + 3 * n * n * (n + 1) + n ** 3
        s = kuhn.assemble_kuhn(m, np.ones(m.nc), 1e-2)
        assert s.n == m.ne - 18 * n * n
        AsG = (s.As @ s.G).tocsr()
        assert np.abs(AsG.data).max(initial=0) <= 1e-12 * np.abs(s.As.data).max()
        assert np.array_equal(np.unique(np.diff(s.G.indptr)), np.unique(np.diff(s.G.indptr)))
        assert set(np.diff(s.G.indptr).tolist()) <= {0, 1, 2}
        d = abs(s.A - s.A.T)
        assert d.nnz == 0 or d.max() == 0.0


def test_stiffness_kernel_dimension_n3():
    m = kuhn.kuhn_mesh(3)
    s = kuhn.assemble_kuhn(m, np.ones(m.nc), 0.0)
    ev = np.linalg.eigvalsh(s.As.toarray())
    nint = int((~m.boundary_vertex).sum())
    assert int(np.sum(np.abs(ev) < 1e-10 * ev.max())) == nint


def test_config1_matches_survey():
    s = kuhn.config_system("c1")
    assert s.n == 3032 and s.A.nnz == 43688
    assert s.G.shape == (3032, 343) and s.G.nnz == 4802
    lone = int(np.sum(np.diff(s.G.indptr) == 1))
    assert lone == 1094
    np.linalg.cholesky(s.A.toarray())  # SPD


def test_rhs_seed():
    b = kuhn.rhs(10, seed=0)
    assert np.array_equal(b, np.random.default_rng(0).uniform(-1, 1, 10))
