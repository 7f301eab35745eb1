"""3D Kuhn-cube input generator (SURVEY.md §A.2 / §A.4 sanity values)."""

import numpy as np
import pytest

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


def test_chain_refine_numbering_and_children():
    meshes, rmaps = kuhn.kuhn_chain(2, 2)
    assert [m.n for m in meshes] == [2, 4, 8]
    for c, f, r in zip(meshes, meshes[1:], rmaps):
        # coarse vertices keep their numbers, midpoints follow in coarse edge order
        assert np.array_equal(f.vertices[: c.nv], c.vertices)
        t, h = c.edges[:, 0], c.edges[:, 1]
        mid = c.nv + np.arange(c.ne)
        assert np.allclose(f.vertices[mid], 0.5 * (c.vertices[t] + c.vertices[h]))
        assert f.nv == c.nv + c.ne
        # children: fine edges (tail, mid) and (head, mid), stored tail < head
        k0, k1 = f.edges[r.coarse_edge_children[:, 0]], f.edges[r.coarse_edge_children[:, 1]]
        assert np.array_equal(np.sort(k0, axis=1), np.sort(np.stack([t, mid], 1), axis=1))
        assert np.array_equal(np.sort(k1, axis=1), np.sort(np.stack([h, mid], 1), axis=1))
        # the renumbered mesh is the same geometric Kuhn mesh (tet by tet)
        ref = kuhn.kuhn_mesh(f.n)
        assert np.allclose(f.vertices[f.tets], ref.vertices[ref.tets])
        assert f.ne == ref.ne and int(f.boundary_edge.sum()) == int(ref.boundary_edge.sum())


def test_chain_system_is_the_same_operator_up_to_renumbering():
    s_chain, meshes, _ = kuhn.config_chain("c1", 8, 2)
    s_lex = kuhn.config_system("c1", 8)
    assert s_chain.n == s_lex.n == 3032
    # match edges geometrically (midpoint) and compare |A| entries
    def mids(s):
        m = s.mesh
        fe = np.flatnonzero(~m.boundary_edge)
        return np.round(0.5 * (m.vertices[m.edges[fe, 0]] + m.vertices[m.edges[fe, 1]]) * 16).astype(int)
    key = lambda g: (g[:, 2] * 17 + g[:, 1]) * 17 + g[:, 0]
    pc, pl = np.argsort(key(mids(s_chain))), np.argsort(key(mids(s_lex)))
    Ac = abs(s_chain.A[pc][:, pc]).toarray()
    Al = abs(s_lex.A[pl][:, pl]).toarray()
    assert np.allclose(Ac, Al, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("n", [2, 5, 8])
def test_gpu_assembly_host_inputs_match_mesh(n):
    """The host inputs of the GPU assembler (csrc/kuhn.cu): tet corners, centroids
    (for the coefficient fields) and the six element matrices equal those of
    kuhn_mesh / assemble_kuhn bit for bit."""
    m = kuhn.kuhn_mesh(n)
    cells = kuhn._KuhnCells(n)
    N = n + 1
    c = cells.tet_corners()
    assert np.array_equal((c[:, :, 2] * N + c[:, :, 1]) * N + c[:, :, 0], m.tets)
    assert np.array_equal(cells.tet_centroids(), m.tet_centroids())
    S6, M6 = kuhn._element_matrices(n)
    for p in range(6):
        S, M = kuhn._tet_element(m.vertices[m.tets[p]])
        assert np.array_equal(S, S6[p]) and np.array_equal(M, M6[p])
    assert np.all(m.tet_edge_signs == 1)  # lexicographic numbering: every local edge rises
