"""The 2D stripes generator (paper_2602_23613_b200/tri2d.py) reproduces the
reference's meshes, refinement maps and assembled systems bit for bit: the
golden fixtures' inputs were produced by the reference itself
(tests/golden/make_golden.py: mesh.refinement_chain + fem.assemble)."""

import numpy as np
import pytest

from paper_2602_23613_b200 import tri2d
from tests.cases import load


@pytest.mark.parametrize("name,L,stripes", [("tri2_alg", 2, False), ("tri3s_alg", 3, True), ("tri3s_ref", 3, True),
                                            ("tri5s_alg", 5, True), ("tri5s_ref", 5, True)])
def test_generator_bit_exact(name, L, stripes):
    c = load(name)
    meshes, rmaps, s = tri2d.tri_chain(L, stripes=stripes)
    for M, R in ((s.A, c.system.A), (s.G, c.system.G)):
        assert M.shape == R.shape
        assert np.array_equal(M.indptr, R.indptr) and np.array_equal(M.indices, R.indices)
        assert np.array_equal(M.data, R.data)
    assert np.array_equal(s.free_edges, c.system.free_edges)
    if c.meshes is not None:
        assert all(np.array_equal(m.edges, cm.edges) for m, cm in zip(meshes, c.meshes))
        assert all(np.array_equal(r.coarse_edge_children, cr.coarse_edge_children) for r, cr in zip(rmaps, c.rmaps))


def test_refinement_counts():
    meshes, rmaps = tri2d.refinement_chain(tri2d.uniform_tri_mesh0(), 4)
    for L, m in enumerate(meshes):
        n = 2 ** L
        assert m.nv == (n + 1) ** 2 and m.nc == 2 * n * n and m.ne == 3 * n * n + 2 * n
        assert m.nv - m.ne + m.nc == 1  # Euler characteristic of the square
