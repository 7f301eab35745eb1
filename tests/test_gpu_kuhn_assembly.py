"""GPU assembly of the Kuhn-cube systems (csrc/kuhn.cu) against the host
generator kuhn.py: identical pattern, gradient and index maps; A equal up to
the summation order of duplicate element contributions (last-bit level); the
hierarchy built from the GPU-assembled system reproduces the reference's
splitting fixture and PCG iteration count."""

import json
import os

import numpy as np
import pytest

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n", [("c1", 4), ("c1", 8), ("c2", 8), ("c2", 16), ("c4", 8)])
def test_gpu_assembly_matches_host(cfg, n):
    host = kuhn.config_system(cfg, n=n)
    dev = kuhn.config_system_gpu(cfg, n=n)
    assert np.array_equal(dev.free_edges, host.free_edges) and np.array_equal(dev.free_nodes, host.free_nodes)
    for X, Y in ((dev.G, host.G), (dev.A, host.A)):
        assert X.shape == Y.shape
        assert np.array_equal(X.indptr, Y.indptr) and np.array_equal(X.indices, Y.indices)
    assert np.array_equal(dev.G.data, host.G.data)
    scale = np.abs(host.A.data).max()
    assert np.abs(dev.A.data - host.A.data).max() <= 1e-14 * scale
    assert (dev.A != dev.A.T).nnz == 0  # exactly symmetric, as the host system


def test_gpu_assembled_hierarchy_matches_reference_fixture():
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "kuhn8_c1.npz"), allow_pickle=True)
    s = kuhn.config_system_gpu("c1", n=8)
    h = P.build_hierarchy(s, "alg")
    sp = h.levels[0].splitting
    assert np.array_equal(np.array([tuple(p) for p in sp.pairs], dtype=np.int64), z["L0_pairs"].reshape(-1, 7))
    assert np.array_equal(sp.interior_dofs, z["L0_interior"])
    x, rep = P.pcg(s.A, kuhn.rhs(s.n, 0), precond=lambda r: P.vcycle(h, r), tol=1e-8)
    assert rep.converged and rep.iterations == 11  # SURVEY A.4 (reference, host-assembled system)
