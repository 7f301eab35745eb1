"""Dense-interpolation regime: 3D Kuhn n = 16, one 20,520-DoF
interior component, dense 2,948-DoF level 1.  The GPU takes the packed-tile
Cholesky / hybrid-P / Schur-Galerkin path; the fixture is the oracle's run
(pinned to the reference on the golden cases; ~10 min on CPU, so only the
integers, norms, the PCG history and x are stored: tests/golden/make_n16.py)."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn

pytestmark = pytest.mark.gpu

FIX = os.path.join(os.path.dirname(__file__), "golden", "kuhn16_c1.npz")


@pytest.fixture(scope="module")
def run():
    z = np.load(FIX)
    meta = json.loads(str(z["meta"]))
    s = kuhn.config_system("c1", n=16)
    h = P.build_hierarchy(s, "alg")
    x, rep = P.pcg(s.A, z["b"], precond=lambda r: P.vcycle(h, r), tol=1e-8)
    return s, h, x, rep, z, meta


def test_integers_bit_exact(run):
    s, h, x, rep, z, meta = run
    assert [lv.n for lv in h.levels] == meta["levels"] and h.stalled == meta["stalled"] and h.notes == meta["notes"]
    sp = h.levels[0].splitting
    assert np.array_equal(np.array([tuple(p) for p in sp.pairs], dtype=np.int64), z["pairs"])
    assert np.array_equal(sp.interior_dofs, z["interior"])
    assert np.array_equal(sp.coarse_nodes, z["cG"])
    Pm = h.levels[0].P
    sha = hashlib.sha256(Pm.indptr.astype(np.int64).tobytes() + Pm.indices.astype(np.int64).tobytes()).hexdigest()
    assert Pm.nnz == meta["P_nnz"] and sha == meta["P_pattern_sha"]
    assert h.levels[1].A.nnz == meta["A1_nnz"]


def test_values(run):
    s, h, x, rep, z, meta = run
    Pm = h.levels[0].P
    assert abs(np.sqrt((Pm.data ** 2).sum()) - meta["P_fro"]) <= 1e-10 * meta["P_fro"]
    cs = np.asarray(Pm.sum(axis=0)).ravel()
    assert np.abs(cs - z["P_colsum"]).max() <= 1e-10 * np.abs(z["P_colsum"]).max()
    A1 = h.levels[1].A
    assert abs(np.sqrt((A1.data ** 2).sum()) - meta["A1_fro"]) <= 1e-10 * meta["A1_fro"]
    assert np.abs(A1.diagonal() - z["A1_diag"]).max() <= 1e-10 * np.abs(z["A1_diag"]).max()
    assert P.operator_complexity(h) == pytest.approx(meta["oc"], rel=1e-12)


def test_pcg(run):
    s, h, x, rep, z, meta = run
    assert rep.converged and abs(rep.iterations - meta["pcg_iters"]) <= 1
    assert np.linalg.norm(x - z["pcg_x"]) <= 1e-10 * np.linalg.norm(z["pcg_x"])
    if rep.iterations == meta["pcg_iters"]:
        assert np.allclose(rep.residual_history, z["pcg_hist"], rtol=1e-6, atol=0)
