"""Dense-interpolation regime on the coefficient field the c2 bench runs
("the giant/factor path is not oracle-checked on the benchmarked
coefficient field"): 3D Kuhn n = 16 with configs[1]'s mu^{-1} (4x4x4
checkerboard of 1 / 1e6, beta = 1e-3).  One 20,520-DoF interior component
above the 4096 cutoff, so the GPU runs exactly the c2 kernels: envelope
Cholesky, Y^T Y Galerkin, the TMA factor sweeps for P / P^T, the grid /
dataflow smoothing leg and the dense coarsest solve.  The fixture is the
oracle's run (tests/golden/make_n16c2.py, ~20 min on CPU) together with its
MEASURED reproducibility floors (the same oracle with a reversed-order LU
component solve): x and P move by ~1e-4 between two valid fp64 solvers on
this field, A_1 by 9e-16 -- tolerances are max(1e-10, 10 x floor)."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn

pytestmark = pytest.mark.gpu

FIX = os.path.join(os.path.dirname(__file__), "golden", "kuhn16_c2.npz")


def tol(floor):
    return max(1e-10, 10.0 * floor)


@pytest.fixture(scope="module", params=["auto", "grid", "flow"])
def run(request):
    z = np.load(FIX)
    meta = json.loads(str(z["meta"]))
    s = kuhn.config_system("c2", n=16)
    h = P.build_hierarchy(s, "alg")
    P.multilevel.set_options(h, sweep=request.param)
    x, rep = P.pcg(s.A, z["b"], precond=lambda r: P.vcycle(h, r), tol=1e-8)
    return s, h, x, rep, z, meta


def test_takes_the_dense_path(run):
    s, h, x, rep, z, meta = run
    info = h.levels[0]._info
    assert int(info.max_component) == 20520 and int(info.factor_bytes) > 0 and int(info.factor_tma) == 1
    assert int(h.levels[1]._info.n) >= 0


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


def test_interpolation_and_coarse_operator(run):
    s, h, x, rep, z, meta = run
    Pm = h.levels[0].P
    cs = np.asarray(Pm.sum(axis=0)).ravel()
    assert np.abs(cs - z["P_colsum"]).max() <= tol(meta["floor_P"]) * np.abs(z["P_colsum"]).max()
    A1 = h.levels[1].A
    scale = np.abs(z["A1_sample"]).max()
    t1 = max(1e-12, 10 * meta["floor_A1"])
    assert np.abs(A1.diagonal() - z["A1_diag"]).max() <= t1 * scale
    assert np.abs(np.asarray(A1.sum(axis=1)).ravel() - z["A1_rowsum"]).max() <= t1 * scale * 10
    rows = A1[z["A1_rows"]].toarray()
    assert np.abs(rows - z["A1_sample"]).max() <= t1 * scale  # entrywise, 64 full rows
    assert P.operator_complexity(h) == pytest.approx(meta["oc"], rel=1e-12)


def test_vcycle_and_pcg(run):
    s, h, x, rep, z, meta = run
    v = P.vcycle(h, z["vcycle_b"])
    assert np.abs(v - z["vcycle_x"]).max() <= tol(meta["floor_vcycle"]) * np.abs(z["vcycle_x"]).max()
    assert rep.converged and abs(rep.iterations - meta["pcg_iters"]) <= 1
    assert np.linalg.norm(x - z["pcg_x"]) <= tol(meta["floor_x"]) * np.linalg.norm(z["pcg_x"])
