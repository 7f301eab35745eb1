"""Row-partitioned multi-GPU solve, checked on one GPU.

Several ranks cannot run concurrently on one GPU (their exchange kernels would
wait on each other), so the N-rank V-cycle is emulated piece by piece through a
debug entry point: every rank runs the part of a piece up to its exchange
signal, then every rank runs the part from the exchange wait on.  The emulated
ranks' results must equal the single-GPU V-cycle bit for bit (the partition
and the two-level restriction sum are rank-count independent by design).
A one-rank distributed handle (exchanging with itself) runs the complete
graph-captured PCG / AMG / V-cycle through the exchange kernels."""

import ctypes as C

import numpy as np
import pytest

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import dist, kuhn
from paper_2602_23613_b200.multilevel import _device_for

pytestmark = pytest.mark.gpu

PC_DOWN, PC_RESTRICT, PC_COARSE, PC_PROLONG, PC_UP = range(5)


def vcycle_pieces(depth):
    seq = []

    def rec(lv):
        if lv == depth - 1:
            seq.append((lv, PC_COARSE))
            return
        seq.extend([(lv, PC_DOWN), (lv, PC_RESTRICT)])
        rec(lv + 1)
        seq.extend([(lv, PC_PROLONG), (lv, PC_UP)])

    rec(0)
    return seq


@pytest.fixture(autouse=True)
def explicit_z(monkeypatch):
    # the row-partitioned solve streams the explicit block Z; compare it with the
    # single-GPU V-cycle on the same representation (the single-GPU default
    # applies A_GG^{-1} through the factor, tests/test_gpu_factor_sweep.py)
    monkeypatch.setenv("HCAMG_PAPPLY", "z")
    # likewise the coarsest inverse: the row-partitioned solve streams the full
    # matrix; the single-GPU default reads its lower triangle (test_gpu_symv.py)
    monkeypatch.setenv("HCAMG_COARSE_SYMV", "0")


@pytest.fixture(scope="module")
def system16():
    return kuhn.config_system("c1", 16)


@pytest.fixture()
def coarse_exchange(monkeypatch):
    # route every coarsest solve through the row GEMV so its exchange is exercised
    monkeypatch.setenv("HCAMG_COARSE_GEMV_MIN", "0")


def _prepare(h, rank, nranks):
    dev = _device_for(h)
    p = C.c_void_p()
    dev.check(dev.lib.hcamg_dist_prepare(dev.h, rank, nranks, None, C.byref(p)))
    return p.value


def _connect_ptrs(h, ptrs):
    dev = _device_for(h)
    arr = (C.c_void_p * len(ptrs))(*ptrs)
    dev.check(dev.lib.hcamg_dist_connect_ptrs(dev.h, arr))


def _piece(h, level, piece, part, b=None, x=None):
    dev = _device_for(h)
    dev.check(dev.lib.hcamg_debug_dist_piece(dev.h, level, piece, part,
                                             None if b is None else b.ctypes.data,
                                             None if x is None else x.ctypes.data))


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_emulated_ranks_vcycle_bitwise(system16, coarse_exchange, nranks):
    b = np.random.default_rng(3).uniform(-1, 1, system16.n)
    ref = P.build_hierarchy(system16, "alg")
    assert max(lv._info.max_component for lv in ref.levels[:-1]) > 4096  # a dense-regime level
    x_ref = P.vcycle(ref, b)
    ranks = [P.build_hierarchy(system16, "alg") for _ in range(nranks)]
    ptrs = [_prepare(h, r, nranks) for r, h in enumerate(ranks)]
    for h in ranks:
        _connect_ptrs(h, ptrs)
    for r, h in enumerate(ranks):
        assert dist.info(h)[:3] == (r, nranks, True)
    for i, (lv, pc) in enumerate(vcycle_pieces(ranks[0].depth)):
        for part in (1, 2):
            for h in ranks:
                _piece(h, lv, pc, part, b=b if i == 0 and part == 1 else None)
    for h in ranks:
        x = np.empty(system16.n)
        _piece(h, 0, -1, 0, x=x)
        assert np.array_equal(x, x_ref)


def test_one_rank_exchange_pcg_amg_vcycle_bitwise(system16, coarse_exchange):
    b = np.random.default_rng(0).uniform(-1, 1, system16.n)
    ref = P.build_hierarchy(system16, "alg")
    x0, rep0 = P.pcg(system16.A, b, precond=lambda r: P.vcycle(ref, r), tol=1e-8)
    a0, arep0 = P.amg_solve(ref, b, tol=1e-6, maxit=40)
    v0 = P.vcycle(ref, b)

    h = P.build_hierarchy(system16, "alg")
    _connect_ptrs(h, [_prepare(h, 0, 1)])
    x1, rep1 = P.pcg(system16.A, b, precond=lambda r: P.vcycle(h, r), tol=1e-8)
    assert rep1.iterations == rep0.iterations and rep1.converged
    assert np.array_equal(x1, x0)
    assert np.array_equal(rep1.residual_history, rep0.residual_history)
    a1, arep1 = P.amg_solve(h, b, tol=1e-6, maxit=40)
    assert np.array_equal(a1, a0) and arep1.iterations == arep0.iterations
    assert np.array_equal(P.vcycle(h, b), v0)
    # and back
    dist.undistribute(h)
    assert dist.info(h)[2] is False
    assert np.array_equal(P.vcycle(h, b), v0)


def test_distribute_world_of_one(system16):
    import os

    import torch.distributed as tdist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29631")
    created = False
    if not tdist.is_initialized():
        tdist.init_process_group("gloo", rank=0, world_size=1)
        created = True
    try:
        b = np.random.default_rng(1).uniform(-1, 1, system16.n)
        ref = P.build_hierarchy(system16, "alg")
        x0, rep0 = P.pcg(system16.A, b, precond=lambda r: P.vcycle(ref, r), tol=1e-8)
        h = P.build_hierarchy(system16, "alg")
        dist.distribute(h)
        assert dist.info(h)[:3] == (0, 1, True)
        x1, rep1 = P.pcg(system16.A, b, precond=lambda r: P.vcycle(h, r), tol=1e-8)
        assert np.array_equal(x1, x0) and rep1.iterations == rep0.iterations
    finally:
        if created:
            tdist.destroy_process_group()


def test_prepare_validates(system16):
    h = P.build_hierarchy(system16, "alg")
    dev = _device_for(h)
    p = C.c_void_p()
    assert dev.lib.hcamg_dist_prepare(dev.h, 2, 2, None, C.byref(p)) != 0
    assert dev.lib.hcamg_dist_prepare(dev.h, 0, 9, None, C.byref(p)) != 0
    assert dev.lib.hcamg_dist_connect_ptrs(dev.h, None) != 0


def _odd_dense_system(n=4097):
    import scipy.sparse as sp
    rng = np.random.default_rng(11)
    main = 2.5 + rng.uniform(0, 1, n)
    off = -np.ones(n - 1)
    return sp.csr_matrix(sp.diags([off, main, off], [-1, 0, 1]))


@pytest.mark.parametrize("zrows", ["1", "0"])
def test_row_gemv_odd_width_unaligned_rows(monkeypatch, zrows):
    """n = 4097 (odd): every other row of the row-major inverse starts 8 bytes
    off a 16-byte boundary; both row-GEMV kernels must handle it."""
    monkeypatch.setenv("HCAMG_COARSE_GEMV_MIN", "0")
    monkeypatch.setenv("HCAMG_ZROWS", zrows)
    A = _odd_dense_system()
    h = P.Hierarchy([P.Level(A=A)], "alg")
    b = np.random.default_rng(2).uniform(-1, 1, A.shape[0])
    x = P.vcycle(h, b)
    xr = np.linalg.solve(A.toarray(), b)
    assert np.linalg.norm(x - xr) <= 1e-12 * np.linalg.norm(xr)


@pytest.mark.parametrize("nranks", [2, 3])
def test_emulated_ranks_wide_coarse_exchange(monkeypatch, nranks):
    """Row-batched GEMV (n >= 4096, odd n) in exchange mode, emulated ranks."""
    monkeypatch.setenv("HCAMG_COARSE_GEMV_MIN", "0")
    A = _odd_dense_system()
    b = np.random.default_rng(4).uniform(-1, 1, A.shape[0])
    x_ref = P.vcycle(P.Hierarchy([P.Level(A=A)], "alg"), b)
    ranks = [P.Hierarchy([P.Level(A=A.copy())], "alg") for _ in range(nranks)]
    ptrs = [_prepare(h, r, nranks) for r, h in enumerate(ranks)]
    for h in ranks:
        _connect_ptrs(h, ptrs)
    for part in (1, 2):
        for h in ranks:
            _piece(h, 0, PC_COARSE, part, b=b if part == 1 else None)
    for h in ranks:
        x = np.empty(A.shape[0])
        _piece(h, 0, -1, 0, x=x)
        assert np.array_equal(x, x_ref)
