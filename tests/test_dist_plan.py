"""Host logic of the row-partitioned multi-GPU solve, on the CPU.

* ``dist.plan`` (the mirror of the C++ partition) covers every row of Z and of
  the coarsest inverse exactly once, ranks own whole chunk groups, and the
  chunking does not depend on the rank count;
* with world_size 2 over gloo: the IPC-handle exchange returns every rank's
  handle in rank order, and the exchange protocol applied to the restriction
  and prolongation of a dense block -- each rank computes only its rows /
  groups, the slices are all-gathered, the consumer folds them -- gives the
  single-process result bit for bit (numpy stands in for the kernels).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as tdist
import torch.multiprocessing as mp

from paper_2602_23613_b200 import dist


@pytest.mark.parametrize("nG,nc", [(20520, 2948), (167784, 26236), (100, 7), (5000, 40000), (16, 3)])
@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 5, 8])
def test_plan_partitions(nG, nc, nranks):
    plans = [dist.plan(nG, nc, r, nranks, n_coarse=nc) for r in range(nranks)]
    base = dist.plan(nG, nc, 0, 1, n_coarse=nc)
    for p in plans:
        assert (p.chunk, p.nchunk, p.groups) == (base.chunk, base.nchunk, base.groups)
    assert plans[0].rows[0] == 0 and plans[-1].rows[1] == nG
    assert plans[0].coarse_rows[0] == 0 and plans[-1].coarse_rows[1] == nc
    for a, b in zip(plans, plans[1:]):
        assert a.rows[1] == b.rows[0] and a.g1 == b.g0 and a.coarse_rows[1] == b.coarse_rows[0]
    for p in plans:
        assert p.rows[0] == min(nG, p.groups[p.g0] * p.chunk)
    assert base.groups[0] == 0 and base.groups[-1] == base.nchunk
    assert base.nchunk * base.chunk >= nG > (base.nchunk - 1) * base.chunk


def test_plan_rejects_bad_ranks():
    with pytest.raises(ValueError):
        dist.plan(10, 10, 0, 9)
    with pytest.raises(ValueError):
        dist.plan(10, 10, 2, 2)


def _chunk_partials(Z, r, p):
    """partial[ch] = sum over the chunk's rows, row by row (the kernel's order is
    its own; what matters here is that every rank uses the same function)."""
    out = np.zeros((p.nchunk, Z.shape[1]))
    for ch in range(p.nchunk):
        acc = np.zeros(Z.shape[1])
        for q in range(ch * p.chunk, min(Z.shape[0], (ch + 1) * p.chunk)):
            acc = acc + Z[q] * r[q]
        out[ch] = acc
    return out


def _group_sums(partial, p, g0, g1):
    gs = np.zeros((dist.GROUPS, partial.shape[1]))
    for g in range(g0, g1):
        acc = np.zeros(partial.shape[1])
        for ch in range(p.groups[g], p.groups[g + 1]):
            acc = acc + partial[ch]
        gs[g] = acc
    return gs


def _fold(gs):
    acc = np.zeros(gs.shape[1])
    for g in range(dist.GROUPS):
        acc = acc + gs[g]
    return acc


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # handle exchange
        local = bytes([rank + 1]) * dist.IPC_HANDLE_BYTES
        allh = dist.exchange_handles(local)
        ok_handles = allh == b"".join(bytes([r + 1]) * 64 for r in range(world))

        # same seeded block on every rank
        rng = np.random.default_rng(7)
        nG, nc = 3000, 37
        Z = rng.standard_normal((nG, nc))
        rG = rng.standard_normal(nG)
        ec = rng.standard_normal(nc)
        p = dist.plan(nG, nc, rank, world)
        # single-process reference (every group, every row)
        ref_partial = _chunk_partials(Z, rG, p)
        ref_bc = _fold(_group_sums(ref_partial, p, 0, dist.GROUPS))
        ref_y = np.array([Z[q] @ ec for q in range(nG)])
        # distributed: my chunks / groups / rows only, then all-gather
        mine = np.zeros_like(ref_partial)
        lo, hi = p.groups[p.g0], p.groups[p.g1]
        mine[lo:hi] = ref_partial[lo:hi]   # chunk partials do not depend on the rank
        gs = _group_sums(mine, p, p.g0, p.g1)
        gathered = [None] * world
        tdist.all_gather_object(gathered, (p.g0, p.g1, gs[p.g0:p.g1]))
        full = np.zeros_like(gs)
        for g0, g1, block in gathered:
            full[g0:g1] = block
        bc = _fold(full)
        q0, q1 = p.rows
        ymine = np.array([Z[q] @ ec for q in range(q0, q1)])
        ys = [None] * world
        tdist.all_gather_object(ys, (q0, q1, ymine))
        y = np.zeros(nG)
        for a, b, v in ys:
            y[a:b] = v
        q.put((rank, ok_handles, bool(np.array_equal(bc, ref_bc)), bool(np.array_equal(y, ref_y))))
    finally:
        tdist.destroy_process_group()


def test_two_rank_exchange_over_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, ok_h, ok_bc, ok_y in sorted(res):
        assert ok_h, f"rank {rank}: handles out of order"
        assert ok_bc, f"rank {rank}: restriction differs"
        assert ok_y, f"rank {rank}: prolongation differs"


def test_representation_per_rank_count():
    """Config 2: the explicit Z (167,784 x 26,236, 35.2 GB)
    is split only when a rank's row block beats the 11.1 GB of envelope-factor
    sweeps every V-cycle applies twice -- from 4 ranks on; the 26,236^2 coarsest
    inverse only when its rows beat the packed triangle -- from 3 ranks on."""
    from paper_2602_23613_b200.dist import representation
    nG, nc, fac, ncs = 167784, 26236, 5337000000 + 5792000000, 26236
    got = {N: representation(nG, nc, fac, ncs, True, N) for N in range(1, 9)}
    assert [N for N in got if got[N][0]] == [4, 5, 6, 7, 8]
    assert [N for N in got if got[N][1]] == [3, 4, 5, 6, 7, 8]
    # without the factor / packed triangle every piece is split (the round-1 layout)
    assert all(representation(nG, nc, 0, ncs, False, N) == (True, True) for N in range(1, 9))
