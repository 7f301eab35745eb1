"""Row-partitioned multi-GPU solve — host side.

The reference is single-process (no communication layer exists); this module is
what a multi-GPU caller of the drop-in adds after ``build_hierarchy``:

    h = build_hierarchy(system, "alg", device=local_rank)   # every rank, same system
    distribute(h)                                           # collective
    x, rep = pcg(system.A, b, precond=lambda r: vcycle(h, r))  # collective, as before

Every rank holds the same hierarchy (the setup is replicated: its greedy
splittings are global sequential greedies).  In the solve, each
rank streams only its rows of every dense interpolation block Z and of the
coarsest inverse, and the kernels that produce those rows store them straight
into every peer's exchange buffer (CUDA IPC over NVLink) and raise a flag there;
the consuming kernels wait for all flags.  The restriction reduces its row-chunk
partials in ``GROUPS`` fixed groups, so the solution is bit-identical to the
single-GPU solve for every rank count (1..8).

The handle exchange rides on ``torch.distributed`` (any backend; 64 bytes per
rank).  ``plan`` mirrors the C++ partition (giant.cu ``hybrid_prepare``,
dist.cuh ``rank_groups`` / ``even_rows``) so the host logic is testable without
a GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from .multilevel import _device_for

GROUPS = 8          # dist.cuh kGroups
MAX_RANKS = 8       # dist.cuh kMaxRanks
SMS = 148           # common.cuh kSMs
ZT_COLS = 1024      # giant.cu kZtCols
IPC_HANDLE_BYTES = 64


@dataclass(frozen=True)
class RankPlan:
    chunk: int          # rows per restriction chunk
    nchunk: int
    groups: tuple       # chunk boundaries of the GROUPS groups (GROUPS + 1 entries)
    g0: int             # groups [g0, g1) of this rank
    g1: int
    rows: tuple         # rows [q0, q1) of Z streamed by this rank
    coarse_rows: tuple  # rows [r0, r1) of an n_coarse-row coarsest inverse


def plan(nG: int, nc: int, rank: int, nranks: int, n_coarse: int = 0) -> RankPlan:
    """The partition of one dense-regime level (and the coarsest inverse)."""
    if not (1 <= nranks <= MAX_RANKS) or not (0 <= rank < nranks):
        raise ValueError("rank / nranks out of range (1..8 ranks)")
    ct = max(1, (nc + ZT_COLS - 1) // ZT_COLS)
    per_group = max(1, (4 * SMS + ct - 1) // ct)
    want = GROUPS * per_group
    chunk = max(16, min(4096, (nG + want - 1) // want))
    nchunk = (nG + chunk - 1) // chunk
    grp = tuple(nchunk * g // GROUPS for g in range(GROUPS + 1))
    g0, g1 = GROUPS * rank // nranks, GROUPS * (rank + 1) // nranks
    rows = (min(nG, grp[g0] * chunk), min(nG, grp[g1] * chunk))
    coarse = (n_coarse * rank // nranks, n_coarse * (rank + 1) // nranks)
    return RankPlan(chunk, nchunk, grp, g0, g1, rows, coarse)


def representation(nG: int, nc: int, factor_bytes: int, n_coarse: int, coarse_symv: bool, nranks: int):
    """Which pieces the distributed solve splits across ranks (mirrors
    capi.cu ``hcamg_dist_prepare``): the dense block when its per-rank row
    block (2 x 8 nG nc / N bytes per V-cycle) is smaller than applying it
    through the envelope factor on every rank (2 x factor_bytes; 0: no
    factor, always split); the coarsest solve when 8 n^2 / N beats the packed
    lower triangle (4 n^2).  Returns (split_dense, split_coarse)."""
    z_rank = 2.0 * 8.0 * nG * nc / nranks
    fac = 2.0 * factor_bytes if factor_bytes > 0 else float("inf")
    rows = 8.0 * n_coarse * n_coarse / nranks
    packed = 4.0 * n_coarse * n_coarse if coarse_symv else float("inf")
    return (nG > 0 and z_rank < fac), (n_coarse > 0 and rows < packed)


def exchange_handles(local: bytes, group=None) -> bytes:
    """All-gather every rank's IPC handle, concatenated in rank order."""
    import torch.distributed as dist

    if len(local) != IPC_HANDLE_BYTES:
        raise ValueError("an IPC handle is 64 bytes")
    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, bytes(local), group=group)
    if any(o is None or len(o) != IPC_HANDLE_BYTES for o in out):
        raise RuntimeError("handle exchange failed")
    return b"".join(out)


def distribute(h, group=None):
    """Make the solve of ``h`` collective over ``group`` (torch.distributed).

    Every rank must have built ``h`` from the same system with the same
    options; afterwards ``vcycle`` / ``pcg`` / ``amg_solve`` on ``h`` must be
    called by all ranks in the same order."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _device_for(h)
    handle = (C.c_char * IPC_HANDLE_BYTES)()
    dptr = C.c_void_p()
    dev.check(dev.lib.hcamg_dist_prepare(dev.h, rank, world, handle, C.byref(dptr)))
    allh = exchange_handles(bytes(handle), group)
    buf = C.create_string_buffer(allh, len(allh))
    dev.check(dev.lib.hcamg_dist_connect(dev.h, buf))
    h._dist = (rank, world)
    return h


def undistribute(h):
    """Back to the single-GPU solve (local; no communication)."""
    dev = _device_for(h)
    dev.check(dev.lib.hcamg_dist_disconnect(dev.h))
    h._dist = None
    return h


def info(h):
    """(rank, nranks, connected, exchange buffer bytes) of ``h``'s handle."""
    dev = _device_for(h)
    r, n, c, b = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
    dev.check(dev.lib.hcamg_dist_info(dev.h, C.byref(r), C.byref(n), C.byref(c), C.byref(b)))
    return r.value, n.value, bool(c.value), b.value
