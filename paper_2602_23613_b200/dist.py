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


# ----------------------------------------------------------------------------------------------
# Subdomain row partition of the sparse regime (the north-star layout, csrc/rows.cuh)
# ----------------------------------------------------------------------------------------------

SEGMENTS = ("vcycle", "pcg_init", "pcg_first", "pcg_body", "gather", "amg_init", "amg_body")


def distribute_rows(h, group=None, min_rows=16384):
    """Partition the solve of ``h`` by rows over ``group`` (torch.distributed).

    Every level with at least ``min_rows`` rows is split into one subdomain per
    rank; coarser levels are agglomerated (every rank keeps them whole).  Every
    rank must have built ``h`` from the same system; afterwards ``vcycle`` and
    ``pcg`` on ``h`` are collective.  Each rank passes the full right-hand side
    and receives the full solution."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _device_for(h)
    handle = (C.c_char * IPC_HANDLE_BYTES)()
    dptr = C.c_void_p()
    dev.check(dev.lib.hcamg_rows_prepare(dev.h, rank, world, int(min_rows), handle, C.byref(dptr)))
    allh = exchange_handles(bytes(handle), group)
    buf = C.create_string_buffer(allh, len(allh))
    dev.check(dev.lib.hcamg_rows_connect(dev.h, buf))
    h._dist = (rank, world)
    return h


def undistribute_rows(h):
    dev = _device_for(h)
    dev.check(dev.lib.hcamg_rows_disconnect(dev.h))
    h._dist = None
    return h


def rows_info(h):
    """Partition statistics of ``h``'s handle (hcamg_rows_info)."""
    import numpy as np

    dev = _device_for(h)
    out = np.zeros(7 + 4 * len(SEGMENTS), dtype=np.int64)
    dev.check(dev.lib.hcamg_rows_info(dev.h, out.ctypes.data, len(out)))
    info = dict(rank=int(out[0]), nranks=int(out[1]), connected=bool(out[2]), split_levels=int(out[3]),
                buffer_bytes=int(out[4]), own_rows0=int(out[5]), ghost_cols0=int(out[6]), segments={})
    for g, name in enumerate(SEGMENTS):
        s = out[7 + 4 * g: 11 + 4 * g]
        info["segments"][name] = dict(steps=int(s[0]), barriers=int(s[1]), push_out=int(s[2]), push_all=int(s[3]))
    return info


def emulate_rows(hs, b, kind="vcycle", tol=1e-8, maxit=500, min_rows=64, poison=True):
    """Lockstep emulation of a ``len(hs)``-rank partitioned solve on ONE GPU.

    ``hs``: hierarchies built from the same system on the same device (one
    handle each).  Prepares them as ranks 0..n-1, connects them through raw
    device pointers and runs the step program rank after rank (every rank's
    boundary push, then every rank's kernel), so no kernel waits for one that
    has not run.  Returns (X, report): X[r] = the full result as rank r holds
    it; report is None for a V-cycle."""
    import numpy as np
    from . import _lib

    n = len(hs)
    devs = [_device_for(h) for h in hs]
    ptrs = []
    for r, dev in enumerate(devs):
        p = C.c_void_p()
        dev.check(dev.lib.hcamg_rows_prepare(dev.h, r, n, int(min_rows), None, C.byref(p)))
        ptrs.append(p.value)
    arr = (C.c_void_p * n)(*ptrs)
    for dev in devs:
        dev.check(dev.lib.hcamg_rows_connect_ptrs(dev.h, arr))
    handles = (C.c_void_p * n)(*[dev.h for dev in devs])
    b = np.ascontiguousarray(b, dtype=np.float64)
    X = np.empty((n, b.shape[0]))
    rep = _lib.Report()
    devs[0].check(devs[0].lib.hcamg_rows_emulate(handles, n, {"vcycle": 0, "pcg": 1, "amg": 2}[kind], b.ctypes.data,
                                                 X.ctypes.data, float(tol), int(maxit), 1 if poison else 0,
                                                 C.byref(rep)))
    return X, (None if kind == "vcycle" else rep)


class Plan:
    """The partition's dataflow planner (host only; csrc/rows_plan.cu)."""

    def __init__(self, nranks, vec_len):
        import numpy as np
        from . import _lib

        self.lib = _lib.load()
        self.nranks = int(nranks)
        lens = np.ascontiguousarray(vec_len, dtype=np.int64)
        self.p = C.c_void_p()
        rc = self.lib.hcamg_plan_create(C.byref(self.p), self.nranks, len(lens), lens.ctypes.data)
        if rc != 0:
            raise ValueError("hcamg_plan_create failed")

    def close(self):
        if self.p:
            self.lib.hcamg_plan_destroy(self.p)
            self.p = None

    __del__ = close

    def set_vector(self, vec, mask, owner=None):
        import numpy as np

        o = None if owner is None else np.ascontiguousarray(owner, dtype=np.int8)
        if self.lib.hcamg_plan_set_vector(self.p, int(vec), int(mask), None if o is None else o.ctypes.data) != 0:
            raise ValueError("hcamg_plan_set_vector failed")

    def invalidate(self, vec):
        if self.lib.hcamg_plan_invalidate(self.p, int(vec)) != 0:
            raise ValueError("hcamg_plan_invalidate failed")

    def step(self, reads, writes):
        """reads / writes: per rank a list of (vec, index array) pairs."""
        import numpy as np

        def flat(acc):
            cnt, vs, ix = [], [], []
            for per_rank in acc:
                c = 0
                for vec, idx in per_rank:
                    idx = np.asarray(idx, dtype=np.int32).ravel()
                    vs.append(np.full(idx.shape, vec, dtype=np.int32))
                    ix.append(idx)
                    c += idx.size
                cnt.append(c)
            cat = lambda a: np.ascontiguousarray(np.concatenate(a) if a else np.zeros(0, np.int32), dtype=np.int32)
            return np.asarray(cnt, dtype=np.int64), cat(vs), cat(ix)

        nr, rv, ri = flat(reads)
        nw, wv, wi = flat(writes)
        if self.lib.hcamg_plan_step(self.p, nr.ctypes.data, rv.ctypes.data, ri.ctypes.data,
                                    nw.ctypes.data, wv.ctypes.data, wi.ctypes.data) != 0:
            raise ValueError("hcamg_plan_step failed")

    def pushes(self):
        """[(boundary, src, dst, vec, indices)], and the number of reads of undefined entries."""
        import numpy as np

        counts = np.zeros(3, dtype=np.int64)
        self.lib.hcamg_plan_counts(self.p, counts.ctypes.data)
        seg = np.zeros((int(counts[0]), 5), dtype=np.int32)
        idx = np.zeros(int(counts[1]), dtype=np.int32)
        self.lib.hcamg_plan_pushes(self.p, seg.ctypes.data, idx.ctypes.data)
        out, o = [], 0
        for b, s, d, v, c in seg:
            out.append((int(b), int(s), int(d), int(v), idx[o:o + c].copy()))
            o += c
        return out, int(counts[2])


def rows_owner(A, nranks):
    """owner[u] = rank of row u: BFS slabs of A's graph with equal nonzero counts (hcamg_rows_owner)."""
    import numpy as np
    from . import _lib

    lib = _lib.load()
    A = A.tocsr()
    ptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
    idx = np.ascontiguousarray(A.indices, dtype=np.int32)
    owner = np.zeros(A.shape[0], dtype=np.int8)
    if lib.hcamg_rows_owner(A.shape[0], ptr.ctypes.data, idx.ctypes.data, int(nranks), owner.ctypes.data) != 0:
        raise ValueError("hcamg_rows_owner failed")
    return owner
