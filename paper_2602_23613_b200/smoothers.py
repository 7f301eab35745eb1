"""Drop-in for ``hcurl_amg.smoothers`` (smoothers.py): the OSS-l1 smoother --
vertex-patch multiplicative Schwarz followed by one l1-Jacobi step -- run by
the device smoothing legs of libhcamg.

* ``build_patches(A, G_level)`` (smoothers.py:60-95) builds the patches, their
  inverses and the wavefront schedule on the GPU (``hcamg_smoother_setup``);
* ``build_l1_jacobi(A)`` (smoothers.py:50-52);
* ``smooth(A, patches, l1, x, b, direction)`` (smoothers.py:112-137) applies
  one forward / backward / symmetric OSS-l1 step on the device
  (``hcamg_smooth``), with the reference's exact multiplicative order.

``PatchSet`` keeps the reference's fields (``patches``, ``factors``,
``update_rows``, ``update_blocks``, smoothers.py:26-40).  The device holds the
patches and their explicit inverses; the reference-layout fields are
materialised on first access for inspection only (the dense patch Cholesky
factors are those of ``A[patch, patch]``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import _lib
from .sparse import NotPositiveDefiniteError, csr

__all__ = ["PatchSet", "L1Jacobi", "build_patches", "build_l1_jacobi", "smooth"]

_DIRECTIONS = {"forward": 0, "backward": 1, "symmetric": 2}


class PatchSet:
    """Per-node edge patches (smoothers.py:26-40) backed by a device level.

    ``patches`` is the reference's list (vertex patches in column order, then
    singletons); ``waves`` the wavefront each patch runs in on the GPU.
    """

    def __init__(self, patches, waves, A=None, dev=None, level=0):
        self.patches = patches
        self.waves = waves
        self._A = A
        self._dev = dev
        self._level = level
        self._ref = None

    def _matrix(self):
        if self._A is None and self._dev is not None:
            from .multilevel import _level_matrix
            self._A = _level_matrix(self._dev, self._level)
        return self._A

    def _reference_fields(self):
        if self._ref is None:
            A = self._matrix()
            Ac = A.tocsc()
            factors, rows_l, blocks = [], [], []
            for pid, p in enumerate(self.patches):
                cols = Ac[:, p]
                rows = np.unique(cols.indices)
                blk = np.asarray(cols[rows, :].todense())
                try:
                    factors.append(np.linalg.cholesky(blk[np.searchsorted(rows, p), :]))
                except np.linalg.LinAlgError as err:
                    raise NotPositiveDefiniteError(0, f"singular patch block {pid}") from err
                rows_l.append(rows)
                blocks.append(blk)
            self._ref = (factors, rows_l, blocks)
        return self._ref

    @property
    def factors(self):
        return self._reference_fields()[0]

    @property
    def update_rows(self):
        return self._reference_fields()[1]

    @property
    def update_blocks(self):
        return self._reference_fields()[2]


@dataclass
class L1Jacobi:
    """Diagonal l1 smoother, d_i = sum_j |A_ij| (smoothers.py:43-52)."""

    d: np.ndarray


def build_l1_jacobi(A):
    """smoothers.py:50-52 (the device level computes the same sums; this is
    the host-side value object the reference API returns)."""
    return L1Jacobi(np.asarray(abs(csr(A)).sum(axis=1)).ravel())


def _export_patches(dev, level, li):
    m, ne = int(li.n_patches), int(li.n_patch_entries)
    pp = np.empty(m + 1, dtype=np.int64)
    dofs = np.empty(max(ne, 1), dtype=np.int64)
    wave = np.empty(max(m, 1), dtype=np.int64)
    dev.check(dev.lib.hcamg_export_patches(dev.h, int(level), _lib.ptr(pp), _lib.ptr(dofs), _lib.ptr(wave)))
    return [dofs[pp[t]:pp[t + 1]].copy() for t in range(m)], wave[:m].copy()


def build_patches(A, G_level, device=0):
    """Vertex patches, patch inverses and the wavefront schedule of one level
    on the GPU (smoothers.py:60-95).  Raises NotPositiveDefiniteError for a
    singular patch block, as the reference does."""
    from .multilevel import _Device

    A, G = csr(A), csr(G_level)
    if A.shape[0] != A.shape[1] or G.shape[0] != A.shape[0]:
        raise ValueError("dimension mismatch: A and G")
    dev = _Device(device)
    hA, hG = _lib.HostCSR(A), _lib.HostCSR(G)
    dev.check(dev.lib.hcamg_smoother_setup(dev.h, hA.ref(), hG.ref()))
    li = dev.level_info(0)
    patches, waves = _export_patches(dev, 0, li)
    return PatchSet(patches, waves, A, dev, 0)


def smooth(A, patches, l1, x, b, direction="forward"):
    """One OSS-l1 application on the device; returns the updated iterate
    (smoothers.py:112-137).  ``patches`` must come from ``build_patches`` or
    from a level of a device hierarchy (``h.levels[l].patches``); the device
    l1 diagonal of that level is the one applied."""
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    n = A.shape[0]
    if n != len(b) or len(x) != len(b):
        raise ValueError("shape mismatch")
    if direction not in _DIRECTIONS:
        raise ValueError(f"unknown direction {direction!r}")
    dev = getattr(patches, "_dev", None)
    if dev is None:
        raise TypeError("patches must come from build_patches() or a device hierarchy level")
    out = np.empty_like(b)
    dev.check(dev.lib.hcamg_smooth(dev.h, int(patches._level), _DIRECTIONS[direction], _lib.ptr(x), _lib.ptr(b),
                                   _lib.ptr(out)))
    return out
