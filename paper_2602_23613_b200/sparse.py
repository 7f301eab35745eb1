"""Sparse-core pieces of the drop-in API (hcurl_amg/sparse.py): the canonical
CSR normal form, the breakdown exception, and a device-backed coarsest-level
Cholesky factor (``cholesky`` / ``solve``, sparse.py:276-321)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _lib

__all__ = ["NotPositiveDefiniteError", "csr", "max_abs", "cholesky", "solve", "CholeskyFactor", "raise_for"]


class NotPositiveDefiniteError(RuntimeError):
    """Cholesky pivot breakdown; ``pivot`` is the failing index (sparse.py:50-55)."""

    def __init__(self, pivot, message=None):
        self.pivot = int(pivot)
        super().__init__(message or f"matrix is not positive definite (pivot {pivot})")


def csr(a, shape=None):
    """Canonical CSR input normal form: sorted, duplicates summed, exact zeros
    removed (sparse.py:58-65).  Host-side argument normalisation only."""
    m = sp.csr_matrix(a, shape=shape, dtype=np.float64)
    m.sum_duplicates()
    m.sort_indices()
    m.eliminate_zeros()
    return m


def max_abs(A):
    return float(np.max(np.abs(A.data))) if A.nnz else 0.0


def raise_for(rc, msg, index=-1):
    """Map a libhcamg status code to the reference's exception types."""
    if rc in (_lib.EINVAL, _lib.ENOTSYM):
        raise ValueError(msg)
    if rc == _lib.ENOTSPD:
        raise NotPositiveDefiniteError(index, msg)
    if rc == _lib.EBREAKDOWN:
        raise RuntimeError(msg)
    if rc == _lib.EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == _lib.ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"libhcamg error {rc}: {msg}")


class CholeskyFactor:
    """Device-resident factor of an SPD matrix (sparse.py:146-165).

    The factorisation runs on the GPU (symmetry check to 1e-12, blocked
    Cholesky with the 1e-13 relative pivot floor) and the solve applies the
    resident inverse.  ``ordering`` (reverse Cuthill-McKee) and ``factor``
    (lower-triangular CSR L with L L^T = A[ordering][:, ordering]) -- the
    reference's fields -- are materialised from the device on first access.
    """

    def __init__(self, matrix, dev=None, level=0):
        self.matrix = matrix
        self._dev = dev
        self._level = level
        self._n = matrix.shape[0] if matrix is not None else 0
        self._ord = None
        self._fac = None

    @property
    def n(self):
        return self._n

    def _materialise(self):
        if self._ord is None:
            n = self.n
            ordering = np.empty(max(n, 1), dtype=np.int64)
            L = np.empty((n, n), dtype=np.float64)
            dev = self._dev
            dev.check(dev.lib.hcamg_cholesky_factor(dev.h, int(self._level), _lib.ptr(ordering), _lib.ptr(L)))
            self._ord = ordering[:n].copy()
            self._fac = csr(L)
        return self._ord, self._fac

    @property
    def ordering(self):
        return self._materialise()[0]

    @property
    def factor(self):
        return self._materialise()[1]

    @classmethod
    def _from_level(cls, dev, idx, n):
        f = cls(None, dev, idx)
        f._n = n
        return f

    @staticmethod
    def matrix_of(cf):
        """The matrix a coarse factor inverts (ours, or a reference-style
        CholeskyFactor(ordering, factor) rebuilt as P^T L L^T P)."""
        if isinstance(cf, CholeskyFactor):
            if cf.matrix is None and cf._dev is not None:
                from .multilevel import _level_matrix
                return _level_matrix(cf._dev, cf._level)
            return cf.matrix
        L = getattr(cf, "factor", None)
        perm = getattr(cf, "ordering", None)
        if L is None or perm is None:
            return None
        L = sp.csr_matrix(L)
        M = (L @ L.T).tocsr()
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(perm))
        return csr(M[inv][:, inv])


def cholesky(A, check_symmetry=True):
    """Factor an SPD matrix on the device (sparse.py:276-301).  Raises
    ValueError for an asymmetric input and NotPositiveDefiniteError(pivot)."""
    from .multilevel import _Device  # local import: avoid a cycle

    A = csr(A)
    if A.shape[0] != A.shape[1]:
        raise ValueError("matrix must be square")
    dev = _Device(0)
    H = _lib.HostCSR(A)
    dev.check(dev.lib.hcamg_hier_begin(dev.h))
    dev.check(dev.lib.hcamg_hier_push(dev.h, H.ref(), None, None))
    info = _lib.Info()
    dev.check(dev.lib.hcamg_hier_end(dev.h, C.byref(info)))
    return CholeskyFactor(A, dev, 0)


def solve(factor, b):
    """Solve A x = b with a device factor (sparse.py:304-321); ``b`` may be a
    vector or an n x k block of right-hand sides."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape[0] != factor.n:
        raise ValueError(f"dimension mismatch: factor {factor.n}, rhs {b.shape}")
    if factor.n == 0:
        return b.copy()
    dev = factor._dev
    cols = b.reshape(b.shape[0], -1)
    out = np.empty_like(cols)
    for j in range(cols.shape[1]):
        bj = np.ascontiguousarray(cols[:, j])
        xj = np.empty_like(bj)
        dev.check(dev.lib.hcamg_coarse_solve(dev.h, int(factor._level), _lib.ptr(bj), _lib.ptr(xj)))
        out[:, j] = xj
    return out.reshape(b.shape)
