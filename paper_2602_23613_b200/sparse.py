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

    The factorisation itself runs on the GPU (symmetry check to 1e-12,
    blocked Cholesky with the 1e-13 relative pivot floor); the matrix is
    kept so a user-assembled hierarchy can attach it as ``coarse_factor``.
    """

    def __init__(self, matrix, dev=None):
        self.matrix = matrix
        self._dev = dev

    @property
    def n(self):
        return self.matrix.shape[0] if self.matrix is not None else self._n

    @property
    def ordering(self):
        return np.arange(self.n, dtype=np.int64)

    @classmethod
    def _from_level(cls, dev, idx, n):
        f = cls.__new__(cls)
        f._dev = dev
        f._level = idx
        f.matrix = None
        f._n = n
        return f

    @staticmethod
    def matrix_of(cf):
        """The matrix a coarse factor inverts (ours, or a reference-style
        CholeskyFactor(ordering, factor) rebuilt as P^T L L^T P)."""
        if isinstance(cf, CholeskyFactor):
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
    return CholeskyFactor(A, dev)


def solve(factor, b):
    """Apply the factor's inverse (sparse.py:304-321)."""
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    if b.shape[0] != factor.n:
        raise ValueError(f"dimension mismatch: factor {factor.n}, rhs {b.shape}")
    out = np.empty_like(b)
    dev = factor._dev
    dev.check(dev.lib.hcamg_vcycle(dev.h, _lib.ptr(b), None, _lib.ptr(out)))
    return out
