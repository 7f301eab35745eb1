"""SpGEMM paths against scipy, bit for bit (csrc/sparse.cu).

The dense-regime coarse operator (BASELINE configs[1]: 26,236^2 entries) is a
CSR with every entry stored; its nodal dual G~^T (A G~) (splitting.py:128-133)
takes the dense-left product (spgemm_dense_left): one thread per output entry,
summed over the rows of G~'s column in ascending order -- scipy's csr_matmat
order, product rounded, then added.  The row kernels (k_spgemm_count / fill)
serve every other product.  Both must reproduce scipy's A @ B exactly:
pattern and values.
"""
import ctypes as C
import os
import sys

import numpy as np
import pytest
import scipy.sparse as sp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import cases  # noqa: E402

pytestmark = pytest.mark.gpu


def gpu_spgemm(A, B):
    from paper_2602_23613_b200 import _lib
    from paper_2602_23613_b200.multilevel import _Device
    dev = _Device(0)
    fn = dev.lib.hcamg_debug_spgemm
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]
    hA, hB = _lib.HostCSR(A), _lib.HostCSR(B)
    nnz = np.zeros(1, dtype=np.int64)
    dev.check(fn(dev.h, hA.ref(), hB.ref(), _lib.ptr(nnz), None, None, None, 0))
    n = int(nnz[0])
    indptr = np.zeros(A.shape[0] + 1, dtype=np.int64)
    indices = np.zeros(max(n, 1), dtype=np.int32)
    data = np.zeros(max(n, 1), dtype=np.float64)
    dev.check(fn(dev.h, hA.ref(), hB.ref(), _lib.ptr(nnz), _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(data), n))
    M = sp.csr_matrix((data[:n], indices[:n], indptr), shape=(A.shape[0], B.shape[1]))
    assert M.has_canonical_format or n == 0
    # the library keeps structural entries whose sum is exactly zero (its symmetrise /
    # canonicalise steps drop them, as scipy's csr_matmat does at once)
    M.eliminate_zeros()
    return M


def scipy_product(A, B):
    M = (A @ B).tocsr()   # csr_matmat drops sums that are exactly zero; row entries unsorted
    M.sort_indices()
    M.eliminate_zeros()
    return M


def fully_stored(A, seed):
    n = A.shape[0]
    v = np.random.default_rng(seed).uniform(0.5, 1.5, n)
    D = A.toarray() + 1e-3 * abs(A).max() * np.outer(v, v)
    assert np.count_nonzero(D) == n * n
    return sp.csr_matrix(D)


@pytest.mark.parametrize("name", ["tri3s_alg", "quad3_alg", "kuhn4_c1", "kuhn8_c2"])
@pytest.mark.parametrize("dense_left", [True, False])
def test_spgemm_matches_scipy_bitwise(name, dense_left):
    from oracle import amg_oracle as O
    c = cases.load(name)
    A = fully_stored(c.system.A, 5) if dense_left else c.system.A
    Gt, _ = O.augment(c.system.G)
    ref = scipy_product(A, Gt)
    got = gpu_spgemm(A, Gt)
    assert got.nnz == ref.nnz
    assert np.array_equal(got.indptr, ref.indptr) and np.array_equal(got.indices, ref.indices)
    assert np.array_equal(got.data, ref.data), float(np.max(np.abs(got.data - ref.data)))
    # second product of the nodal dual: G~^T (A G~), a sparse left factor with dense-ish rows
    ref2 = scipy_product(sp.csr_matrix(Gt.T), ref)
    got2 = gpu_spgemm(sp.csr_matrix(Gt.T), got)
    assert np.array_equal(got2.indptr, ref2.indptr) and np.array_equal(got2.indices, ref2.indices)
    assert np.array_equal(got2.data, ref2.data)
