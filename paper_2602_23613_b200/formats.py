"""The reference's on-disk formats for parity artefacts.

* ``dump_splitting`` / ``parse_splitting`` -- the text form of a splitting, one
  line per exterior pair (reference splitting.py:375-395);
* ``write_matrix_market`` / ``read_matrix_market`` / ``mm_to_string`` --
  MatrixMarket coordinate files, 1-based, real general (reference
  sparse.py:324-338).

Host-side text IO only; these never touch the device.
"""
from __future__ import annotations

import io

import numpy as np
import scipy.io
import scipy.sparse as sp

from .multilevel import ExteriorPair, Splitting
from .sparse import csr

__all__ = ["dump_splitting", "parse_splitting", "write_matrix_market", "read_matrix_market", "mm_to_string"]


def dump_splitting(split) -> str:
    """``n <n>`` header, then ``tail mid head dof1 sign1 dof2 sign2`` per pair."""
    lines = [f"n {int(split.n)}"]
    for p in split.pairs:
        p = ExteriorPair(*(int(v) for v in p))
        lines.append(f"{p.tail} {p.mid} {p.head} {p.dof1} {p.sign1} {p.dof2} {p.sign2}")
    return "\n".join(lines) + "\n"


def parse_splitting(text: str) -> Splitting:
    """Inverse of ``dump_splitting``; interior = every DoF not in a pair."""
    rows = [ln for ln in text.splitlines() if ln.strip()]
    if not rows or not rows[0].startswith("n "):
        raise ValueError("missing size header")
    n = int(rows[0].split()[1])
    pairs, taken = [], set()
    for ln in rows[1:]:
        fields = ln.split()
        if len(fields) != 7:
            raise ValueError(f"malformed pair line: {ln!r}")
        t, k, h, d1, s1, d2, s2 = (int(x) for x in fields)
        pairs.append(ExteriorPair(d1, d2, s1, s2, t, k, h))
        taken.update((d1, d2))
    interior = np.array(sorted(set(range(n)) - taken), dtype=np.int64)
    return Splitting(pairs, interior, n)


def write_matrix_market(A, path):
    scipy.io.mmwrite(path, sp.coo_matrix(A), field="real", symmetry="general")


def read_matrix_market(path):
    """A MatrixMarket file as canonical CSR (sorted, duplicates summed, no stored zeros)."""
    return csr(scipy.io.mmread(path))


def mm_to_string(A) -> str:
    buf = io.BytesIO()
    scipy.io.mmwrite(buf, sp.coo_matrix(A), field="real", symmetry="general")
    return buf.getvalue().decode()
