"""The reference's parity-artefact formats (splitting.py:375-395,
sparse.py:324-338), host side: the splitting text of every golden case's
reference pairs hashes to the reference's own dump, parses back to the same
pairs / interior set, and MatrixMarket round-trips to canonical CSR."""
import hashlib

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2602_23613_b200 import formats
from paper_2602_23613_b200.multilevel import ExteriorPair, Splitting
from tests.cases import CASES, load


@pytest.mark.parametrize("name", CASES)
def test_dump_splitting_matches_reference(name):
    c = load(name)
    for ell, ref in enumerate(c.meta["levels"]):
        if "dump_sha" not in ref:
            continue
        pairs = [ExteriorPair(*(int(v) for v in row)) for row in c.z[f"L{ell}_pairs"]]
        split = Splitting(pairs, c.z[f"L{ell}_interior"], ref["n"])
        text = formats.dump_splitting(split)
        assert hashlib.sha256(text.encode()).hexdigest() == ref["dump_sha"]
        back = formats.parse_splitting(text)
        assert back.n == ref["n"] and back.pairs == pairs
        assert np.array_equal(back.interior_dofs, c.z[f"L{ell}_interior"])


def test_parse_rejects_malformed():
    with pytest.raises(ValueError):
        formats.parse_splitting("1 2 3\n")
    with pytest.raises(ValueError):
        formats.parse_splitting("n 4\n1 2 3\n")


def test_matrix_market_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    M = sp.random(40, 30, density=0.1, random_state=1, format="csr")
    M.data = rng.standard_normal(M.nnz)
    path = tmp_path / "m.mtx"
    formats.write_matrix_market(M, str(path))
    R = formats.read_matrix_market(str(path))
    assert R.shape == M.shape and R.has_canonical_format
    assert abs(R - M).max() == 0.0
    text = formats.mm_to_string(M)
    assert text.startswith("%%MatrixMarket matrix coordinate real general")
