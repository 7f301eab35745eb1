"""Level-0 splitting at the BASELINE config sizes: the full
hierarchy is infeasible for the reference there, but its integer splitting is
not.  Fixtures are the reference's own output (tests/golden/make_split_fixtures.py).
CPU: the oracle reproduces them; GPU: libhcamg reproduces them bit for bit."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import amg_oracle as O
from paper_2602_23613_b200 import kuhn

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = [("c2", 32), ("c3", 64)]


def digests(pairs, interior, cg, n):
    text = "\n".join([f"n {n}"] + [f"{p[4]} {p[5]} {p[6]} {p[0]} {p[2]} {p[1]} {p[3]}" for p in pairs]) + "\n"
    return {"dump_sha": hashlib.sha256(text.encode()).hexdigest(),
            "interior_sha": hashlib.sha256(np.asarray(interior, np.int64).tobytes()).hexdigest(),
            "cG_sha": hashlib.sha256(np.asarray(cg, np.int64).tobytes()).hexdigest()}


def check(cfg, n, pairs, interior, cg):
    z = np.load(os.path.join(GOLD, f"split_{cfg}_n{n}.npz"))
    meta = json.loads(str(z["meta"]))
    assert len(pairs) == meta["n_pairs"] and len(interior) == meta["n_interior"] and len(cg) == meta["n_cG"]
    d = digests(pairs, interior, cg, meta["dofs"])
    assert d["dump_sha"] == meta["dump_sha"]
    assert d["interior_sha"] == meta["interior_sha"]
    assert d["cG_sha"] == meta["cG_sha"]
    if "pairs" in z:
        assert np.array_equal(np.asarray(pairs, np.int64).reshape(-1, 7), z["pairs"])


@pytest.mark.parametrize("cfg,n", CASES)
def test_oracle_split_matches_reference(cfg, n):
    s = kuhn.config_system(cfg, n=n)
    sp = O.algebraic_split(s.A, s.G)
    pairs = [(p.dof1, p.dof2, p.sign1, p.sign2, p.tail, p.mid, p.head) for p in sp.pairs]
    check(cfg, n, pairs, sp.interior_dofs, sp.coarse_nodes)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,n", CASES)
def test_gpu_split_matches_reference(cfg, n):
    import paper_2602_23613_b200.multilevel as M
    s = kuhn.config_system(cfg, n=n)
    sp = M.algebraic_splitting(s.A, s.G)
    check(cfg, n, [tuple(p) for p in sp.pairs], sp.interior_dofs, sp.coarse_nodes)
