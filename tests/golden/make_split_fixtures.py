"""Level-0 algebraic splittings at the BASELINE config sizes, produced by the
UNMODIFIED reference (splitting.build_algebraic_splitting) on the shared Kuhn
generator.  The full hierarchy is infeasible there but the
integer splitting is oracle-checkable.  n=32 stores arrays,
n=64 stores sha256 digests.  Build container only:
    python tests/golden/make_split_fixtures.py"""
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
import numpy as np

from hcurl_amg.splitting import build_algebraic_splitting, dump_splitting
from paper_2602_23613_b200 import kuhn


def digests(sp):
    return {"dump_sha": hashlib.sha256(dump_splitting(sp).encode()).hexdigest(),
            "interior_sha": hashlib.sha256(np.asarray(sp.interior_dofs, np.int64).tobytes()).hexdigest(),
            "cG_sha": hashlib.sha256(np.asarray(sp.coarse_nodes, np.int64).tobytes()).hexdigest(),
            "n_pairs": sp.n_pairs, "n_interior": int(len(sp.interior_dofs)), "n_cG": int(len(sp.coarse_nodes))}


for cfg, n, full in (("c2", 32, True), ("c3", 64, False)):
    s = kuhn.config_system(cfg, n=n)
    t = time.time()
    sp = build_algebraic_splitting(s.A, s.G)
    meta = dict(digests(sp), config=cfg, n=n, dofs=int(s.n), reference_seconds=time.time() - t)
    out = {"meta": np.array(json.dumps(meta))}
    if full:
        out["pairs"] = np.array([tuple(p) for p in sp.pairs], dtype=np.int64)
        out["interior"] = np.asarray(sp.interior_dofs, np.int64)
        out["cG"] = np.asarray(sp.coarse_nodes, np.int64)
    np.savez_compressed(os.path.join(HERE, f"split_{cfg}_n{n}.npz"), **out)
    print(json.dumps(meta), flush=True)
