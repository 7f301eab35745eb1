"""Oracle fixtures for the 2D stripes family (the reference's own sparse
regime): tri_chain(L, stripes=True), beta = 0.01,
"alg" hierarchy, PCG from x0 = 0 on rhs default_rng(0).uniform(-1, 1).
Integers are stored as SHA-256 digests (pairs, interior sets, every level's
A / P / G patterns); floating point as seeded random projections (64 rows
drawn from default_rng(99)) of x, of every P and of every A_l, so the test
checks them to max(1e-10, 10 x the measured floor) without a multi-MB
fixture; the floors (oracle vs the oracle with a reversed-order LU component
solve) are stored with them.  The system generator
(paper_2602_23613_b200/tri2d.py) is bit-identical to the reference's
(tests/test_tri2d.py); the hierarchy and solve come from the ORACLE, pinned to
the reference on the golden cases.  Run in the build container:
    python tests/golden/make_2d.py 7 9"""
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
import numpy as np

from oracle import amg_oracle as O
from paper_2602_23613_b200 import tri2d


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def proj(v, k=64, seed=99):
    R = np.random.default_rng(seed).standard_normal((k, len(v)))
    return R @ v


def main(L):
    meshes, rmaps, s = tri2d.tri_chain(L, stripes=True)
    b = np.random.default_rng(0).uniform(-1.0, 1.0, s.n)
    t0 = time.time()
    h = O.hierarchy(s, "alg")
    ts = time.time() - t0
    t0 = time.time()
    x, rep = O.pcg(s.A, b, precond=lambda r: O.vcycle(h, r), tol=1e-8)
    tsol = time.time() - t0
    # measured fp64 reproducibility floor: the same oracle with its component
    # Cholesky swapped for a reversed-order LU
    hf = O.hierarchy(s, "alg", floor_solver=True)
    xf, _ = O.pcg(s.A, b, precond=lambda r: O.vcycle(hf, r), tol=1e-8)

    def rel(a, c):
        return float(np.abs(a - c).max() / np.abs(c).max())
    floors = {"P": max(rel(f.P.data, o.P.data) for f, o in zip(hf.levels[:-1], h.levels[:-1])),
              "A": max(rel(f.A.data, o.A.data) for f, o in zip(hf.levels, h.levels)),
              "x": float(np.linalg.norm(xf - x) / np.linalg.norm(x))}
    levels = []
    for lv in h.levels:
        d = {"n": lv.n, "A_pattern": sha(lv.A.indptr.astype(np.int64), lv.A.indices.astype(np.int64)),
             "A_proj": proj(lv.A.data).tolist(), "A_nnz": int(lv.A.nnz),
             "G_pattern": sha(lv.G.indptr.astype(np.int64), lv.G.indices.astype(np.int64), lv.G.data)}
        if lv.P is not None:
            sp_ = lv.splitting
            pairs = np.array([[p.dof1, p.dof2, p.sign1, p.sign2, p.tail, p.mid, p.head] for p in sp_.pairs],
                             dtype=np.int64)
            d.update({"pairs": sha(pairs), "interior": sha(sp_.interior_dofs.astype(np.int64)),
                      "coarse_nodes": sha(np.asarray(sp_.coarse_nodes, dtype=np.int64)),
                      "P_pattern": sha(lv.P.indptr.astype(np.int64), lv.P.indices.astype(np.int64)),
                      "P_proj": proj(lv.P.data).tolist(), "P_nnz": int(lv.P.nnz), "n_patches": len(lv.patches.patches)})
        levels.append(d)
    meta = {"L": L, "n": int(s.n), "levels": levels, "stalled": h.stalled, "notes": h.notes,
            "oc": O.operator_complexity(h), "pcg_iters": rep.iterations, "pcg_hist": rep.residual_history.tolist(),
            "x_proj": proj(x).tolist(), "x_norm": float(np.linalg.norm(x)), "setup_s": ts, "solve_s": tsol,
            "floors": floors}
    with open(os.path.join(HERE, f"tri{L}s_large.json"), "w") as f:
        json.dump(meta, f)
    print(L, s.n, [lv.n for lv in h.levels], rep.iterations, f"setup {ts:.1f}s solve {tsol:.1f}s")


if __name__ == "__main__":
    for L in sys.argv[1:] or ["7", "9"]:
        main(int(L))
