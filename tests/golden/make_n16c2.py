"""Oracle fixture for the 3D Kuhn n=16 system with BASELINE configs[1]'s
coefficients (mu^{-1} = 4x4x4 checkerboard of 1 / 1e6 subcubes, beta = 1e-3):
the dense-interpolation regime on the field the c2 bench runs (VERDICT r1
"parity gap: the giant/factor path is not oracle-checked on the benchmarked
coefficient field").  ~20 min on CPU (dense 20k Cholesky + Galerkin over the
dense P block, twice: the second run swaps the component Cholesky for a
reversed-order LU to MEASURE the fp64 reproducibility floor).
A_1 (2,948^2, 70 MB) is too large to commit: its diagonal, row sums and 64
seeded full rows are stored.  Generated with the ORACLE (pinned bit-exactly to
the reference on the golden cases); run in the build container:
    python tests/golden/make_n16c2.py"""
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
import numpy as np

from oracle import amg_oracle as O
from paper_2602_23613_b200 import kuhn

s = kuhn.config_system("c2", n=16)
b = kuhn.rhs(s.n, seed=0)


def run(floor):
    t0 = time.time()
    h = O.hierarchy(s, "alg", floor_solver=floor)
    ts = time.time() - t0
    t0 = time.time()
    x, rep = O.pcg(s.A, b, precond=lambda r: O.vcycle(h, r), tol=1e-8)
    return h, x, rep, ts, time.time() - t0


h, x, rep, t_setup, t_solve = run(False)
hf, xf, repf, _, _ = run(True)
L0, L1 = h.levels[0], h.levels[1]
sp = L0.splitting
pairs = np.array([[p.dof1, p.dof2, p.sign1, p.sign2, p.tail, p.mid, p.head] for p in sp.pairs], dtype=np.int64)
rows = np.sort(np.random.default_rng(0).choice(L1.n, size=64, replace=False))
A1 = L1.A.toarray()
A1f = hf.levels[1].A.toarray()
vb = np.random.default_rng(1).standard_normal(s.n)
v = O.vcycle(h, vb)
vf = O.vcycle(hf, vb)
meta = {"n": int(s.n), "levels": [lv.n for lv in h.levels], "stalled": h.stalled, "notes": h.notes,
        "oc": O.operator_complexity(h), "pcg_iters": rep.iterations, "pcg_iters_floor": repf.iterations,
        "setup_s": t_setup, "solve_s": t_solve, "P_nnz": int(L0.P.nnz), "A1_nnz": int(L1.A.nnz),
        "P_pattern_sha": hashlib.sha256(L0.P.indptr.astype(np.int64).tobytes()
                                        + L0.P.indices.astype(np.int64).tobytes()).hexdigest(),
        "P_fro": float(np.sqrt((L0.P.data ** 2).sum())), "A1_fro": float(np.sqrt((L1.A.data ** 2).sum())),
        # measured floors: oracle vs the same oracle with a reversed-order LU component solve
        "floor_P": float(np.abs(hf.levels[0].P.data - L0.P.data).max() / np.abs(L0.P.data).max()),
        "floor_A1": float(np.abs(A1f - A1).max() / np.abs(A1).max()),
        "floor_x": float(np.linalg.norm(xf - x) / np.linalg.norm(x)),
        "floor_vcycle": float(np.abs(vf - v).max() / np.abs(v).max()),
        "true_relres": float(np.linalg.norm(s.A @ x - b) / np.linalg.norm(b))}
np.savez_compressed(os.path.join(HERE, "kuhn16_c2.npz"), pairs=pairs, interior=sp.interior_dofs,
                    cG=sp.coarse_nodes, A1_diag=L1.A.diagonal(), A1_rowsum=A1.sum(axis=1), A1_rows=rows,
                    A1_sample=A1[rows], P_colsum=np.asarray(L0.P.sum(axis=0)).ravel(), pcg_hist=rep.residual_history,
                    pcg_x=x, b=b, vcycle_b=vb, vcycle_x=v, meta=np.array(json.dumps(meta)))
print(json.dumps(meta))
