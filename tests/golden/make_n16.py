"""Oracle summary for the 3D Kuhn n=16 system (config-1 coefficients): the
dense-interpolation regime (one 20,520-DoF interior component, dense level 1).
The full reference takes ~11 min here, so the fixture stores the integer
splitting of level 0, norms/diagonals of P and A_1, and the PCG result.
Generated with the ORACLE (pinned bit-exactly to the reference on the smaller
golden cases); run in the build container:  python tests/golden/make_n16.py"""
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

t0 = time.time()
s = kuhn.config_system("c1", n=16)
h = O.hierarchy(s, "alg")
t_setup = time.time() - t0
b = kuhn.rhs(s.n, seed=0)
t0 = time.time()
x, rep = O.pcg(s.A, b, precond=lambda r: O.vcycle(h, r), tol=1e-8)
t_solve = time.time() - t0
L0, L1 = h.levels[0], h.levels[1]
sp = L0.splitting
pairs = np.array([[p.dof1, p.dof2, p.sign1, p.sign2, p.tail, p.mid, p.head] for p in sp.pairs], dtype=np.int64)
meta = {"n": int(s.n), "levels": [lv.n for lv in h.levels], "stalled": h.stalled, "notes": h.notes,
        "oc": O.operator_complexity(h), "pcg_iters": rep.iterations, "setup_s": t_setup, "solve_s": t_solve,
        "P_nnz": int(L0.P.nnz), "A1_nnz": int(L1.A.nnz),
        "P_pattern_sha": hashlib.sha256(L0.P.indptr.astype(np.int64).tobytes() + L0.P.indices.astype(np.int64).tobytes()).hexdigest(),
        "P_fro": float(np.sqrt((L0.P.data ** 2).sum())), "A1_fro": float(np.sqrt((L1.A.data ** 2).sum()))}
np.savez_compressed(os.path.join(HERE, "kuhn16_c1.npz"), pairs=pairs, interior=sp.interior_dofs,
                    cG=sp.coarse_nodes, A1_diag=L1.A.diagonal(), P_colsum=np.asarray(L0.P.sum(axis=0)).ravel(),
                    pcg_hist=rep.residual_history, pcg_x=x, b=b, meta=np.array(json.dumps(meta)))
print(json.dumps(meta))
