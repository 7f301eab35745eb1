"""GPU setup + PCG on a larger Kuhn cube (dense-interpolation regime); compares
with tests/golden/kuhn16_c1.npz when present."""
import json
import os
import sys
import time

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)
import numpy as np

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
t0 = time.time()
s = kuhn.config_system(cfg, n=n)
print(f"assembled n={s.n} nnz={s.A.nnz} in {time.time() - t0:.1f}s", flush=True)
t0 = time.time()
h = P.build_hierarchy(s, "alg")
print(f"setup {time.time() - t0:.2f}s (device {h.setup_seconds:.2f}s) levels {[lv.n for lv in h.levels]} "
      f"stalled {h.stalled} notes {h.notes} OC {P.operator_complexity(h):.3f}", flush=True)
b = kuhn.rhs(s.n, seed=0)
for rep in range(3):
    t0 = time.time()
    x, r = P.pcg(s.A, b, precond=lambda v: P.vcycle(h, v), tol=1e-8)
    print(f"pcg iters {r.iterations} conv {r.converged} time {time.time() - t0:.4f}s", flush=True)
print("hist", " ".join(f"{v:.3e}" for v in r.residual_history))
print("true relres", np.linalg.norm(s.A @ x - b) / np.linalg.norm(b))
fx = os.path.join(ROOT, "tests", "golden", f"kuhn{n}_{cfg}.npz")
if os.path.exists(fx):
    z = np.load(fx)
    meta = json.loads(str(z["meta"]))
    L0 = h.levels[0]
    sp = L0.splitting
    pairs = np.array([tuple(p) for p in sp.pairs], dtype=np.int64)
    print("pairs equal", np.array_equal(pairs, z["pairs"]), "interior equal", np.array_equal(sp.interior_dofs, z["interior"]),
          "cG equal", np.array_equal(sp.coarse_nodes, z["cG"]))
    print("levels", [lv.n for lv in h.levels], "oracle", meta["levels"], "iters", r.iterations, "oracle", meta["pcg_iters"])
    Pm = L0.P
    import hashlib
    sha = hashlib.sha256(Pm.indptr.astype(np.int64).tobytes() + Pm.indices.astype(np.int64).tobytes()).hexdigest()
    print("P nnz", Pm.nnz, meta["P_nnz"], "pattern equal", sha == meta["P_pattern_sha"],
          "P fro rel", abs(np.sqrt((Pm.data ** 2).sum()) - meta["P_fro"]) / meta["P_fro"])
    cs = np.asarray(Pm.sum(axis=0)).ravel()
    print("P colsum rel", np.abs(cs - z["P_colsum"]).max() / np.abs(z["P_colsum"]).max())
    A1 = h.levels[1].A
    print("A1 nnz", A1.nnz, meta["A1_nnz"], "A1 fro rel", abs(np.sqrt((A1.data ** 2).sum()) - meta["A1_fro"]) / meta["A1_fro"],
          "A1 diag rel", np.abs(A1.diagonal() - z["A1_diag"]).max() / np.abs(z["A1_diag"]).max())
    print("x rel", np.linalg.norm(x - z["pcg_x"]) / np.linalg.norm(z["pcg_x"]))
