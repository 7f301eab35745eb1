"""A_1 of the dense-regime hierarchy with the residual term Z^T rho in TF32
(default) vs FP64 (HCAMG_GALERKIN_E=fp64): relative differences."""
import os
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s = kuhn.config_system(cfg, n=n)
b = kuhn.rhs(s.n, seed=0)
out = {}
for mode in ("tf32", "fp64"):
    if mode == "fp64":
        os.environ["HCAMG_GALERKIN_E"] = "fp64"
    else:
        os.environ.pop("HCAMG_GALERKIN_E", None)
    h = P.build_hierarchy(s, "alg")
    A1 = h.levels[1].A.toarray()
    x, rep = P.pcg(s.A, b, precond=lambda v: P.vcycle(h, v), tol=1e-8)
    out[mode] = (A1, x, rep.iterations, rep.residual_history)
    del h
a, b_ = out["tf32"][0], out["fp64"][0]
print(f"{cfg} n={n}: A1 max|diff|/max|A1| = {np.abs(a - b_).max() / np.abs(b_).max():.3e}; "
      f"fro rel = {np.linalg.norm(a - b_) / np.linalg.norm(b_):.3e}; "
      f"x rel = {np.linalg.norm(out['tf32'][1] - out['fp64'][1]) / np.linalg.norm(out['fp64'][1]):.3e}; "
      f"iters {out['tf32'][2]} / {out['fp64'][2]}")
