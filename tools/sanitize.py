"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every solve-phase kernel family on tiny golden cases -- cluster leg, grid
leg, dataflow leg, per-wave launches, the TMA factor sweeps (dense regime
forced), the explicit-Z kernels, the packed-triangle coarsest solve -- plus
one full setup each.  usage: compute-sanitizer --tool T python tools/sanitize.py"""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np

import paper_2602_23613_b200 as P
from paper_2602_23613_b200.multilevel import set_options
from tests.cases import load

runs = [("tri3s_alg", {}, ["leg", "grid", "wave", "flow"]),
        ("kuhn4_c1", {"giant_min": 100, "coarse_gemv_min": 0, "coarse_symv": 1}, ["leg", "grid", "flow"]),
        ("kuhn4_c1", {"giant_min": 100, "coarse_gemv_min": 0, "coarse_symv": 0, "factor_apply": 0}, ["leg"])]
for name, opts, sweeps in runs:
    c = load(name)
    h = P.build_hierarchy(c.system, c.meta["method"], meshes=c.meshes, rmaps=c.rmaps, options=opts)
    b = c.z["pcg_b"]
    for sw in sweeps:
        set_options(h, sweep=sw)
        x, rep = P.pcg(c.system.A, b, precond=lambda r: P.vcycle(h, r), tol=1e-8, maxit=3)
        print(name, opts, sw, "pcg iters", rep.iterations, flush=True)
print("sanitize workload done")
