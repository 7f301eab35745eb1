import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn, _lib
h = P.build_hierarchy(kuhn.config_system("c2"), "alg")
dev = h._dev
e = np.random.default_rng(0).uniform(-1, 1, h.levels[1].n); out = np.zeros(h.levels[0].n)
for _ in range(3):
    dev.check(dev.lib.hcamg_debug_apply_p(dev.h, 0, 0, _lib.ptr(e), _lib.ptr(out)))
os.environ["HCAMG_TRI_DBG"] = "4"
os.environ["HCAMG_TRI_DUMP"] = "gpurun_out/tl"
for _ in range(int(os.environ.get("TL_REPS", "1"))):
    dev.check(dev.lib.hcamg_debug_apply_p(dev.h, 0, 0, _lib.ptr(e), _lib.ptr(out)))
