import os, sys, ctypes as C
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn, _lib
h = P.build_hierarchy(kuhn.config_system("c2"), "alg")
dev = h._dev
e = np.zeros(h.levels[1].n); out = np.zeros(h.levels[0].n)
os.environ["HCAMG_TRI_DBG"] = "3"
for _ in range(5):
    dev.check(dev.lib.hcamg_debug_apply_p(dev.h, 0, 0, _lib.ptr(e), _lib.ptr(out)))
os.environ["HCAMG_TRI_DBG"] = "0"
dev.check(dev.lib.hcamg_debug_apply_p(dev.h, 0, 0, _lib.ptr(e), _lib.ptr(out)))
print("10 sweeps traced")
