"""Time each V-cycle piece alone on the GPU (hcamg_profile_vcycle)."""
import ctypes as C
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import _lib, kuhn

NAMES = {0: "down leg", 1: "restrict", 2: "coarse", 3: "prolong", 4: "up leg"}
cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else None
h = P.build_hierarchy(kuhn.config_system(cfg, n=n), "alg")
dev = h._dev
cap = 64
kind = np.zeros(cap, np.int32); level = np.zeros(cap, np.int32); us = np.zeros(cap); nl = np.zeros(cap, np.int64)
cnt = C.c_int32()
import os

# optional: "ENV=v1,v2,..." as argv[3] re-times the pieces once per value of ENV;
# "opt:KEY=v1,v2" sets the handle option KEY instead (e.g. opt:sweep=2,4)
sweeps = [(None, None)]
if len(sys.argv) > 3:
    var, vals = sys.argv[3].split("=")
    sweeps = [(var, v) for v in vals.split(",")]
for var, val in sweeps:
    if var and var.startswith("opt:"):
        dev.set_option(var[4:], float(val))
        print(f"-- option {var[4:]}={val}")
    elif var:
        os.environ[var] = val
        print(f"-- {var}={val}")
    dev.check(dev.lib.hcamg_profile_vcycle(dev.h, 10 if h.levels[0].n > 100000 else 50, cap, _lib.ptr(kind),
                                           _lib.ptr(level), _lib.ptr(us), _lib.ptr(nl), C.byref(cnt)))
    tot = 0
    for i in range(cnt.value):
        print(f"L{level[i]} {NAMES[kind[i]]:10s} {us[i]:9.2f} us  launches {nl[i]}")
        tot += us[i]
    print(f"V-cycle sum {tot:.1f} us; levels {[lv.n for lv in h.levels]}; waves {[lv._info.n_waves for lv in h.levels]}")
