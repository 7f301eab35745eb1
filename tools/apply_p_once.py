"""Build the config-2 hierarchy and apply the factored interpolation block once
(for ncu captures of the sweep kernel: ncu --profile-from-start off -k regex:k_tri_tma -c 1 ...)."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn, _lib
h = P.build_hierarchy(kuhn.config_system("c2"), "alg")
dev = h._dev
e = np.random.default_rng(0).uniform(-1, 1, h.levels[1].n); out = np.zeros(h.levels[0].n)
import torch
torch.cuda.profiler.start()  # ncu --profile-from-start off: skip the setup's calibration launches
for _ in range(2):
    dev.check(dev.lib.hcamg_debug_apply_p(dev.h, 0, 0, _lib.ptr(e), _lib.ptr(out)))
print("ok")
