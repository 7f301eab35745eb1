"""Run the level-0 dataflow smoothing leg of CONFIG a few times (ncu target)."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
h = P.build_hierarchy(kuhn.config_system(cfg), "alg")
P.multilevel.set_options(h, sweep="flow")
b = np.random.default_rng(0).standard_normal(h.levels[0].n)
for _ in range(3):
    P.vcycle(h, b)
print("ok")
