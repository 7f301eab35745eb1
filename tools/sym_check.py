import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn
from paper_2602_23613_b200.multilevel import set_options
s = kuhn.config_system(sys.argv[1] if len(sys.argv) > 1 else "c2")
h = P.build_hierarchy(s, "alg")
rng = np.random.default_rng(2)
x, y = rng.uniform(-1, 1, s.n), rng.uniform(-1, 1, s.n)
A = s.A
L0 = h.levels[0]
for sw in ("grid", "wave", "flow"):
    set_options(h, sweep=sw)
    bx, by = P.vcycle(h, x), P.vcycle(h, y)
    sym = abs(bx @ y - x @ by) / (np.linalg.norm(bx) * np.linalg.norm(y))
    f = P.smoothers.smooth(A, L0.patches, None, np.zeros(s.n), x, "forward")
    g = P.smoothers.smooth(A, L0.patches, None, np.zeros(s.n), y, "backward")
    adj = abs(f @ y - x @ g) / (np.linalg.norm(f) * np.linalg.norm(y))
    print(sw, "vcycle asym %.2e" % sym, "smoother fw/bw adjoint asym %.2e" % adj, flush=True)
