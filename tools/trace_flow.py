"""Per-patch timeline of the dataflow smoothing leg (flow.cu trace):
usage: python tools/trace_flow.py CONFIG [N]  -> per-wave link costs."""
import ctypes as C
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else None
h = P.build_hierarchy(kuhn.config_system(cfg, n=n), "alg")
P.multilevel.set_options(h, sweep="flow")
dev = h._dev
waves = np.sort(h.levels[0].patches.waves)        # wave of each execution position (down leg)
m = len(waves)
out = np.zeros(4 * m + 16, dtype=np.int64)
fn = dev.lib.hcamg_debug_trace_leg
fn.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
dev.check(fn(dev.h, 1, out.ctypes.data_as(C.c_void_p), len(out)))
t = out[:4 * m].reshape(m, 4).astype(np.float64)
t0 = t[:, 0].min()
ready, pulled, stored = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
W = waves.max() + 1
print(f"{cfg}: {m} patches, {W} waves, sweep span {stored.max():.1f} us (from the first record ready)")
prev = 0.0
for w in range(W):
    sel = waves == w
    print(f"wave {w:3d} n={sel.sum():5d} ready [{ready[sel].min():7.2f},{ready[sel].max():7.2f}] "
          f"pulled max {pulled[sel].max():7.2f} stored [{stored[sel].min():7.2f},{stored[sel].max():7.2f}] "
          f"compute {np.median(stored[sel] - pulled[sel]):5.2f} link {stored[sel].max() - prev:6.2f}")
    prev = stored[sel].max()
