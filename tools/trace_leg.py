"""Per-phase timeline of the level-0 cluster smoothing leg (debug trace)."""
import ctypes as C
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import _lib, kuhn

import os

# usage: trace_leg.py CONFIG [N] [down|up] ; HCAMG_SWEEP=grid traces the cooperative-grid leg
cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
down = 1 if (len(sys.argv) <= 3 or sys.argv[3] == "down") else 0
h = P.build_hierarchy(kuhn.config_system(cfg, n), "alg")
dev = h._dev
W = int(h.levels[0]._info.n_waves)
grid = os.environ.get("HCAMG_SWEEP") == "grid"
nw = (int(os.environ.get("HCAMG_GRID_BLOCKS", 148)) if grid else 16) * 512 // 32
cap = W * nw * 2
buf = np.zeros(cap, dtype=np.int64)
fn = dev.lib.hcamg_debug_trace_leg
fn.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
dev.check(fn(dev.h, down, buf.ctypes.data, cap))
t = buf.reshape(W, nw, 2).astype(np.float64)
t0 = t[0, :, 0].min()
print("phase  start(us)  work_max(us)  patchwarps_max  rowwarps_max  phase_len(us)")
for s in range(W):
    st = t[s, :, 0].min()
    work = t[s, :, 1] - t[s, :, 0]
    nxt = t[s + 1, :, 0].min() if s + 1 < W else t[s, :, 1].max()
    print(f"{s:5d} {(st - t0) / 1e3:9.2f} {work.max() / 1e3:12.2f} {work[: nw // 4].max() / 1e3:14.2f} {work[3 * nw // 4 :].max() / 1e3:13.2f} {(nxt - st) / 1e3:12.2f}")
if os.environ.get("TRACE_DUMP"):
    np.save(os.environ["TRACE_DUMP"], t)
