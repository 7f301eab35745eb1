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
out = np.zeros(6 * m + 16, dtype=np.int64)
fn = dev.lib.hcamg_debug_trace_leg
fn.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64]
dev.check(fn(dev.h, 1, out.ctypes.data_as(C.c_void_p), len(out)))
t = out[:6 * m].reshape(m, 6).astype(np.float64)
t0 = t[:, 0].min()
ready, pulled, stored = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3
rvt, mvt = (t[:, 4] - t0) / 1e3, (t[:, 5] - t0) / 1e3
W = waves.max() + 1
print(f"{cfg}: {m} patches, {W} waves, sweep span {stored.max():.1f} us (from the first record ready)")
prev = 0.0
for w in range(W):
    sel = waves == w
    print(f"wave {w:3d} n={sel.sum():5d} ready [{ready[sel].min():7.2f},{ready[sel].max():7.2f}] "
          f"pulled max {pulled[sel].max():7.2f} stored [{stored[sel].min():7.2f},{stored[sel].max():7.2f}] "
          f"compute {np.median(stored[sel] - pulled[sel]):5.2f} link {stored[sel].max() - prev:6.2f}")
    prev = stored[sel].max()

# per-patch link latency: pulled(q) - max over its predecessors p of stored(p)
ps = h.levels[0].patches
A = h.levels[0].A.tocsr()
orig_waves = ps.waves
order = np.lexsort((np.arange(m), orig_waves))          # exec position -> original patch id
pos = np.empty(m, dtype=np.int64)
pos[order] = np.arange(m)
owner = [[] for _ in range(A.shape[0])]
for pid, dofs in enumerate(ps.patches):
    for d in dofs:
        owner[d].append(pid)
lat, nterm = [], []
for q in range(m):
    preds = set()
    for u in ps.patches[q]:
        for j in A.indices[A.indptr[u]:A.indptr[u + 1]]:
            for p in owner[j]:
                if p != q and orig_waves[p] < orig_waves[q]:
                    preds.add(p)
    if preds:
        last = max(stored[pos[p]] for p in preds)
        lat.append(pulled[pos[q]] - last)
        nterm.append(len(preds))
lat = np.array(lat)
print(f"link latency (pulled - last predecessor stored) over {len(lat)} patches: "
      f"p10 {np.percentile(lat, 10):.2f} median {np.median(lat):.2f} p90 {np.percentile(lat, 90):.2f} "
      f"max {lat.max():.2f} us; predecessors per patch median {np.median(nterm):.0f}")

# critical chain: from the last-finishing patch back through its last-finishing predecessor
predl = [None] * m
for q in range(m):
    preds = set()
    for u in ps.patches[q]:
        for j in A.indices[A.indptr[u]:A.indptr[u + 1]]:
            for p in owner[j]:
                if p != q and orig_waves[p] < orig_waves[q]:
                    preds.add(p)
    predl[q] = preds
q = int(order[int(np.argmax(stored))])
chain = []
while q is not None:
    i = pos[q]
    chain.append((q, orig_waves[q], ready[i], rvt[i], pulled[i], mvt[i], stored[i], int(t[i, 3])))
    ps_ = predl[q]
    q = max(ps_, key=lambda p: stored[pos[p]]) if ps_ else None
print("critical chain (patch, wave, ready, r0 loaded, pulled, matvec done, stored, warp):")
for c in chain[::-1]:
    print("  %5d w%3d ready %7.2f r0 %7.2f pulled %7.2f matvec %7.2f stored %7.2f warp %d" % c)
