"""Per-step, per-CTA timeline of the TMA sweep (HCAMG_TRI_DBG=4 dumps):
where the step time goes and whether the slow CTAs are slow because of their
bytes, their task count, or something static (their SM)."""
import glob
import sys

import numpy as np

files = sorted(glob.glob((sys.argv[1] if len(sys.argv) > 1 else "tri_timeline") + ".*.bin"))
for fn in files[-2:]:
    raw = np.fromfile(fn, np.int64)
    nst, G = raw[:2]
    r = raw[2:].reshape(nst, G, 4).astype(np.float64)
    done, pas, tasks, by = r[..., 0], r[..., 1], r[..., 2], r[..., 3]
    # step work of CTA c in step st: from passing barrier st-1 to done st
    start = np.concatenate([done[:1].min(1, keepdims=True).repeat(G, 1) * 0 + done[:1].min(), pas[:-1]], 0)
    work = (done - start)[1:]
    wby, wt = by[1:], tasks[1:]
    spread = done.max(1) - done.min(1)
    rel = pas.min(1) - done.max(1)  # barrier release after last arrival
    total = pas[-2, :].max() - pas[0, :].min() if nst > 2 else 0
    print(f"{fn}: steps {nst} G {G} span {total/1e3:.1f} us ({total/1e3/(nst-2):.2f} us/step)")
    print(f"  work per step (us): mean {work.mean()/1e3:.2f}  max-over-CTAs mean {work.max(1).mean()/1e3:.2f}  min {work.min(1).mean()/1e3:.2f}")
    print(f"  arrival spread mean {spread[1:].mean()/1e3:.2f} us; release after last arrival mean {rel[1:-1].mean()/1e3:.2f} us")
    print(f"  stage+desc (pass -> start of tasks) not separated; bytes/CTA/step mean {wby.mean()/1e3:.1f} KB, max {wby.max(1).mean()/1e3:.1f} KB")
    # correlation of per-(step,CTA) work with bytes and tasks
    x = np.stack([wby.ravel(), wt.ravel(), np.ones(wby.size)], 1)
    coef, *_ = np.linalg.lstsq(x, work.ravel(), rcond=None)
    pred = x @ coef
    res = work.ravel() - pred
    print(f"  fit work = {coef[0]*1e3/1e3:.3f} ns/B*1e3 ... ns per KB {coef[0]*1e3:.1f}, ns per task {coef[1]:.1f}, const {coef[2]:.0f} ns; R^2 {1 - res.var()/work.var():.3f}")
    cta_bias = (work - pred.reshape(work.shape)).mean(0)
    print(f"  static per-CTA bias (us): std {cta_bias.std()/1e3:.3f}, min {cta_bias.min()/1e3:.2f} (cta {cta_bias.argmin()}), max {cta_bias.max()/1e3:.2f} (cta {cta_bias.argmax()})")
    slow = work.argmax(1)
    print(f"  slowest CTA per step: distinct {len(set(slow.tolist()))} of {nst-1}; most frequent {np.bincount(slow).max()}")
    print(f"  slowest CTA's bytes vs mean: {np.mean(wby[np.arange(nst-1), slow] / wby.mean(1)):.3f}; tasks vs mean {np.mean(wt[np.arange(nst-1), slow] / wt.mean(1)):.3f}")
