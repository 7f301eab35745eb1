"""Setup stage times (HCAMG_SETUP_TIMING=1) for one configuration; three builds."""
import os, sys, time
if not os.environ.get("HCAMG_NO_STAGES"):
    os.environ["HCAMG_SETUP_TIMING"] = "1"  # HCAMG_NO_STAGES=1: wall time per build only (stage marks synchronise)
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import kuhn
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg.startswith("2d-L"):
    from paper_2602_23613_b200 import tri2d
    s = tri2d.stripes_system(int(cfg[4:]))
else:
    s = kuhn.config_system(cfg)
h = None
for rep in range(int(os.environ.get("HCAMG_BUILDS", "3"))):
    h = None
    t = time.perf_counter(); h = P.build_hierarchy(s, "alg"); print(f"== build {rep}: {time.perf_counter() - t:.3f} s", file=sys.stderr)
