"""Host (kuhn.py) vs GPU (csrc/kuhn.cu) assembly time of a config system."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
from paper_2602_23613_b200 import kuhn
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
kuhn.config_system_gpu(cfg, n=4)  # context warm-up
t = time.perf_counter(); d = kuhn.config_system_gpu(cfg, n=n); tg = time.perf_counter() - t
t = time.perf_counter(); h = kuhn.config_system(cfg, n=n); th = time.perf_counter() - t
same = np.array_equal(d.A.indices, h.A.indices) and np.abs(d.A.data - h.A.data).max() <= 1e-14 * np.abs(h.A.data).max()
print(f"{cfg} n={n or kuhn.CONFIGS[cfg]['n']}: {d.n} DoFs, nnz(A) {d.A.nnz}; host {th:.3f} s, GPU {tg:.3f} s "
      f"(incl. host coefficient field and export); A equal to 1e-14: {same}")
