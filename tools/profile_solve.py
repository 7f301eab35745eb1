"""Run one device-resident PCG solve between cudaProfilerStart/Stop (for
`ncu --profile-from-start off`), after setup and warm-up outside the range."""
import argparse
import ctypes as C
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch

import paper_2602_23613_b200 as P
from paper_2602_23613_b200 import _lib, kuhn

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--solves", type=int, default=1)
args = ap.parse_args()
system = kuhn.config_system(args.config, n=args.n)
h = P.build_hierarchy(system, "alg")
dev = h._dev
b = torch.from_numpy(kuhn.rhs(system.n, seed=0)).cuda()
x = torch.zeros_like(b)
rep = _lib.Report()
for _ in range(3):
    dev.check(dev.lib.hcamg_pcg_device(dev.h, C.c_void_p(b.data_ptr()), None, 1e-8, 500, C.c_void_p(x.data_ptr()),
                                       C.byref(rep)))
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(args.solves):
    dev.check(dev.lib.hcamg_pcg_device(dev.h, C.c_void_p(b.data_ptr()), None, 1e-8, 500, C.c_void_p(x.data_ptr()),
                                       C.byref(rep)))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("iterations", rep.iterations, "launches pre/body", dev.lib.hcamg_graph_launches(dev.h, 1),
      dev.lib.hcamg_graph_launches(dev.h, 2))
