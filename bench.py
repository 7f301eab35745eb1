"""AMG-PCG solve throughput on the seeded 3D Kuhn-cube configurations.

One "step" = one full PCG solve (x0 = 0, V(1,1) OSS-l1 preconditioner, relative
residual 1e-8) over the resident hierarchy: metric DoF*iters/s = n * iterations
/ t_solve (BASELINE.json), plus achieved HBM GB/s from the fixed algorithmic
byte model of SURVEY.md §8(d) and the device-synchronised setup time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1]

* value: device-resident solve (b, x in HBM; hcamg_pcg_device), timed with
  CUDA events on the library's stream, L2 flushed (256 MiB write) before
  every timed step, outside the timed interval;
* e2e: the same solve through the C-ABI host-buffer call hcamg_pcg (b from
  pinned host memory, x and the report read back each step);
* --impl reference: the CPU oracle (oracle/amg_oracle.py, a faithful numpy /
  scipy restatement of the reference; the reference itself is a pure-Python
  package that cannot travel to the GPU box) on the same config.
Multi-GPU (torchrun): independent replicas, one problem per rank (weak
scaling); max over ranks of the device time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return PEAKS_FALLBACK, "fallback"


def algorithmic_bytes(h):
    """B_iter of SURVEY.md §8(d): bytes one PCG iteration must move, whatever
    the implementation.  B(M) = 12 nnz + 4 (rows + 1); B(P) = min(CSR, hybrid
    dense-block); S_l = sum_p [8 k_p (k_p+1)/2 + 12 nnz(A[:, patch_p])]; 3 A
    applications per smoothed level; 2 * 8 * n_c (n_c+1)/2 for the coarsest."""
    def B(nnz, rows):
        return 12 * nnz + 4 * (rows + 1)

    L0 = h.levels[0]
    total = B(int(L0._info.nnz_A), L0.n) + 64 * L0.n
    for ell, lv in enumerate(h.levels):
        info = lv._info
        n = int(info.n)
        if info.coarsest:
            total += 2 * 8 * n * (n + 1) // 2
            continue
        A = lv.A
        colnnz = np.diff(A.tocsc().indptr)
        S = 0
        for p in lv.patches.patches:
            k = len(p)
            S += 8 * k * (k + 1) // 2 + 12 * int(colnnz[p].sum())
        nc = int(h.levels[ell + 1]._info.n)
        n_int = int(info.n_interior)
        csr_p = B(int(info.nnz_P), n)
        hybrid = 8 * n_int * nc + B(2 * int(info.n_pairs), n)
        total += 3 * B(int(info.nnz_A), n) + 2 * min(csr_p, hybrid) + 2 * S + 96 * n
    return int(total)


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        self.result = {"sm_mhz": None, "sm_max_mhz": None, "reasons": []}
        if self.proc is None:
            return False
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if sm:
            self.result = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                           "samples": len(sm)}
        return False


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist_
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist_.init_process_group("gloo")
        dist = dist_
    return world, rank, local, dist


def reduce_max(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(dist, v):
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return 1


def oracle_solve_rate(system, b, min_seconds, max_solves=None):
    """Time the CPU oracle's PCG solves (setup excluded) -> (DoF*iters/s, solves, seconds, iters, setup_s)."""
    from oracle import amg_oracle as O
    t0 = time.perf_counter()
    ho = O.hierarchy(system, "alg")
    setup_s = time.perf_counter() - t0
    n = system.n
    done, work, t = 0, 0, 0.0
    iters = 0
    while True:
        t0 = time.perf_counter()
        x, rep = O.pcg(system.A, b, precond=lambda r: O.vcycle(ho, r), tol=1e-8)
        t += time.perf_counter() - t0
        done += 1
        iters = rep.iterations
        work += n * rep.iterations
        if t >= min_seconds or (max_solves and done >= max_solves):
            break
    return work / t, done, t, iters, setup_s


def run_reference(args, world, rank, dist):
    from paper_2602_23613_b200 import kuhn
    if rank != 0:
        return
    system = kuhn.config_system(args.config)
    b = kuhn.rhs(system.n, seed=0)
    from oracle import amg_oracle as O
    t0 = time.perf_counter()
    ho = O.hierarchy(system, "alg")
    setup_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        O.pcg(system.A, b, precond=lambda r: O.vcycle(ho, r), tol=1e-8)
    t = 0.0
    work = 0
    iters = 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        x, rep = O.pcg(system.A, b, precond=lambda r: O.vcycle(ho, r), tol=1e-8)
        t += time.perf_counter() - t0
        iters = rep.iterations
        work += system.n * rep.iterations
    value = work / t
    cores = cpu_threads()
    line = {
        "impl": "reference", "metric": "AMG-PCG solve DoF*iters/s", "value": value, "unit": "DoF*iters/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"kuhn {args.config} (n={system.n} DoFs, alg, PCG tol 1e-8, x0=0, rhs seed 0)",
                   "pcg_iterations": iters, "setup_s": setup_s},
        "cpu_baseline": {"value": value, "unit": "DoF*iters/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} full PCG solves of {args.config} after {args.warmup} warm-up, "
                                   "oracle/amg_oracle.py (numpy/scipy restatement of the reference)"},
        "e2e": {"value": value, "unit": "DoF*iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local, dist):
    import ctypes as C

    import torch

    import paper_2602_23613_b200 as P
    from paper_2602_23613_b200 import _lib, kuhn

    torch.cuda.set_device(local)
    system = kuhn.config_system(args.config)
    n = system.n
    b_host = kuhn.rhs(n, seed=0)
    # setup (the first call also pays context / module load; report the best of two)
    setups = []
    for _ in range(2):
        h = P.build_hierarchy(system, "alg", device=local)
        setups.append(h.setup_seconds)
    dev = h._dev
    lib = dev.lib
    stream = torch.cuda.ExternalStream(int(lib.hcamg_stream(dev.h)), device=f"cuda:{local}")
    b_dev = torch.from_numpy(b_host).to(f"cuda:{local}")
    x_dev = torch.zeros(n, dtype=torch.float64, device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    torch.cuda.synchronize()
    rep = _lib.Report()

    def solve_dev(report=None):
        dev.check(lib.hcamg_pcg_device(dev.h, C.c_void_p(b_dev.data_ptr()), None, 1e-8, 500,
                                       C.c_void_p(x_dev.data_ptr()), C.byref(report) if report else None))

    solve_dev(rep)
    iters = int(rep.iterations)
    assert rep.converged, "PCG did not converge"
    for _ in range(args.warmup):
        solve_dev()
    torch.cuda.synchronize()
    launches_per_solve = int(lib.hcamg_graph_launches(dev.h, 1)) + iters * int(lib.hcamg_graph_launches(dev.h, 2))
    barrier(dist)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        barrier(dist)
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                ev[k][0].record(stream)
            solve_dev()
            with torch.cuda.stream(stream):
                ev[k][1].record(stream)
        torch.cuda.synchronize()
        barrier(dist)
    t_steps = [a.elapsed_time(bb) * 1e-3 for a, bb in ev]
    t_total = reduce_max(dist, sum(t_steps))
    solve_dev(rep)
    assert int(rep.iterations) == iters
    work_total = reduce_sum(dist, float(n * iters * args.steps))
    value = work_total / t_total
    ms_per_step = 1e3 * t_total / args.steps

    # e2e: host buffers through the C-ABI (H2D of b, D2H of x + report inside the timed region)
    b_pin = torch.from_numpy(b_host).pin_memory()
    x_pin = torch.empty(n, dtype=torch.float64).pin_memory()
    hist = np.empty(500, dtype=np.float64)
    bp, xp = b_pin.numpy(), x_pin.numpy()
    for _ in range(max(1, args.warmup)):
        dev.check(lib.hcamg_pcg(dev.h, _lib.ptr(bp), None, 1e-8, 500, _lib.ptr(xp), _lib.ptr(hist), C.byref(rep)))
    te = 0.0
    barrier(dist)
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.check(lib.hcamg_pcg(dev.h, _lib.ptr(bp), None, 1e-8, 500, _lib.ptr(xp), _lib.ptr(hist), C.byref(rep)))
        te += time.perf_counter() - t0
    te = reduce_max(dist, te)
    e2e_value = work_total / te
    xs = x_pin.numpy()
    rel = float(np.linalg.norm(system.A @ xs - b_host) / np.linalg.norm(b_host))
    assert rel <= 1e-8 * 1.01, rel

    B_iter = algorithmic_bytes(h)
    peaks, peak_kind = measured_peaks()
    t_step = t_total / args.steps
    achieved = B_iter * iters / t_step / 1e9
    peak = float(peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    prof = None
    prof_path = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(prof_path):
        try:
            with open(prof_path) as f:
                prof = json.load(f)
        except Exception:
            prof = None

    line = {
        "metric": "AMG-PCG solve DoF*iters/s", "value": value, "unit": "DoF*iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {
            "workload": f"BASELINE {args.config}: unit cube, {kuhn.CONFIGS[args.config]['n']}^3 hexes x 6 Kuhn tets, "
                        f"{n} free edge DoFs, alg hierarchy, PCG tol 1e-8 from x0=0, rhs uniform[-1,1] seed 0",
            "levels": [lv.n for lv in h.levels], "pcg_iterations": iters,
            "setup_s": min(setups), "setup_s_first_call": setups[0],
            "operator_complexity": P.operator_complexity(h),
            "l2": "flushed (256 MiB write) before every timed step",
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
            "why_not_configs1": "BASELINE configs[1] (n=32) needs a 113 GB dense interior Cholesky + 35 GB dense "
                                "P block (SURVEY.md F3); round 1 runs the largest config that fits this build",
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": prof.get("dram_bytes_per_iteration") if prof else None,
                     "kernel": "one PCG iteration (CUDA-graph body: SpMV + vector ops + V-cycle kernels)",
                     "algorithmic_bytes_per_iteration": B_iter, "peak_kind": peak_kind,
                     "note": "config 1's hierarchy (~17 MB) is L2-resident; the solve is launch/latency-bound"},
        "e2e": {"value": e2e_value, "unit": "DoF*iters/s", "h2d_bytes_per_step": 8 * n + 128,
                "d2h_bytes_per_step": 8 * n + 8 * iters + 128},
        "gpu_launches": launches_per_solve * args.steps,
        "clocks": clk.result,
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        rate, solves, secs, it_o, setup_o = oracle_solve_rate(system, b_host, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": "DoF*iters/s", "cores": cpu_threads(), "kind": "port",
                                "sample": f"{solves} full PCG solves of {args.config} ({it_o} iterations each, "
                                          f"{secs:.1f} s) by oracle/amg_oracle.py; oracle setup {setup_o:.2f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world, rank, local, dist = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, world, rank, dist)
    else:
        run_ours(args, world, rank, local, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
