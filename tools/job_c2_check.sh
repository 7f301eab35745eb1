set -x
mkdir -p gpurun_out
HCAMG_SETUP_TIMING=1 timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/c.bench_c2.log 2>&1
grep "hcamg setup" gpurun_out/c.bench_c2.log | head -40
tail -1 gpurun_out/c.bench_c2.log | cut -c1-900
