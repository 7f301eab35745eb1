# 2D stripes L=9: smoothing-leg modes side by side
set -x
mkdir -p gpurun_out
for m in auto wave flow; do
  HCAMG_SWEEP=$m timeout 900 python bench.py --config 2d-L9 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/m.bench_2d_$m.log 2>&1
  tail -c 1500 gpurun_out/m.bench_2d_$m.log | grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*\|"avg_launch_us": [0-9.]*\|"kernel": "[^"]*"' 
done
