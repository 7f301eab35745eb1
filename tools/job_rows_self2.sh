set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rows.py -x -q > gpurun_out/rs2.pytest.log 2>&1; tail -2 gpurun_out/rs2.pytest.log
for L in 9; do
for mode in plain self; do
  extra=""; [ $mode = self ] && extra="--rows-self"
  timeout 900 python bench.py --config 2d-L$L --steps 5 --warmup 2 --no-cpu-baseline $extra > gpurun_out/rs2.bench_2d_L${L}_$mode.log 2>&1
  grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*' gpurun_out/rs2.bench_2d_L${L}_$mode.log | head -2
done
done
