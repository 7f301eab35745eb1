set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_forced_paths.py tests/test_gpu_parity.py tests/test_gpu_rows.py tests/test_gpu_2d_large.py -x -q > gpurun_out/b.pytest.log 2>&1; tail -3 gpurun_out/b.pytest.log
for L in 9 10 11; do
  SECONDS=0
  timeout 1500 python bench.py --config 2d-L$L --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b.bench_2d_L$L.log 2> gpurun_out/b.bench_2d_L$L.err
  echo "L=$L wall ${SECONDS}s"
  grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*\|"avg_launch_us": [0-9.]*\|"kernel": "[^"]*"\|"frac": [0-9.]*\|"levels": [^]]*\]\|"pcg_iterations": [0-9]*\|"setup_s": [0-9.]*' gpurun_out/b.bench_2d_L$L.log | head -12
  tail -3 gpurun_out/b.bench_2d_L$L.err
done
