set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_forced_paths.py tests/test_gpu_smoothers.py tests/test_gpu_2d_large.py tests/test_gpu_parity.py tests/test_gpu_rows.py tests/test_gpu_api.py -x -q > gpurun_out/s.pytest.log 2>&1; tail -5 gpurun_out/s.pytest.log
for L in 9 10; do
timeout 900 python bench.py --config 2d-L$L --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/s.bench_2d_L$L.log 2>&1
grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*\|"setup_s": [0-9.]*\|"avg_launch_us": [0-9.]*\|"kernel": "[^"]*"\|"frac": [0-9.]*' gpurun_out/s.bench_2d_L$L.log | head -8
done
HCAMG_HOST_LOOP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s.2d_L10_launches.csv python bench.py --config 2d-L10 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/s.ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/s.2d_L10_launches.csv | head -24
