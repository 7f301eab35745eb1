# new per-wave kernel: parity tests + 2D bench
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_forced_paths.py tests/test_gpu_smoothers.py tests/test_gpu_2d_large.py tests/test_gpu_parity.py -x -q > gpurun_out/w2.pytest.log 2>&1; tail -5 gpurun_out/w2.pytest.log
timeout 900 python bench.py --config 2d-L9 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/w2.bench_2d.log 2>&1
grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*\|"avg_launch_us": [0-9.]*\|"kernel": "[^"]*"\|"frac": [0-9.]*' gpurun_out/w2.bench_2d.log | head
HCAMG_HOST_LOOP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w2.2d_launches.csv python bench.py --config 2d-L9 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/w2.ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/w2.2d_launches.csv | head -24
