set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_split_large.py tests/test_gpu_2d_large.py tests/test_gpu_kuhn_assembly.py -x -q > gpurun_out/g.pytest.log 2>&1; tail -5 gpurun_out/g.pytest.log
HCAMG_SETUP_TIMING=1 timeout 900 python bench.py --config 2d-L10 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/g.bench_2d_L10.log 2>&1
grep "hcamg setup" gpurun_out/g.bench_2d_L10.log | head -14
grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*\|"setup_s": [0-9.]*' gpurun_out/g.bench_2d_L10.log | head -4
