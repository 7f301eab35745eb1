set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/y.pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/y.pytest.log
tail -3 gpurun_out/y.pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y.smoke.log 2>&1; tail -1 gpurun_out/y.smoke.log
timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/y.bench_c1.log 2>&1; grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*' gpurun_out/y.bench_c1.log | head -2
timeout 900 python bench.py --config 2d-L9 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/y.bench_2d_L9.log 2>&1; grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*' gpurun_out/y.bench_2d_L9.log | head -2
