set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/so.pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/so.pytest.log
tail -4 gpurun_out/so.pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/so.smoke.log 2>&1; tail -1 gpurun_out/so.smoke.log
timeout 600 python bench.py --config c1 > gpurun_out/so.bench_c1.log 2>&1; tail -c 300 gpurun_out/so.bench_c1.log
HCAMG_SWEEP=leg timeout 600 python bench.py --config c1 --no-cpu-baseline > gpurun_out/so.bench_c1_leg.log 2>&1; grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*' gpurun_out/so.bench_c1_leg.log | head -2
timeout 900 python bench.py --config 2d-L9 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/so.bench_2d_L9.log 2>&1; grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*' gpurun_out/so.bench_2d_L9.log | head -2
timeout 900 python bench.py --config 2d-L10 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/so.bench_2d_L10.log 2>&1; grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*' gpurun_out/so.bench_2d_L10.log | head -2
python tools/profile_pieces.py c1 > gpurun_out/so.c1_pieces.log 2>&1; tail -8 gpurun_out/so.c1_pieces.log
