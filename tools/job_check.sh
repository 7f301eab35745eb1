set -x
mkdir -p gpurun_out
./tools/probe/dblas_probe | grep -E "TF|diff"
timeout 600 python tools/profile_pieces.py c2 "" "opt:sweep=2,4" | grep -E "leg|sum"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g.pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/g.pytest.log
tail -3 gpurun_out/g.pytest.log
HCAMG_SETUP_TIMING=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g.bench_c2.log 2>&1; tail -c 400 gpurun_out/g.bench_c2.log; grep "bench\] setup" gpurun_out/g.bench_c2.log
timeout 900 python bench.py --config 2d-L9 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/g.bench_2d.log 2>&1; grep -o '"value": [0-9.e+-]*' gpurun_out/g.bench_2d.log | head -2
