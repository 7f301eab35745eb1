set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_rows.py -x -q > gpurun_out/r.pytest.log 2>&1; tail -30 gpurun_out/r.pytest.log
