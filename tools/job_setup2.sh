set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_forced_paths.py tests/test_gpu_dense_regime.py tests/test_gpu_dense_c2field.py tests/test_gpu_factor_sweep.py tests/test_gpu_api.py tests/test_gpu_full_c2.py -x -q -m gpu > gpurun_out/sp.pytest.log 2>&1; tail -3 gpurun_out/sp.pytest.log
HCAMG_SETUP_TIMING=1 timeout 900 python tools/setup_timing.py > gpurun_out/sp.log 2>&1
grep "hcamg setup\|== build" gpurun_out/sp.log | tail -48
