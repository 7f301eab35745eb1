set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_forced_paths.py tests/test_gpu_dense_regime.py tests/test_gpu_dense_c2field.py tests/test_gpu_factor_sweep.py tests/test_gpu_full_c2.py tests/test_gpu_dist.py -x -q > gpurun_out/dt.pytest.log 2>&1; tail -3 gpurun_out/dt.pytest.log
