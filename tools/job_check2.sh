set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/x.pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/x.pytest.log
tail -3 gpurun_out/x.pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x.smoke.log 2>&1; tail -1 gpurun_out/x.smoke.log
timeout 900 python bench.py > gpurun_out/x.bench_c2.log 2>&1; tail -c 2500 gpurun_out/x.bench_c2.log | grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*\|"setup_s": [0-9.]*\|"frac": [0-9.]*\|"true_relres": [0-9.e-]*\|"pcg_iterations": [0-9]*' | head -10
