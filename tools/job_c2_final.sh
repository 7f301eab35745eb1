set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/z.pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/z.pytest.log
tail -3 gpurun_out/z.pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z.smoke.log 2>&1; tail -1 gpurun_out/z.smoke.log
timeout 900 python bench.py > gpurun_out/z.bench_c2.log 2>&1; tail -c 300 gpurun_out/z.bench_c2.log
timeout 600 python bench.py --config c1 > gpurun_out/z.bench_c1.log 2>&1; tail -c 200 gpurun_out/z.bench_c1.log
