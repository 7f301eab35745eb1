set -x
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/t.pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/t.pytest.log
tail -5 gpurun_out/t.pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t.smoke.log 2>&1; tail -2 gpurun_out/t.smoke.log
