# usage (on the GPU box, via gpurun): bash tools/gpujob.sh TAG "pytest args" [bench]
set -x
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$TAG.smi 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q ${2:-} > gpurun_out/$TAG.pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/$TAG.pytest.log
tail -3 gpurun_out/$TAG.pytest.log
if [ "${3:-}" = "bench" ]; then
  HCAMG_SETUP_TIMING=1 timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/$TAG.bench.log 2>&1; echo bench_rc=$? >> gpurun_out/$TAG.bench.log
  tail -c 3000 gpurun_out/$TAG.bench.log
fi
