set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests3.log 2>&1; echo pytest_rc=$? >> gpurun_out/gputests3.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_c2.json.log 2>&1
timeout 300 python bench.py --config c1 > gpurun_out/bench_c1.json.log 2>&1
HCAMG_HOST_LOOP=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --profile-from-start off -k regex:k_tri_tma -c 1 --set full --clock-control none --import-source on -o gpurun_out/tri_tma_full python tools/apply_p_once.py > gpurun_out/ncu_tri.log 2>&1
ls -la gpurun_out
