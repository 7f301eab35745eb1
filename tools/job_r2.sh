# round-2 final measurement job: tests, smoke, bench lines, launch lists and ncu captures
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f.pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/f.pytest.log
tail -3 gpurun_out/f.pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f.smoke.log 2>&1; tail -2 gpurun_out/f.smoke.log
timeout 900 python bench.py > gpurun_out/f.bench_c2.log 2>&1; tail -c 300 gpurun_out/f.bench_c2.log
timeout 600 python bench.py --config c1 > gpurun_out/f.bench_c1.log 2>&1; tail -c 300 gpurun_out/f.bench_c1.log
timeout 900 python bench.py --config 2d-L9 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/f.bench_2d.log 2>&1; tail -c 300 gpurun_out/f.bench_2d.log
HCAMG_HOST_LOOP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f.c2_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/f.ncu_bench.log 2>&1
HCAMG_HOST_LOOP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f.2d_bench_launches.csv python bench.py --config 2d-L9 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/f.ncu_bench2d.log 2>&1
timeout 900 ncu -k regex:k_flow_leg -s 2 -c 2 --set full --import-source on --clock-control none -o gpurun_out/f_flow_c2 python tools/flow_once.py c2 > gpurun_out/f.ncu_flow.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:k_tri_tma -c 2 --set full --import-source on --clock-control none -o gpurun_out/f_tri_c2 python tools/apply_p_once.py > gpurun_out/f.ncu_tri.log 2>&1
ls -la gpurun_out | tail -5
