# round-2 final measurement job: tests, smoke, bench lines, reference arms, launch lists, ncu captures
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/z.pytest.log 2>&1; echo pytest_rc=$? >> gpurun_out/z.pytest.log
tail -3 gpurun_out/z.pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z.smoke.log 2>&1; tail -2 gpurun_out/z.smoke.log
timeout 900 python bench.py > gpurun_out/z.bench_c2.log 2>&1; tail -c 300 gpurun_out/z.bench_c2.log
timeout 600 python bench.py --config c1 > gpurun_out/z.bench_c1.log 2>&1; tail -c 300 gpurun_out/z.bench_c1.log
timeout 900 python bench.py --config 2d-L9 --steps 5 --warmup 3 > gpurun_out/z.bench_2d_L9.log 2>&1; tail -c 300 gpurun_out/z.bench_2d_L9.log
timeout 900 python bench.py --config 2d-L10 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/z.bench_2d_L10.log 2>&1; tail -c 300 gpurun_out/z.bench_2d_L10.log
HCAMG_HOST_LOOP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z.c2_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/z.ncu_bench.log 2>&1
HCAMG_HOST_LOOP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z.2d_L9_bench_launches.csv python bench.py --config 2d-L9 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/z.ncu_bench2d.log 2>&1
HCAMG_HOST_LOOP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/z.2d_L10_bench_launches.csv python bench.py --config 2d-L10 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/z.ncu_bench2d10.log 2>&1
timeout 900 ncu -k regex:k_flow_leg -s 2 -c 2 --set full --import-source on --clock-control none -o gpurun_out/z_flow_c2 python tools/flow_once.py c2 > gpurun_out/z.ncu_flow.log 2>&1
timeout 900 ncu --profile-from-start off -k regex:k_tri_tma -c 2 --set full --import-source on --clock-control none -o gpurun_out/z_tri_c2 python tools/apply_p_once.py > gpurun_out/z.ncu_tri.log 2>&1
for f in z_flow_c2 z_tri_c2; do ncu -i gpurun_out/$f.ncu-rep --page details > gpurun_out/$f.details.txt 2>&1; done
timeout 600 python bench.py --impl reference --config c1 --steps 20 --warmup 5 > gpurun_out/z.ref.c1.log 2>&1; tail -c 600 gpurun_out/z.ref.c1.log
timeout 1800 python bench.py --impl reference --config 2d-L9 --steps 1 --warmup 0 > gpurun_out/z.ref.2d.log 2>&1; tail -c 600 gpurun_out/z.ref.2d.log
timeout 2400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/z.ref.c2.log 2>&1; tail -c 1500 gpurun_out/z.ref.c2.log
ls -la gpurun_out | tail -30
