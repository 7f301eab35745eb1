# what the row partition costs on one GPU: the default kernels with and without the
# partitioned step program (row lists / compacted records, one boundary kernel per step, split reductions)
mkdir -p gpurun_out
for L in 9 10; do
for mode in plain self; do
  extra=""; [ $mode = self ] && extra="--rows-self"
  timeout 900 python bench.py --config 2d-L$L --steps 5 --warmup 2 --no-cpu-baseline $extra > gpurun_out/rsa.bench_2d_L${L}_$mode.log 2>&1
  grep -o 'one-rank row partition.*' gpurun_out/rsa.bench_2d_L${L}_$mode.log | cut -c1-700
  grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*\|"gpu_launches": [0-9]*\|"pcg_iterations": [0-9]*' gpurun_out/rsa.bench_2d_L${L}_$mode.log | head -5
done
done
