set -x
mkdir -p gpurun_out
SECONDS=0
HCAMG_SETUP_TIMING=1 timeout 2400 python bench.py --config 2d-L11 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/l11.bench.log 2>&1
echo "wall ${SECONDS}s"
grep "hcamg setup\] \(splitting\|interpolation\|galerkin\|smoother\)" gpurun_out/l11.bench.log | head -8
grep -o '"value": [0-9.]*, "unit"\|"ms_per_step": [0-9.]*\|"setup_s": [0-9.]*\|"frac": [0-9.]*\|"levels": [^]]*\]\|"pcg_iterations": [0-9]*' gpurun_out/l11.bench.log | head -10
tail -3 gpurun_out/l11.bench.log | cut -c1-300
