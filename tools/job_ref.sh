mkdir -p gpurun_out
timeout 2400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.c2.log 2>&1; tail -c 1500 gpurun_out/ref.c2.log
timeout 600 python bench.py --impl reference --config c1 --steps 20 --warmup 5 > gpurun_out/ref.c1.log 2>&1; tail -c 600 gpurun_out/ref.c1.log
timeout 1800 python bench.py --impl reference --config 2d-L9 --steps 1 --warmup 0 > gpurun_out/ref.2d.log 2>&1; tail -c 600 gpurun_out/ref.2d.log
