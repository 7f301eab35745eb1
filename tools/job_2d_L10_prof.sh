set -x
mkdir -p gpurun_out
HCAMG_SETUP_TIMING=1 HCAMG_HOST_LOOP=1 timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p.2d_L10_launches.csv python bench.py --config 2d-L10 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/p.ncu1.log 2>&1
grep "hcamg setup" gpurun_out/p.ncu1.log | head -60
python tools/launch_summary.py gpurun_out/p.2d_L10_launches.csv | head -30
