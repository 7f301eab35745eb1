set -x
mkdir -p gpurun_out
HCAMG_SETUP_TIMING=1 timeout 900 python tools/setup_timing.py > gpurun_out/sp2.log 2>&1
grep "hcamg setup\|== build" gpurun_out/sp2.log | tail -45
