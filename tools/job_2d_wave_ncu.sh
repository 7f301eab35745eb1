# 2D stripes L=9, per-wave smoothing path: launch list + full ncu of the wave kernels
set -x
mkdir -p gpurun_out
HCAMG_SWEEP=wave HCAMG_HOST_LOOP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w.2d_wave_launches.csv python bench.py --config 2d-L9 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/w.ncu1.log 2>&1
python tools/launch_summary.py gpurun_out/w.2d_wave_launches.csv | head -30
HCAMG_SWEEP=wave HCAMG_HOST_LOOP=1 timeout 900 ncu --profile-from-start off -k regex:k_wave -s 1 -c 8 --set full --import-source on --clock-control none -o gpurun_out/w_2d_wave python bench.py --config 2d-L9 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/w.ncu2.log 2>&1
ncu -i gpurun_out/w_2d_wave.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,dram__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/w.2d_wave_raw.csv 2>&1
tail -12 gpurun_out/w.2d_wave_raw.csv
