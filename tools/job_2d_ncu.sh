# 2D stripes L=10: full ncu captures of the sparse-regime kernels (level-0 launches are the first of each V-cycle)
set -x
mkdir -p gpurun_out
HCAMG_HOST_LOOP=1 timeout 1200 ncu --profile-from-start off -k regex:k_flow_wave -c 14 --set full --import-source on --clock-control none -o gpurun_out/n_2d_flow_wave python bench.py --config 2d-L10 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/n.ncu1.log 2>&1
HCAMG_HOST_LOOP=1 timeout 1200 ncu --profile-from-start off -k regex:k_spmv_sell -c 8 --set full --import-source on --clock-control none -o gpurun_out/n_2d_spmv_sell python bench.py --config 2d-L10 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/n.ncu2.log 2>&1
for f in n_2d_flow_wave n_2d_spmv_sell; do
ncu -i gpurun_out/$f.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,lts__t_sector_hit_rate.pct,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_barrier.ratio,l1tex__t_sector_hit_rate.pct > gpurun_out/$f.raw.csv 2>&1
ncu -i gpurun_out/$f.ncu-rep --page details > gpurun_out/$f.details.txt 2>&1
done
cut -d, -f5,12- gpurun_out/n_2d_flow_wave.raw.csv | head -20
cut -d, -f5,12- gpurun_out/n_2d_spmv_sell.raw.csv | head -12
