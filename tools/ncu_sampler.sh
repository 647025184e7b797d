# instruction counts of every kernel of one sampling batch + a full capture of the L2 lane kernel
mkdir -p gpurun_out/ncu
A3G_DIAG_SKIP_COMPUTE=1 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/ncu/samp_metrics.csv python bench.py --steps 3 --warmup 3 --pipeline 0 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream_lane -s 3 -c 1 -o gpurun_out/ncu/lane_l2 python bench.py --steps 3 --warmup 3 --pipeline 0 --no-cpu-baseline > gpurun_out/ncu/lane_l2.log 2>&1
ncu -i gpurun_out/ncu/lane_l2.ncu-rep --page details --csv > gpurun_out/ncu/lane_l2_details.csv 2>/dev/null
ncu -i gpurun_out/ncu/lane_l2.ncu-rep --page raw --csv > gpurun_out/ncu/lane_l2_raw.csv 2>/dev/null
ls -la gpurun_out/ncu
