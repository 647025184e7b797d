# bench lines (C2 default with cpu_baseline; C1/C3/C5), launch lists, ncu --set full of the main kernels
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final/smi.txt 2>&1
python bench.py > gpurun_out/final/bench_c2.json 2> gpurun_out/final/bench_c2.err
python bench.py --config c1 --no-cpu-baseline > gpurun_out/final/bench_c1.json 2>/dev/null
python bench.py --config c3 --no-cpu-baseline > gpurun_out/final/bench_c3.json 2>/dev/null
timeout 1500 python bench.py --config c5 --steps 10 --no-cpu-baseline > gpurun_out/final/bench_c5.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/final/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/final/launches_c3.csv python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for spec in "k_agg1:3" "k_stream_lane:4" "k_stream_grp:2" "k_dw1_fma:3" "k_hub_merge:4"; do
  k=${spec%%:*}; sk=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c 1 -o gpurun_out/final/prof_$k python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream_lane_mixed -s 2 -c 1 -o gpurun_out/final/prof_k_stream_lane_mixed python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/final
# summaries on the box; keep only two full reports (gpurun_out/ must stay < 64 MiB)
for f in gpurun_out/final/prof_*.ncu-rep; do
  python tools/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>/dev/null
done
python tools/kernel_table.py gpurun_out/final/launches_c2.csv > gpurun_out/final/launches_c2.txt 2>/dev/null
python tools/kernel_table.py gpurun_out/final/launches_c3.csv > gpurun_out/final/launches_c3.txt 2>/dev/null
python tools/ncu_lines.py gpurun_out/final/prof_k_stream_lane.ncu-rep k_stream_lane 40 > gpurun_out/final/lines_k_stream_lane.txt 2>/dev/null
python tools/ncu_lines.py gpurun_out/final/prof_k_agg1.ncu-rep k_agg1 40 > gpurun_out/final/lines_k_agg1.txt 2>/dev/null
for k in k_dw1_fma k_hub_merge k_stream_grp k_stream_lane_mixed; do rm -f gpurun_out/final/prof_$k.ncu-rep; done
du -sh gpurun_out
