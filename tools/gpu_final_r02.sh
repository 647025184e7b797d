# r02 final evidence: full GPU suite, smoke, bench lines (C2 default with cpu_baseline, reference arm),
# launch lists (C2, C3), ncu --set full of k_agg1 (k_agg1_tma at C2) and the sampler's lane kernel
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/final/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -rA > gpurun_out/final/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1
python bench.py > gpurun_out/final/bench_c2.json 2> gpurun_out/final/bench_c2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final/ref_c2.json 2> gpurun_out/final/ref_c2.err
python bench.py --config c1 --no-cpu-baseline > gpurun_out/final/bench_c1.json 2>/dev/null
python bench.py --config c3 --no-cpu-baseline > gpurun_out/final/bench_c3.json 2>/dev/null
timeout 1500 python bench.py --config c5 --steps 20 --no-cpu-baseline > gpurun_out/final/bench_c5.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/final/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/final/launches_c3.csv python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_agg1 -s 3 -c 1 -o gpurun_out/final/prof_k_agg1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/final/prof_k_agg1.ncu-rep > gpurun_out/final/prof_k_agg1.txt 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream_lane_s -s 6 -c 1 -o gpurun_out/final/prof_lane python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/final/prof_lane.ncu-rep > gpurun_out/final/prof_lane.txt 2>/dev/null
python tools/ncu_lines.py gpurun_out/final/prof_lane.ncu-rep k_stream_lane 40 > gpurun_out/final/prof_lane_lines.txt 2>/dev/null
python tools/ncu_lines.py gpurun_out/final/prof_k_agg1.ncu-rep k_agg1 40 > gpurun_out/final/prof_k_agg1_lines.txt 2>/dev/null
python tools/kernel_table.py gpurun_out/final/launches_c2.csv > gpurun_out/final/launches_c2.txt 2>/dev/null
python tools/kernel_table.py gpurun_out/final/launches_c3.csv > gpurun_out/final/launches_c3.txt 2>/dev/null
ncu -i gpurun_out/final/prof_k_agg1.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
for row in r[2:]:
    d=dict(zip(h,row)); print('k_agg1 dram read', d.get('dram__bytes_read.sum'), 'write', d.get('dram__bytes_write.sum'), 'time', d.get('gpu__time_duration.sum'))
" > gpurun_out/final/k_agg1_traffic.txt
tail -3 gpurun_out/final/pytest_gpu.txt; tail -1 gpurun_out/final/smoke.txt
for f in gpurun_out/final/bench_*.json gpurun_out/final/ref_c2.json; do echo "== $f"; tail -1 $f | cut -c1-300; done
# the reports stay on the box (gpurun copies back at most 64 MiB); summaries above
rm -f gpurun_out/final/*.ncu-rep
