# wide-hidden (tcgen05 dense update) tests + C3 bench lines at H = 16 / 128 / 256 + ncu of the GEMMs
mkdir -p gpurun_out/wide
timeout 900 python -m pytest tests/test_trainer_gpu.py -x -q --timeout 600 2>&1 | tail -3
for h in 128 256; do
  python bench.py --config c3 --hidden $h --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/wide/c3_h$h.json 2> gpurun_out/wide/c3_h$h.err
  tail -1 gpurun_out/wide/c3_h$h.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('H', d['config']['hidden'], 'ms/step', round(d['ms_per_step'],4), 'seeds/s %.3g'%d['value'], json.dumps(d.get('tensor_roofline')))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_h1_tc|k_dw1_tc" -s 4 -c 2 -o gpurun_out/wide/tc_h128 python bench.py --config c3 --hidden 128 --steps 3 --warmup 3 --no-cpu-baseline --pipeline 0 > gpurun_out/wide/ncu.log 2>&1
ncu -i gpurun_out/wide/tc_h128.ncu-rep --page details --csv > gpurun_out/wide/tc_h128_details.csv 2>/dev/null
ncu -i gpurun_out/wide/tc_h128.ncu-rep --page raw --csv > gpurun_out/wide/tc_h128_raw.csv 2>/dev/null
