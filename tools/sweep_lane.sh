# frontier-bound threshold of the lane-per-item stream kernels
for c in ${CONFIGS:-c3 c5 c2}; do for t in ${THRS:-32768 65536 131072}; do
A3G_LANE_MIN_ROWS=$t timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/sw.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); print('$c', $t, round(d['ms_per_step'],4))" || tail -2 gpurun_out/sw.log
done; done
