for c in c2 c1 c3; do for t in 1024 8192 32768 1000000000; do
A3G_LANE_MIN_ROWS=$t timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/sw.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); print('$c', $t, round(d['ms_per_step'],4))"
done; done
