for c in ${CONFIGS:-c2 c3}; do for v in ${SEGS:-1024 2048 4096}; do
A3G_SEG=$v timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/sw.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); print('$c seg', $v, round(d['ms_per_step'],4), 'seq', round(d['roofline']['sequential_ms_per_step'],4))" || tail -2 gpurun_out/sw.log
done; done
