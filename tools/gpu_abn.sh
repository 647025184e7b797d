# A/B/n: bench each config with each ab/<variant>.so, alternating, 2 reps
for rep in 1 2; do
for c in ${CONFIGS:-c2 c3}; do
  for v in ${VARIANTS:-base}; do
    export A3G_LIB=$PWD/ab/$v.so
    timeout 600 python bench.py --config $c --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/abn.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/abn.log').read().strip().splitlines()[-1]); print('$c $v', round(d['ms_per_step'],4), 'seq', round(d['roofline']['sequential_ms_per_step'],4))" 2>/dev/null || echo "$c $v failed"
  done
done
done
