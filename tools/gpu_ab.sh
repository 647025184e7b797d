# A/B: bench each config with ab/old.so and the in-tree library, alternating
mkdir -p gpurun_out
for rep in 1 2; do
for c in ${CONFIGS:-c2 c3}; do
  for v in old new; do
    if [ $v = old ]; then export A3G_LIB=$PWD/ab/old.so; else unset A3G_LIB; fi
    timeout 600 python bench.py --config $c --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/ab_${c}_${v}.log 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/ab_${c}_${v}.log').read().strip().splitlines()[-1]); print('$c $v', round(d['ms_per_step'],4), 'seq', round(d['roofline']['sequential_ms_per_step'],4))" 2>/dev/null || echo "$c $v failed"
  done
done
done
