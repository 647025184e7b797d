# sweep env knobs on C2/C3: lines "<config> <env> ms_per_step"
for c in ${CONFIGS:-c2 c3}; do
  for e in "X=0" "A3G_AGG_WARPS=16" "A3G_MERGE_CTAS4=2" "A3G_MERGE_CTAS4=4" "A3G_AGG_WARPS=16 A3G_MERGE_CTAS4=4"; do
    env $e timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/sw.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); print('$c', '$e', round(d['ms_per_step'],4))" || tail -2 gpurun_out/sw.log
  done
done
