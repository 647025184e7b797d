# A/B of library env knobs on the bench (C2 default): VARIANTS="A3G_LANE_CTA=64;A3G_LANE_CTA=128" CONFIG=c2
mkdir -p gpurun_out/ab
IFS=';' read -ra VS <<< "${VARIANTS}"
for rep in 1 2; do
for v in "" "${VS[@]}"; do
  tag=$(echo "base$v" | tr ' =/.' '____')
  env $v python bench.py --config ${CONFIG:-c2} --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline > gpurun_out/ab/$tag.json 2>/dev/null
  env $v A3G_DIAG_SKIP_COMPUTE=1 python bench.py --config ${CONFIG:-c2} --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline > gpurun_out/ab/$tag.samp.json 2>/dev/null
  python -c "
import json
a=json.loads(open('gpurun_out/ab/$tag.json').read().strip().splitlines()[-1]); b=json.loads(open('gpurun_out/ab/$tag.samp.json').read().strip().splitlines()[-1])
print('$rep %-40s step %.4f ms  sampling-only %.4f ms  agg-frac %.3f pipelined %.3f' % ('$tag', a['ms_per_step'], b['ms_per_step'], a['roofline']['frac'], a['roofline']['pipelined']['frac']))"
done
done
