# bench lines per store placement (per-resource roofline): C2 default, C3 and C5 with the
# tiered store (20% cache in HBM, misses over PCIe), C5 replicated; logs under gpurun_out/
mkdir -p gpurun_out/tiers
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tiers/c2.json 2> gpurun_out/tiers/c2.err
python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tiers/c3_hbm.json 2> gpurun_out/tiers/c3_hbm.err
python bench.py --config c3 --store cache --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tiers/c3_cache.json 2> gpurun_out/tiers/c3_cache.err
timeout 1200 python bench.py --config c5 --store cache --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/tiers/c5_cache.json 2> gpurun_out/tiers/c5_cache.err
timeout 1200 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/tiers/c5_hbm.json 2> gpurun_out/tiers/c5_hbm.err
for f in gpurun_out/tiers/*.json; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d['roofline']
print(d['config']['workload'], d['config'].get('store'), 'ms/step %.3f'%d['ms_per_step'], 'seeds/s %.3g'%d['value'], 'e2e %.3g'%d['e2e']['value'], 'frac %.3f'%r['frac'], 'pipelined %.3f'%r['pipelined']['frac'])
print(json.dumps(r.get('resources')), r.get('bound_resource'))
" 2>&1 | tail -3; done
