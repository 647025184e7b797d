# A/B of two library builds on one box: GPU tests on the in-tree build, then
# bench (C2, C3) alternating the in-tree build and $PWD/liba3g_old.so (A3G_LIB).
# Usage: cp the baseline .so to liba3g_old.so, rebuild, gpurun -- 'bash tools/ab_agg.sh'
python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/ab_tests.log
for cfg in c2 c3; do for r in 1 2; do
 for lib in new old; do
  if [ $lib = old ]; then export A3G_LIB=$PWD/liba3g_old.so; else unset A3G_LIB; fi
  python bench.py --config $cfg --no-cpu-baseline > /tmp/o.json 2>/tmp/e.log || tail -3 /tmp/e.log
  python -c "import json,sys;d=json.load(open('/tmp/o.json'));r=d['roofline'];print('$cfg','$lib',round(d['ms_per_step'],4),round(d['e2e']['value']/1e6,3),'agg_ms',round(r['ms_per_launch']*1000,1),'frac',round(r['frac'],3),'pipe_agg',round(r['pipelined']['ms_per_launch']*1000,1))" >> gpurun_out/ab.txt
 done; done; done
tail -2 gpurun_out/ab_tests.log; cat gpurun_out/ab.txt
