cp paper_2511_07421_b200/liba3g_b200.so /tmp/lib2048.so
for K in 2048 4096 8192; do
  if [ $K != 2048 ]; then cp tools/kseg_exp/lib$K.so paper_2511_07421_b200/liba3g_b200.so; else cp /tmp/lib2048.so paper_2511_07421_b200/liba3g_b200.so; fi
  for c in c2 c3; do python bench.py --config $c --no-cpu-baseline > gpurun_out/kseg_${K}_$c.json 2>/dev/null; done
done
cp /tmp/lib2048.so paper_2511_07421_b200/liba3g_b200.so
