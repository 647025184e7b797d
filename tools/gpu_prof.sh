# tests + bench + launch list + ncu --set full of the named kernels (KERNELS="k_agg1 k_h1_tc")
mkdir -p gpurun_out
bash tools/gpu_tests.sh
python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > /dev/null 2>&1
for k in ${KERNELS:-k_agg1}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_$k python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/ncu_$k.log 2>&1
done
