# one ncu --set full capture: KERNEL regex, SKIP launches, OUT name
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL} -s ${SKIP:-0} -c ${COUNT:-1} -o gpurun_out/${OUT} python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/${OUT}.log 2>&1
