# tests + C2 bench (+ optional extra configs) on the box; logs under gpurun_out/
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-c2}; do
  timeout 600 python bench.py --config $c ${BENCH_ARGS:-} > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/bench_$c.log | cut -c1-600
done
