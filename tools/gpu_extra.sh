mkdir -p gpurun_out
timeout 1200 python tools/sweep_c4.py --out gpurun_out/r01_c4_sweep.md > gpurun_out/sweep.log 2>&1
timeout 900 python bench.py --config c3 --steps 10 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --impl reference --steps 6 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --config c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
