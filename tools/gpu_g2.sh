bash tools/gpu_tests.sh
python bench.py --no-cpu-baseline > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err
A3G_SIMT_GEMM=1 python bench.py --no-cpu-baseline > gpurun_out/bench_simt.json 2> gpurun_out/bench_simt.err
tail -3 gpurun_out/bench_tc.err
