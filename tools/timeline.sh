# per-kernel end times of two pipelined steps (A3G_TIMELINE=1) at 1 and 8 sampling streams, sampling only
mkdir -p gpurun_out/tl
for p in 1 8; do
  A3G_TIMELINE=1 A3G_DIAG_SKIP_COMPUTE=1 python bench.py --steps 8 --warmup 3 --pipeline $p --no-cpu-baseline > gpurun_out/tl/p$p.json 2> gpurun_out/tl/p$p.err
  A3G_STEP_TIMES=1 A3G_DIAG_SKIP_COMPUTE=1 python bench.py --steps 16 --warmup 3 --pipeline $p --no-cpu-baseline > /dev/null 2> gpurun_out/tl/steps_p$p.err
done
