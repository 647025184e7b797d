for c in 0 1 2 3 4; do A3G_AGG_CFG=$c python bench.py --no-cpu-baseline --steps 20 > gpurun_out/agg_cfg$c.json 2>/dev/null; done
