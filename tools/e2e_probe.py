import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import bench
from paper_2511_07421_b200 import cache as CA, train as T, dp
cfg = sys.argv[1]
n, m, F, fan, B, frac, _ = bench.CONFIGS[cfg]
g = bench.make_graph(cfg)
synth = cfg in bench.SYNTH
cache = CA.build_static_cache(g, CA.CacheConfig(int(frac * n) * (1 if synth else F) * 4, 1))
tr = T.Trainer(g, cache, T.ModelSpec(F, 16, 4), fan, max_seeds=B, feat_dtype=1 if synth else 0, synth_seed=1 if synth else None)
gb, gs = dp.global_batches(g.train_nodes, B, 1, 70, 1)
tr.steps(gb[:3], gs[:3], 8.0, 0)
for K in (20, 20, 40):
    t0 = time.perf_counter(); tr.steps(gb[3:3 + K], gs[3:3 + K], 8.0, 0); t1 = time.perf_counter()
    print(cfg, K, "wall ms/step %.3f" % ((t1 - t0) * 1e3 / K), "device ms/step %.3f" % (tr.timing()["total_ms"] / K), flush=True)
