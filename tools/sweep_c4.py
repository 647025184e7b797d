"""BASELINE config 4: cache-ratio x locality-bias sweep on the products-shaped
graph (C3: 2.45M nodes / 65M edges, F=100, fanout [15,10,5], batch 4096).

For every (cache ratio, gamma) cell the trainer places features with the
tiered store (A3G_STORE_CACHE: cached rows in HBM, misses in pinned host
memory read zero-copy over PCIe -- the B200 meaning of the reference's static
cache), trains K pipelined steps and reports
  * hit rate over the sampled unique nodes (the reference's epoch hit rate),
  * seeds/s (device-timed, the whole pipelined step),
  * mean loss over the K steps and its delta vs uniform sampling
    (SamplerKind::uniform_baseline) at the same cache ratio.
bias b = 1 - 1/gamma: gamma {1,2,4,8,16,32} <-> b {0,.5,.75,.875,.94,.97}.
Power-law labels are random (generators.cpp:142-145), so loss deltas carry no
accuracy signal on this graph; they are reported as
the reference reports them.

    python tools/sweep_c4.py [--steps K] [--out profiles/r01_c4_sweep.md]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--ratios", default="0.05,0.1,0.2,0.5,1.0")
    ap.add_argument("--gammas", default="1,2,4,8,16,32")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_c4_sweep.md"))
    ap.add_argument("--nodes", type=int, default=2_450_000)
    args = ap.parse_args()
    from paper_2511_07421_b200 import cache as CA, dp, graph as G, train as T
    F, fan, B = 100, [15, 10, 5], 4096
    t0 = time.time()
    g = G.generate_power_law(args.nodes, 9, 2.5, F, 1)
    gen_s = time.time() - t0
    gb, seeds = dp.global_batches(g.train_nodes, B, 1, args.steps + 2)
    rows = []
    for ratio in [float(x) for x in args.ratios.split(",")]:
        cache = CA.build_static_cache(g, CA.CacheConfig(int(ratio * g.num_nodes) * F * 4, 1))
        tr = T.Trainer(g, cache, T.ModelSpec(F, 16, 4), fan, max_seeds=B,
                       placement=dict(policy=G.STORE_CACHE if ratio < 1.0 else G.STORE_HBM))
        results = {}
        for kind, gamma in [(1, 1.0)] + [(0, float(x)) for x in args.gammas.split(",")]:
            tr.steps(gb[:2], seeds[:2], gamma, kind)  # warm-up
            losses = tr.steps(gb[2:], seeds[2:], gamma, kind)
            tm = tr.timing()
            st = tr.step_stats(args.steps).astype(np.int64)
            hits, misses = int(st[:, T.STAT_HITS].sum()), int(st[:, T.STAT_MISSES].sum())
            r = dict(cache_ratio=ratio, gamma=gamma, bias=1 - 1 / gamma, kind="uniform" if kind else "weighted",
                     hit_rate=hits / max(1, hits + misses), seeds_per_s=B * args.steps / (tm["total_ms"] / 1e3),
                     ms_per_step=tm["total_ms"] / args.steps, mean_loss=float(np.mean(losses)),
                     unique_per_batch=float(st[:, T.STAT_UNIQUE].mean()))
            results[(kind, gamma)] = r
        base = results[(1, 1.0)]["mean_loss"]
        for r in results.values():
            r["loss_delta_vs_uniform"] = r["mean_loss"] - base
            rows.append(r)
            print(json.dumps(r), flush=True)
        del tr
    with open(args.out, "w") as f:
        f.write("# C4: cache ratio x locality bias on the products-shaped graph (B200, 1 GPU)\n\n")
        f.write(f"Graph: generate_power_law({args.nodes}, 9, 2.5, F={F}, seed 1) ({gen_s:.0f} s host generation), "
                f"fanout {fan}, batch {B}, {args.steps} timed steps per cell after 2 warm-up steps. Feature "
                f"placement: tiered store, cached rows in HBM, misses in pinned host memory read zero-copy over "
                f"PCIe (ratio 1.0: all rows in HBM). Labels are random on power-law graphs, so loss deltas carry no "
                f"accuracy signal (SURVEY section 0 item 7).\n\n")
        f.write("| cache | sampler | gamma | bias | hit rate | unique/batch | ms/step | seeds/s | mean loss | "
                "loss - uniform |\n|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['cache_ratio']:.2f} | {r['kind']} | {r['gamma']:g} | {r['bias']:.3f} | {r['hit_rate']:.3f} | "
                    f"{r['unique_per_batch']:.0f} | {r['ms_per_step']:.2f} | {r['seeds_per_s']:.0f} | "
                    f"{r['mean_loss']:.4f} | {r['loss_delta_vs_uniform']:+.4f} |\n")
    print("wrote", args.out)


if __name__ == "__main__":
    main()
