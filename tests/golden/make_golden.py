"""Generate tests/golden/*.npz from the COMPILED, UNMODIFIED reference.

Runs only where /root/reference exists (this container): builds oracle/_ref
(the reference's own sources via oracle/Makefile) and records its outputs on
small inputs. The fixtures are committed; tests compare the C restatement
(oracle/) and the product against them anywhere, including the GPU box.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, n, min_degree, feat_dim, seed)
GRAPHS = [("pl500", 500, 2, 8, 3), ("pl3000", 3000, 3, 16, 1)]
# (fanouts, gamma, kind, rng_seed, cache_frac)
SAMPLE_CFGS = [([10, 5], 1.0, 0, 11, 0.2), ([10, 5], 8.0, 0, 12, 0.2), ([15, 10, 5], 4.0, 0, 13, 0.5),
               ([3], 2.0, 0, 14, 0.1), ([10, 5], 1.0, 1, 15, 0.2), ([5, 3, 2], 32.0, 0, 16, 1.0),
               ([40, 2], 8.0, 0, 17, 0.3), ([40], 1.0, 1, 18, 0.3)]


def main():
    oracle.build(ref=True)
    ref = oracle.RefLib()
    ref.L.ref_set_backend(0)  # scalar kernel table: the arithmetic order the C restatement follows
    for name, n, m, F, seed in GRAPHS:
        g = ref.power_law(n, m, 2.5, F, seed)
        rec = dict(row_offsets=g.row_offsets.copy(), col_indices=g.col_indices.copy(),
                   features=g.features.copy(), labels=g.labels.copy(), train_mask=g.train_mask.copy(),
                   test_mask=g.test_mask.copy(), gen=np.array([n, m, F, seed], dtype=np.uint64))
        rng = np.random.default_rng(seed)
        for ci, (fan, gamma, kind, rs, frac) in enumerate(SAMPLE_CFGS):
            vol = int(frac * n) * F * 4
            dm = ref.build_static_cache(g, vol, 1)
            seeds = rng.choice(n, size=min(64, n), replace=False).astype(np.uint32)
            seeds = np.concatenate([seeds, seeds[:5]])  # duplicate seeds are part of the contract
            b = ref.sample_khop(g, seeds, fan, gamma, kind, rs, dm)
            p = f"s{ci}_"
            rec[p + "cfg"] = np.array([gamma, kind, rs, vol], dtype=np.float64)
            rec[p + "fanouts"] = np.array(fan, dtype=np.uint32)
            rec[p + "seeds"] = seeds
            rec[p + "device_map"] = dm
            rec[p + "unique"] = b.unique_nodes
            rec[p + "meta"] = np.array([b.num_seed_unique, b.num_duplicates_removed], dtype=np.uint64)
            for l, (d, s) in enumerate(b.layers):
                rec[p + f"l{l}_dst"] = d
                rec[p + f"l{l}_src"] = s
        # cache over 2 and 4 devices
        for nd in (1, 2, 4):
            rec[f"cache{nd}"] = ref.build_static_cache(g, (n // 10) * F * 4, nd)
        # trainer: 2-layer, H=8, C=4, 6 steps at lr 0.2
        w1, w2 = ref.init_model(F, 8, 4, 1)
        rec["init_w1"], rec["init_w2"] = w1, w2
        dm = ref.build_static_cache(g, (n // 5) * F * 4, 1)
        rec["train_device_map"] = dm
        out = ref.train_steps(g, dm, [10, 5], 8.0, 0, 5, 64, 8, 4, 0.2, w1, w2, 6)
        rec["train_losses"], rec["train_w1"], rec["train_w2"] = out["losses"], out["w1"], out["w2"]
        one = ref.train_steps(g, dm, [10, 5], 8.0, 0, 5, 64, 8, 4, 0.0, w1, w2, 1)
        rec["step0_loss"] = one["losses"]
        # reference train(): loss curve over 2 epochs + accuracy
        tr = ref.train(g, dm, [10, 5], 8.0, 0, 5, 64, 2, 8, 4, 0.2, 1)
        rec["train_curve"], rec["train_hit_rates"] = tr["loss_curve"], tr["hit_rates"]
        rec["train_accuracy"] = np.array([tr["accuracy"]])
        tn = np.flatnonzero(g.train_mask).astype(np.uint32)
        rec["plan_e3"] = ref.plan_epoch_order(tn, 3, 99)
        rec["sampling_seeds"] = np.array([ref.sampling_seed(1, e, s, 0) for e in range(3) for s in range(4)],
                                         dtype=np.uint64)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        print("wrote", name, sum(v.nbytes for v in rec.values()), "bytes")
    # forward KAT (test_trainer.cpp:71-87): path fixture 0 <- 1 <- 2
    kat = ref.grad_on_edges(2, 2, 2, np.array([1.0, 0.5, -0.25, 1.0]), np.array([2.0, -1.0, 0.5, 3.0]), 3, 1,
                            [(np.array([0], np.uint32), np.array([1], np.uint32)),
                             (np.array([1], np.uint32), np.array([2], np.uint32))],
                            np.array([1, 2, 3, 4, -1, 6], np.float32), np.array([0], np.uint32))
    np.savez_compressed(os.path.join(OUT, "kat_path.npz"), logits=kat["logits"], loss=np.array([kat["loss"]]),
                        gw1=kat["gw1"], gw2=kat["gw2"])
    print("wrote kat_path")


if __name__ == "__main__":
    main()
