"""Fingerprints of the REFERENCE generator's graphs at the BASELINE scales.

Runs only where /root/reference exists (this container): the compiled,
unmodified reference (oracle/_ref) generates generate_power_law(n, m, 2.5, F,
seed 1) for C1, C2, C3 and C5 (C5 at F = 1: 1.6B edges,
~30 min and ~23 GB here) and records a sha256 per array. The product's
multithreaded generator must reproduce them (tests/test_host.py for C1-C3,
tests/test_scale_gpu.py for C5).

    python tests/golden/make_generator_hashes.py [c1 c2 c3 c5]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "generator_hashes.json")
CONFIGS = {"c1": (100_000, 3, 128), "c2": (233_000, 165, 602), "c3": (2_450_000, 9, 100),
           "c5": (111_000_000, 5, 1)}


def fingerprint(g) -> dict:
    out = {"num_nodes": int(len(g.labels)), "num_edges": int(len(g.col_indices))}
    for name in ("row_offsets", "col_indices", "features", "labels", "train_mask", "test_mask"):
        out[name] = hashlib.sha256(memoryview(getattr(g, name)).cast("B")).hexdigest()
    return out


def main(names):
    oracle.build(ref=True)
    ref = oracle.RefLib()
    rec = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        n, m, F = CONFIGS[name]
        t0 = time.time()
        g = ref.power_law(n, m, 2.5, F, 1)
        rec[name] = dict(gen=[n, m, F, 1], **fingerprint(g), reference_seconds=round(time.time() - t0, 1))
        del g
        with open(OUT, "w") as f:
            json.dump(rec, f, indent=1, sort_keys=True)
        print(name, rec[name]["num_edges"], rec[name]["reference_seconds"], flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3"])
