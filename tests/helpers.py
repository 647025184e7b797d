"""Shared test helpers: golden fixtures as product/oracle graphs, batch compare."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def golden_graph(rec):
    from paper_2511_07421_b200 import graph as G
    return G.from_arrays(rec["row_offsets"], rec["col_indices"], rec["features"], rec["labels"],
                         rec["train_mask"], rec["test_mask"])


def golden_cfgs(rec):
    i = 0
    while f"s{i}_cfg" in rec:
        p = f"s{i}_"
        gamma, kind, rs, vol = rec[p + "cfg"]
        fan = rec[p + "fanouts"]
        layers = [(rec[p + f"l{l}_dst"], rec[p + f"l{l}_src"]) for l in range(len(fan))]
        yield dict(fanouts=[int(x) for x in fan], gamma=float(gamma), kind=int(kind), rng_seed=int(rs),
                   volume=int(vol), seeds=rec[p + "seeds"], device_map=rec[p + "device_map"],
                   unique=rec[p + "unique"], num_seed_unique=int(rec[p + "meta"][0]),
                   dups=int(rec[p + "meta"][1]), layers=layers)
        i += 1


def assert_same_batch(a, b, ctx=""):
    """Bit-exact SampleBatch equality (unique order, edges per layer, counters)."""
    au = np.asarray(a.unique_nodes)
    bu = np.asarray(b["unique"] if isinstance(b, dict) else b.unique_nodes)
    assert au.shape == bu.shape and np.array_equal(au, bu), f"{ctx}: unique_nodes differ"
    ns = b["num_seed_unique"] if isinstance(b, dict) else b.num_seed_unique
    dd = b["dups"] if isinstance(b, dict) else b.num_duplicates_removed
    assert a.num_seed_unique == ns, f"{ctx}: num_seed_unique {a.num_seed_unique} != {ns}"
    assert a.num_duplicates_removed == dd, f"{ctx}: dups {a.num_duplicates_removed} != {dd}"
    bl = b["layers"] if isinstance(b, dict) else b.layers
    assert len(a.layers) == len(bl)
    for l, ((d1, s1), (d2, s2)) in enumerate(zip(a.layers, bl)):
        assert np.array_equal(np.asarray(d1), np.asarray(d2)), f"{ctx}: layer {l} dst differ"
        assert np.array_equal(np.asarray(s1), np.asarray(s2)), f"{ctx}: layer {l} src differ"


def rel_err(a, b, floor=1e-6):
    """Norm-wise relative error ||a-b|| / max(||b||, floor)."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), floor))
