"""Feature cache on the device vs the oracle / reference tests (test_cache.cpp)."""
import numpy as np
import pytest

import oracle
from helpers import golden_graph, load_golden
from paper_2511_07421_b200 import _lib, cache as CA, graph as G, sampling as S

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["pl500", "pl3000"])
def test_static_cache_golden(name):
    rec = load_golden(name)
    g = golden_graph(rec)
    for nd in (1, 2, 4):
        c = CA.build_static_cache(g, CA.CacheConfig((g.num_nodes // 10) * g.feat_dim * 4, nd))
        assert np.array_equal(c.device_map, rec[f"cache{nd}"])


def test_static_cache_vs_oracle_sweep():
    orc = oracle.Oracle()
    g = G.generate_power_law(20_000, 3, 2.5, 16, 3)
    for vol_nodes in (0, 1, 7, 100, 2000, 20_000, 40_000):
        for nd in (1, 2, 3, 8):
            c = CA.build_static_cache(g, CA.CacheConfig(vol_nodes * 64, nd))
            assert np.array_equal(c.device_map, orc.build_static_cache(g, vol_nodes * 64, nd)), (vol_nodes, nd)
    with pytest.raises(_lib.ParameterError):
        CA.build_static_cache(g, CA.CacheConfig(64, 0))


def test_hotness_exact_set():
    """test_cache.cpp:30-49."""
    g = G.generate_power_law(1000, 2, 2.5, 16, 3)
    c = CA.build_static_cache(g, CA.CacheConfig(6400, 1))
    assert c.total_cached() == 100
    deg = np.diff(g.row_offsets)
    order = sorted(range(1000), key=lambda v: (-int(deg[v]), v))
    assert all(c.is_cached(v) for v in order[:100])


def test_retrieve_features_rows_and_bytes():
    """test_cache.cpp:100-131: exact rows, B = 64 / 800, accounting."""
    g = G.generate_power_law(50, 2, 2.5, 16, 9)
    c = CA.build_static_cache(g, CA.CacheConfig(0, 1))
    acc = CA.CacheAccounting(1)
    lone = S.SampleBatch(np.array([3], np.uint32), np.array([3], np.uint32), 1, [])
    f1, st1 = CA.retrieve_features(lone, c, g, acc)
    assert st1.batch_bytes == 64 and st1.num_edges == 0
    uniq = np.arange(10, dtype=np.uint32)
    d = np.array([e % 10 for e in range(20)], np.uint32)
    s = np.array([(e + 1) % 10 for e in range(20)], np.uint32)
    b = S.SampleBatch(np.array([0], np.uint32), uniq, 1, [(d, s)])
    feats, st = CA.retrieve_features(b, c, g, acc)
    assert st.batch_bytes == 800
    assert np.array_equal(feats.reshape(10, 16), g.features[:10])
    assert acc.total() == 11 and acc.misses == 11
    with pytest.raises(_lib.ParameterError):
        CA.hit_rate(CA.CacheAccounting(1))


def test_retrieve_features_sampled_batch_vs_oracle():
    orc = oracle.Oracle()
    g = G.generate_power_law(30_000, 3, 2.5, 100, 2)
    c = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * 400, 1))
    seeds = np.arange(0, 30_000, 31, dtype=np.uint32)
    ds = S.DeviceSampler(g, c, len(seeds), [15, 10, 5])
    ds.sample(seeds, 8.0, 0, 123)
    rows, hits, misses, B = ds.retrieve_features()
    ob = orc.sample_khop(g, seeds, [15, 10, 5], 8.0, 0, 123, c.device_map)
    orows, oh, om, oB = orc.retrieve_features(g, ob, c.device_map)
    assert np.array_equal(rows, orows)  # bit-exact gathered rows
    assert (hits, misses, B) == (oh, om, oB)
    acc = CA.CacheAccounting(1)
    CA.retrieve_features(ds.batch(), c, g, acc)
    assert abs(CA.hit_rate(acc) - oh / (oh + om)) < 1e-12


def test_lookup_on_device_two_devices():
    """cache.cpp:48-68 lookup on the device: per-id devices, any-device hit,
    per-device hits, over a 2-device round-robin placement."""
    g = G.generate_power_law(20_000, 3, 2.5, 8, 4)
    c = CA.build_static_cache(g, CA.CacheConfig(2000 * 8 * 4, 2))
    ids = np.arange(0, 20_000, 3, dtype=np.uint32)
    acc = CA.CacheAccounting(2)
    dev = CA.lookup(c, ids, acc)
    want = c.device_map[ids]
    assert np.array_equal(dev, want)
    assert acc.hits == int((want >= 0).sum()) and acc.misses == int((want < 0).sum())
    assert acc.per_device_hits == [int((want == 0).sum()), int((want == 1).sum())]
    with pytest.raises(_lib.ParameterError):
        CA.lookup(c, [20_000], acc)
