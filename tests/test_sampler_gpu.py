"""Parity of the sm_100a k-hop sampler against the oracle (bit-exact): golden
vectors from the compiled reference, C1-scale batches, a Reddit-shaped (C2)
slice with hubs, and the reference's own sampler tests (test_sampler.cpp)."""
import numpy as np
import pytest

import oracle
from helpers import assert_same_batch, golden_cfgs, golden_graph, load_golden
from paper_2511_07421_b200 import _lib, cache as CA, graph as G, sampling as S, train as T

pytestmark = pytest.mark.gpu


def cache_of(n, cached):
    dm = np.full(n, -1, dtype=np.int32)
    dm[np.asarray(cached, dtype=np.int64)] = 0
    return CA.CacheState(dm, 1)


def run(g, seeds, fanouts, gamma, kind, rng_seed, cache):
    cfg = S.SamplerConfig(list(fanouts), gamma, rng_seed, S.SamplerKind(kind))
    return S.sample_khop(g, seeds, cfg, cache)


@pytest.fixture(scope="module")
def orc():
    return oracle.Oracle()


@pytest.mark.parametrize("name", ["pl500", "pl3000"])
def test_golden_batches(name):
    rec = load_golden(name)
    g = golden_graph(rec)
    for i, c in enumerate(golden_cfgs(rec)):
        cache = CA.CacheState(c["device_map"], 1)
        b = run(g, c["seeds"], c["fanouts"], c["gamma"], c["kind"], c["rng_seed"], cache)
        assert_same_batch(b, c, f"{name} cfg{i}")


@pytest.fixture(scope="module")
def c1():
    """Config 1 graph: power law 100K nodes, m=3, F=128 (generators.cpp, seed 1)."""
    return G.generate_power_law(100_000, 3, 2.5, 128, 1)


@pytest.mark.parametrize("gamma,kind", [(1.0, 0), (8.0, 0), (32.0, 0), (1.0, 1)])
def test_c1_batches_vs_oracle(c1, orc, gamma, kind):
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    batches = T.plan_epoch_batches(g.train_nodes, 0, 1024, orc.hash2(1, 0))
    for step in range(6):
        rs = T.sampling_seed(1, 0, step, 0)
        a = run(g, batches[step], [10, 5], gamma, kind, rs, cache)
        b = orc.sample_khop(g, batches[step], [10, 5], gamma, kind, rs, cache.device_map)
        assert_same_batch(a, b, f"c1 step {step} gamma {gamma} kind {kind}")


def test_c1_three_hops_and_wide_fanout(c1, orc):
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.5 * g.num_nodes) * g.feat_dim * 4, 1))
    seeds = np.arange(0, 100_000, 97, dtype=np.uint32)
    for fan, gamma in [([15, 10, 5], 4.0), ([40, 3], 8.0), ([1, 1, 1, 1], 2.0), ([32], 8.0), ([33], 8.0)]:
        a = run(g, seeds, fan, gamma, 0, 77, cache)
        b = orc.sample_khop(g, seeds, fan, gamma, 0, 77, cache.device_map)
        assert_same_batch(a, b, f"fan {fan}")
        a = run(g, seeds, fan, 1.0, 1, 78, cache)
        b = orc.sample_khop(g, seeds, fan, 1.0, 1, 78, cache.device_map)
        assert_same_batch(a, b, f"uniform fan {fan}")


@pytest.mark.parametrize("gamma", [2.0, 8.0, 1000.0])
def test_c1_full_cache_integer_keys(c1, orc, gamma):
    """Every neighbour cached: the sampler compares u-space integer keys
    (PolGammaAll) with exact pow only on near-ties; must equal the oracle."""
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(g.num_nodes * g.feat_dim * 4, 1))
    seeds = np.arange(3, 100_000, 53, dtype=np.uint32)
    for fan in ([15, 10, 5], [25, 3]):
        a = run(g, seeds, fan, gamma, 0, 4242, cache)
        b = orc.sample_khop(g, seeds, fan, gamma, 0, 4242, cache.device_map)
        assert_same_batch(a, b, f"full cache gamma {gamma} fan {fan}")


@pytest.mark.parametrize("gamma,ratio", [(1.0, 1.0), (8.0, 1.0), (8.0, 0.3), (2.0, 0.05)])
def test_lane_per_item_stream_layers(c1, orc, gamma, ratio):
    """Layers whose frontier bound reaches 32768 rows run the lane-per-item
    stream (register reservoirs of 5, 8, 10 or 16 slots; integer keys with a full
    cache, fp64 keys over the per-edge cached bits with a partial one);
    [20, 12] / [40, 7] from ~1900 seeds put layer 1 there with m = 12 and
    m = 7 (hubs included)."""
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(ratio * g.num_nodes) * g.feat_dim * 4, 1))
    seeds = np.arange(5, 100_000, 53, dtype=np.uint32)
    for fan in ([20, 12], [40, 7], [20, 10], [30, 5]):  # register reservoirs of 16, 8, 10 and 5 slots
        assert len(seeds) * fan[0] >= 32768
        a = run(g, seeds, fan, gamma, 0, 99, cache)
        b = orc.sample_khop(g, seeds, fan, gamma, 0, 99, cache.device_map)
        assert_same_batch(a, b, f"lane gamma {gamma} fan {fan}")


@pytest.mark.slow
def test_c2_reddit_shaped_slice(orc):
    """Config 2 shape: 233K nodes, m=165 (mean deg ~484, hubs up to n-1),
    [15,10,5], B=1024, full cache, gamma 8 -> every key is a gamma key."""
    g = G.generate_power_law(233_000, 165, 2.5, 1, 1)
    cache = CA.build_static_cache(g, CA.CacheConfig(g.num_nodes * g.feat_dim * 4, 1))
    assert cache.total_cached() == g.num_nodes
    batches = T.plan_epoch_batches(g.train_nodes, 0, 1024, orc.hash2(1, 0))
    for step, gamma in [(0, 8.0), (1, 1.0)]:
        rs = T.sampling_seed(1, 0, step, 0)
        a = run(g, batches[step], [15, 10, 5], gamma, 0, rs, cache)
        b = orc.sample_khop(g, batches[step], [15, 10, 5], gamma, 0, rs, cache.device_map)
        assert_same_batch(a, b, f"c2 step {step}")


def test_isolated_seed_and_errors():
    """test_sampler.cpp:158-169."""
    g = G.from_edges(3, [(1, 2)], 2)
    c = cache_of(3, [])
    b = run(g, [0], [5], 1.0, 0, 4, c)
    assert b.unique_nodes.tolist() == [0] and b.total_edges() == 0
    assert S.dedup_ratio(b) == 0.0
    with pytest.raises(_lib.ParameterError):
        run(g, [7], [5], 1.0, 0, 4, c)
    with pytest.raises(_lib.ParameterError):
        run(g, [], [5], 1.0, 0, 4, c)
    with pytest.raises(_lib.ParameterError):
        run(g, [1], [0], 1.0, 0, 4, c)
    with pytest.raises(_lib.ParameterError):  # assign_weights gamma < 1 (seed has neighbours)
        run(g, [1], [5], 0.5, 0, 4, c)
    b = run(g, [0], [5], 0.5, 0, 4, c)  # isolated seed: the reference never calls assign_weights
    assert b.total_edges() == 0


def test_exhaustive_fanout_reproduces_all_edges():
    """test_sampler.cpp:171-187 (all nodes as seeds, fanout = max degree)."""
    g = G.generate_power_law(300, 2, 2.5, 4, 5)
    fan = int(np.diff(g.row_offsets).max())
    b = run(g, np.arange(300), [fan], 1.0, 0, 6, cache_of(300, []))
    assert b.total_edges() == g.num_edges
    got = sorted(zip(b.unique_nodes[b.layers[0][0]].tolist(), b.unique_nodes[b.layers[0][1]].tolist()))
    want = sorted((v, int(u)) for v in range(300) for u in g.out_neighbors(v))
    assert got == want
    S.validate_batch(g, b)


def test_determinism_and_validity():
    """test_sampler.cpp:189-203."""
    g = G.generate_power_law(300, 2, 2.5, 4, 8)
    c = cache_of(300, [1, 2, 3, 4, 5])
    a = run(g, [10, 20, 30], [5, 3], 4.0, 0, 42, c)
    b = run(g, [10, 20, 30], [5, 3], 4.0, 0, 42, c)
    assert np.array_equal(a.unique_nodes, b.unique_nodes)
    for (d1, s1), (d2, s2) in zip(a.layers, b.layers):
        assert np.array_equal(d1, d2) and np.array_equal(s1, s2)
    S.validate_batch(g, a)


def test_star_dedup_ratio():
    """test_sampler.cpp:241-256: (s-1)/(2s-1)."""
    s = 6
    g = G.from_edges(s, [(leaf, 0) for leaf in range(1, s)], 2)
    b = run(g, np.arange(s), [1], 1.0, 0, 1, cache_of(s, []))
    assert b.num_duplicates_removed == s - 1 and len(b.unique_nodes) == s
    assert abs(S.dedup_ratio(b) - (s - 1) / (2 * s - 1)) < 1e-12


def test_biased_draw_probability_at_scale():
    """test_sampler.cpp:145-156 through the real kernel: 100K frontier nodes
    each choose 1 of {A, B} with B cached at gamma=4 -> P(B) = 4/5."""
    N = 100_000
    A, B = N, N + 1
    edges = [(v, A) for v in range(N)] + [(v, B) for v in range(N)]
    g = G.from_edges(N + 2, edges, 1)
    b = run(g, np.arange(N), [1], 4.0, 0, 99, cache_of(N + 2, [B]))
    src_nodes = b.unique_nodes[b.layers[0][1]]
    p = float((src_nodes == B).mean())
    assert abs(p - 0.8) < 0.0125 * 0.8
    b = run(g, np.arange(N), [1], 1.0, 1, 98, cache_of(N + 2, [B]))  # uniform baseline: 1/2
    p = float((b.unique_nodes[b.layers[0][1]] == B).mean())
    assert abs(p - 0.5) < 0.01


def test_bias_raises_cached_fraction_and_dedup():
    """test_sampler.cpp:205-239 and :258-288."""
    g = G.generate_power_law(1000, 2, 2.5, 4, 17)
    deg = np.diff(g.row_offsets)
    order = sorted(range(1000), key=lambda v: (-int(deg[v]), v))
    c = cache_of(1000, order[:100])

    def stats(gamma):
        frac = ratio = 0.0
        for seed in range(20):
            seeds = np.random.default_rng(seed).integers(0, 1000, 32)
            b = run(g, seeds, [10, 5], gamma, 0, seed, c)
            frac += np.mean([c.is_cached(int(v)) for v in b.unique_nodes])
            ratio += S.dedup_ratio(b)
        return frac / 20, ratio / 20

    f1, r1 = stats(1.0)
    f8, r8 = stats(8.0)
    assert f8 > f1
    assert r8 >= r1 - 1e-9


def test_explicit_reservoirs_vs_oracle(orc):
    rng = np.random.default_rng(3)
    for t in range(30):
        n = int(rng.integers(0, 300))
        nb = rng.integers(0, 10**6, size=n).astype(np.uint32)
        w = rng.choice([1.0, 9.0, 0.2, 4.0], size=n)
        m = int(rng.integers(1, 45))
        key = orc.hash2(int(rng.integers(0, 2**62)), t)
        ctr0 = int(rng.integers(0, 3))
        a, _ = S.weighted_reservoir_sample(nb, w, m, key, ctr0)
        b, _ = orc.weighted_reservoir(nb, w, m, key, ctr0)
        assert np.array_equal(a, b), f"weighted trial {t}"
        a, _ = S.uniform_reservoir_sample(nb, m, key, ctr0)
        b, _ = orc.uniform_reservoir(nb, m, key, ctr0)
        assert np.array_equal(a, b), f"uniform trial {t}"
    with pytest.raises(_lib.ParameterError):
        S.weighted_reservoir_sample([1, 2], [1.0, 0.0], 1, 5)
    with pytest.raises(_lib.ParameterError):
        S.weighted_reservoir_sample([1, 2], [1.0, 1.0], 0, 5)
    assert len(S.weighted_reservoir_sample([], [], 3, 5)[0]) == 0
