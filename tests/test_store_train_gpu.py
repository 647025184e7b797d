"""Tiered feature store, per-step statistics, the device train() loop and the
full-graph evaluation (trainer.cpp:241-303, 350-424) against the reference.

* store placement must not change any result: the same rows are read from
  HBM, pinned host or a peer shard, in the same order -> bit-identical losses
  and gradients across policies;
* train(): loss curve within 1e-3 relative of the fp64 reference, epoch hit
  rates exact (they count unique nodes, sampling is bit-exact), accuracy
  within 2 test nodes (fp32 vs fp64 argmax near-ties);
* evaluate_full_graph against a numpy fp64 restatement (test infrastructure).
"""
import numpy as np
import pytest

import oracle
from helpers import golden_graph, load_golden, rel_err
from paper_2511_07421_b200 import cache as CA, graph as G, sampling as S, train as T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    return oracle.Oracle()


@pytest.fixture(scope="module")
def c1():
    return G.generate_power_law(100_000, 3, 2.5, 128, 1)


def _steps(tr, g, K=4, B=512, gamma=8.0):
    batches = T.plan_epoch_batches(g.train_nodes, 0, B, 77)[:K]
    seeds = np.concatenate(batches)
    off = np.cumsum([0] + [len(b) for b in batches]).astype(np.uint64)
    rs = [T.sampling_seed(1, 0, s, 0) for s in range(K)]
    losses = tr.steps_v(seeds, off, rs, gamma, 0)
    return losses, tr.get_weights(), tr.step_stats(K)


@pytest.fixture(scope="module")
def c1w():
    """Long rows (300-d: the TMA bulk-copy gather) for the store tiers."""
    return G.generate_power_law(60_000, 3, 2.5, 300, 1)


@pytest.mark.parametrize("feat_dtype,wide", [(0, False), (1, False), (0, True)])
def test_store_policies_bit_identical(c1, c1w, feat_dtype, wide):
    g = c1w if wide else c1
    spec = T.ModelSpec(g.feat_dim, 16, 4)
    cache2 = CA.build_static_cache(g, CA.CacheConfig(int(0.1 * g.num_nodes) * g.feat_dim * 4, 2))
    base = T.Trainer(g, cache2, spec, [10, 5], max_seeds=512, feat_dtype=feat_dtype)
    ref_l, (rw1, rw2), ref_st = _steps(base, g)
    for pol in (G.STORE_HBM, G.STORE_CACHE):
        tr = T.Trainer(g, cache2, spec, [10, 5], max_seeds=512, feat_dtype=feat_dtype,
                       placement=dict(policy=pol))
        info = tr.store.info()
        if pol == G.STORE_CACHE:
            assert info["local_rows"] == cache2.total_cached() and info["host_rows"] == g.num_nodes - info[
                "local_rows"]
        l, (w1, w2), st = _steps(tr, g)
        assert np.array_equal(l, ref_l) and np.array_equal(w1, rw1) and np.array_equal(w2, rw2), pol
        assert np.array_equal(st, ref_st)
    # sharded over 2 "ranks" on one GPU: rank 1's shard is another store's
    # buffer, reached through the peer-pointer path of the gather
    tr = T.Trainer(g, cache2, spec, [10, 5], max_seeds=512, feat_dtype=feat_dtype,
                   placement=dict(policy=G.STORE_SHARDED, rank=0, nranks=2))
    dg1 = G.DeviceGraph(g, 0, feat_dtype, upload_features=False)
    s1 = G.Store(dg1, g.features, cache2.device_map, G.STORE_SHARDED, 1, 2)
    tr.store.set_peer(1, s1.local_ptr())
    info = tr.store.info()
    assert info["local_rows"] + info["remote_rows"] == cache2.total_cached()
    l, (w1, w2), st = _steps(tr, g)
    assert np.array_equal(l, ref_l) and np.array_equal(w1, rw1) and np.array_equal(w2, rw2)


def test_step_stats_match_oracle_batches(orc, c1):
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    tr = T.Trainer(g, cache, T.ModelSpec(g.feat_dim, 16, 4), [10, 5], max_seeds=512)
    batches = T.plan_epoch_batches(g.train_nodes, 0, 512, 77)[:3]
    _, _, st = _steps(tr, g, K=3)
    for i, seeds in enumerate(batches):
        b = orc.sample_khop(g, seeds, [10, 5], 8.0, 0, T.sampling_seed(1, 0, i, 0), cache.device_map)
        hits = int((cache.device_map[b.unique_nodes] != -1).sum())
        assert st[i, T.STAT_UNIQUE] == len(b.unique_nodes)
        assert st[i, T.STAT_EDGES] == b.total_edges()
        assert st[i, T.STAT_SEEDS] == b.num_seed_unique
        assert st[i, T.STAT_HITS] == hits and st[i, T.STAT_MISSES] == len(b.unique_nodes) - hits
        assert st[i, T.STAT_POSITIONS] == b.keys_scanned  # one draw per neighbour of every frontier row


def test_retrieve_features_through_store(c1):
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    dg = G.DeviceGraph(g, 0, 0, upload_features=False)
    st = G.Store(dg, g.features, cache.device_map, G.STORE_CACHE)
    ids = np.random.default_rng(3).choice(g.num_nodes, 5000, replace=False).astype(np.uint32)
    import ctypes as C
    from paper_2511_07421_b200._lib import check, f32p, i32p, lib, ptr, u32p, vp
    hc = vp()
    dm = np.ascontiguousarray(cache.device_map, np.int32)
    check(lib().a3g_cache_from_map(dg.h, ptr(dm, i32p), 1, C.byref(hc)))
    out = np.empty((len(ids), g.feat_dim), np.float32)
    h, m = C.c_uint64(), C.c_uint64()
    check(lib().a3g_gather_rows(dg.h, hc, ptr(ids, u32p), len(ids), ptr(out, f32p), C.byref(h), C.byref(m)))
    lib().a3g_cache_destroy(hc)
    assert np.array_equal(out, g.features[ids])
    assert h.value == int((cache.device_map[ids] != -1).sum()) and h.value + m.value == len(ids)
    del st


def _eval_numpy(g, w1, w2, F, H, Cc):
    """fp64 restatement of evaluate_full_graph (trainer.cpp:241-303)."""
    import scipy.sparse as sp
    n = g.num_nodes
    deg = np.diff(g.row_offsets).astype(np.float64)
    A = sp.csr_matrix((np.ones(g.num_edges), g.col_indices.astype(np.int64), g.row_offsets.astype(np.int64)),
                      shape=(n, n))
    X = g.features.astype(np.float64)

    def agg(T_):
        s = A @ T_
        out = s / np.maximum(deg, 1)[:, None]
        out[deg == 0] = T_[deg == 0]
        return out

    h1 = np.maximum(agg(X) @ w1.reshape(F, H), 0)
    logits = agg(h1) @ w2.reshape(H, Cc)
    pred = logits.argmax(1)
    m = g.test_mask.astype(bool)
    return float((pred[m] == g.labels[m]).mean())


@pytest.mark.parametrize("H", [16, 8])
def test_evaluate_full_graph_vs_numpy(c1, H):
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    spec = T.ModelSpec(g.feat_dim, H, 4)
    tr = T.Trainer(g, cache, spec, [10, 5], max_seeds=256)
    rng = np.random.default_rng(H)
    w1 = rng.normal(0, 0.2, g.feat_dim * H)
    w2 = rng.normal(0, 0.5, H * 4)
    tr.set_weights(w1, w2)
    acc = tr.evaluate_full_graph()
    ref = _eval_numpy(g, w1.astype(np.float32).astype(np.float64), w2.astype(np.float32).astype(np.float64),
                      g.feat_dim, H, 4)
    ntest = int(g.test_mask.sum())
    assert abs(acc - ref) <= 3.0 / ntest, (acc, ref)


def test_evaluate_full_graph_hub_split():
    """A star whose centre has deg > 8192 exercises the split-row reduction."""
    n = 20000
    edges = [(0, v) for v in range(1, n)] + [(v, 0) for v in range(1, n)]
    g = G.from_edges(n, edges, 4)
    rng = np.random.default_rng(0)
    g.features[:] = rng.normal(size=(n, 4)).astype(np.float32)
    g.labels[:] = rng.integers(0, 3, n).astype(np.uint32)
    g.test_mask[:] = 1
    c = CA.CacheState(np.full(n, -1, np.int32), 1)
    tr = T.Trainer(g, c, T.ModelSpec(4, 8, 3), [5], max_seeds=4)
    w1 = rng.normal(size=32)
    w2 = rng.normal(size=24)
    tr.set_weights(w1, w2)
    ref = _eval_numpy(g, w1.astype(np.float32).astype(np.float64), w2.astype(np.float32).astype(np.float64), 4, 8,
                      3)
    assert abs(tr.evaluate_full_graph() - ref) <= 3.0 / n


@pytest.mark.parametrize("name", ["pl500", "pl3000"])
def test_train_report_vs_reference(name):
    """train() on the device vs the reference's train() (golden: 2 epochs,
    B=64, [10,5], gamma 8, H=8, C=4, lr 0.2, rng seed 5, model seed 1)."""
    rec = load_golden(name)
    g = golden_graph(rec)
    c = CA.CacheState(rec["train_device_map"], 1)
    rep = T.train(g, T.ModelSpec(g.feat_dim, 8, 4, learning_rate=0.2), S.SamplerConfig([10, 5], 8.0, 5), c,
                  T.TrainOptions(batch_size=64, epochs=2, model_seed=1))
    assert rel_err(rep.loss_curve, rec["train_curve"]) < 1e-3
    np.testing.assert_array_equal(rep.epoch_hit_rates, rec["train_hit_rates"])
    ntest = int(rec["test_mask"].sum())
    assert abs(rep.test_accuracy - rec["train_accuracy"][0]) <= 2.0 / ntest
    assert rep.epochs_run == 2 and rep.param_bytes == (g.feat_dim * 8 + 8 * 4) * 4


def test_train_rejects_partitioned_workers():
    rec = load_golden("pl500")
    g = golden_graph(rec)
    c = CA.CacheState(rec["train_device_map"], 1)
    with pytest.raises(T.ConfigError):
        T.train(g, T.ModelSpec(g.feat_dim, 8, 4), S.SamplerConfig([10, 5], 8.0, 5), c, T.TrainOptions(u=2))


def test_nccl_gradient_sync_world1(c1):
    """The DP exchange on the device (k_scale_for_sync -> ncclAllReduce ->
    k_sgd dividing by sum n_k) on a 1-rank communicator equals the local step."""
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    spec = T.ModelSpec(g.feat_dim, 16, 4)
    a = T.Trainer(g, cache, spec, [10, 5], max_seeds=512)
    la, (a1, a2), _ = _steps(a, g, K=3)
    b = T.Trainer(g, cache, spec, [10, 5], max_seeds=512)
    comm = T.Comm(T.Comm.unique_id(), 1, 0, 0)
    b.set_comm(comm)
    lb, (b1, b2), _ = _steps(b, g, K=3)
    np.testing.assert_allclose(lb, la, rtol=1e-6)
    assert rel_err(b1, a1) < 1e-6 and rel_err(b2, a2) < 1e-6
    b.set_comm(None)
    del comm


@pytest.mark.parametrize("feat_dtype", [0, 1])
def test_device_feature_synthesis_matches_generator(feat_dtype):
    """Papers-scale inputs: features synthesized on the device from the
    generator's streams (generators.cpp:12-24) are BIT-IDENTICAL to the host
    generator's (bf16: after the same RNE rounding). Elements whose fp64 value
    sits near a float rounding boundary are recomputed with glibc (synth.cu);
    200K x 64 elements list a few dozen of them."""
    import ctypes as C
    from paper_2511_07421_b200._lib import check, f32p, lib, ptr, u32p, vp
    n, F = 200_000, 64
    full = G.generate_power_law(n, 3, 2.5, F, 7)
    topo = G.generate_power_law(n, 3, 2.5, 1, 7)
    assert np.array_equal(full.col_indices, topo.col_indices) and np.array_equal(full.labels, topo.labels)
    dg = G.DeviceGraph(topo, 0, feat_dtype, upload_features=False)
    check(lib().a3g_graph_synthesize_features(dg.h, F, feat_dtype, 7))
    patched = lib().a3g_graph_synth_patched(dg.h)
    assert 0 < patched < 1e-4 * n * F, patched
    hc = vp()
    check(lib().a3g_cache_from_map(dg.h, None, 1, C.byref(hc)))
    ids = np.arange(n, dtype=np.uint32)
    out = np.empty((n, F), np.float32)
    h, m = C.c_uint64(), C.c_uint64()
    check(lib().a3g_gather_rows(dg.h, hc, ptr(ids, u32p), n, ptr(out, f32p), C.byref(h), C.byref(m)))
    lib().a3g_cache_destroy(hc)
    want = full.features
    if feat_dtype == 1:
        u = want.view(np.uint32).astype(np.uint64)
        want = (((u + 0x7fff + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32).view(np.float32)
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32)), int((out != want).sum())


def test_pipeline_shapes_bit_identical(c1):
    """Sequential mode and 1..12 concurrent sampling streams only change the
    schedule (pipeline.hpp:107-109): losses, weights and per-step statistics
    are bit-identical for every shape, over more steps than arenas."""
    g = c1
    spec = T.ModelSpec(g.feat_dim, 16, 4)
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    ref = None
    for n in (0, 1, 2, 4, 8, 12):
        tr = T.Trainer(g, cache, spec, [10, 5], max_seeds=512)
        tr.set_pipeline(n)
        got = _steps(tr, g, K=15)
        if ref is None:
            ref = got
        else:
            assert np.array_equal(got[0], ref[0]), n
            assert all(np.array_equal(a, b) for a, b in zip(got[1], ref[1])), n
            assert np.array_equal(got[2], ref[2]), n
    with pytest.raises(Exception):
        tr.set_pipeline(13)


def test_device_resident_seeds_are_validated(c1):
    """Seeds already in HBM (a3g_train_steps(..., seeds_on_device=1)): an
    out-of-range seed is clamped on the device and raises ParameterError at
    the call's sync (sampler.cpp:92-94); gamma < 1 raises before any launch
    (assign_weights, sampler.cpp:62); valid device seeds train as host seeds."""
    import ctypes as C
    import torch
    from paper_2511_07421_b200._lib import ParameterError, check, f64p, lib, ptr, u64p
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    tr = T.Trainer(g, cache, T.ModelSpec(g.feat_dim, 16, 4), [10, 5], max_seeds=256)
    rs = np.array([T.sampling_seed(1, 0, s, 0) for s in range(2)], dtype=np.uint64)
    losses = np.empty(2)

    def run(seeds, gamma=8.0):
        d = torch.from_numpy(np.ascontiguousarray(seeds, dtype=np.int32)).cuda()
        check(lib().a3g_train_steps(tr.h, C.cast(C.c_void_p(d.data_ptr()), C.POINTER(C.c_uint32)), seeds.shape[1],
                                    2, ptr(rs, u64p), gamma, 0, 1, ptr(losses, f64p)))
        return losses.copy()

    good = np.stack(T.plan_epoch_batches(g.train_nodes, 0, 256, 9)[:2])
    ref = T.Trainer(g, cache, T.ModelSpec(g.feat_dim, 16, 4), [10, 5], max_seeds=256).steps(good, rs, 8.0, 0)
    np.testing.assert_array_equal(run(good), ref)
    bad = good.copy()
    bad[1, 7] = g.num_nodes + 5
    with pytest.raises(ParameterError, match="seed out of range"):
        run(bad)
    with pytest.raises(ParameterError, match="gamma"):
        run(good, gamma=0.5)
