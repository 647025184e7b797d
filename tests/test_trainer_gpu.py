"""Device 2-layer mean-GCN step vs the fp64 oracle. Tolerance (fp32 device vs
fp64 reference): norm-wise relative error <= 1e-3 for loss, logits, gradients
and intermediates (BASELINE.json north_star). bf16 feature mode has the same
stated tolerance, 1e-3, against the fp64 oracle fed the same bf16-rounded
features (the rows are exact; only the fp32 accumulation differs)."""
import numpy as np
import pytest

import oracle
from helpers import golden_graph, load_golden, rel_err
from paper_2511_07421_b200 import cache as CA, graph as G, sampling as S, train as T

pytestmark = pytest.mark.gpu
TOL = 1e-3


@pytest.fixture(scope="module")
def orc():
    return oracle.Oracle()


def test_forward_kat_path_fixture():
    """test_trainer.cpp:71-87: path 0 <- 1 <- 2 gives logits 2.75 / 16.5.
    Out-edges 0->1, 1->2 with fanouts >= degree sample exactly that batch."""
    g = G.from_edges(3, [(0, 1), (1, 2)], 2)
    g.features[:] = np.array([[1, 2], [3, 4], [-1, 6]], np.float32)
    c = CA.CacheState(np.full(3, -1, np.int32), 1)
    tr = T.Trainer(g, c, T.ModelSpec(2, 2, 2), [5, 5], max_seeds=4)
    tr.set_weights([1.0, 0.5, -0.25, 1.0], [2.0, -1.0, 0.5, 3.0])
    kat = load_golden("kat_path")
    loss, (gw1, gw2) = tr.grad_on_batch([0], 1.0, 0, 7)
    fwd = tr.last_forward(8)
    np.testing.assert_allclose(fwd["logits"][:2], [2.75, 16.5], rtol=1e-6)
    assert abs(loss - kat["loss"][0]) <= 1e-5 * max(1.0, abs(kat["loss"][0]))
    assert rel_err(gw1, kat["gw1"]) < TOL and rel_err(gw2, kat["gw2"]) < TOL


def test_isolated_seed_fallback():
    """test_trainer.cpp:89-108: self-fallback, zero features -> zero logits."""
    g = G.from_edges(2, [(1, 0)], 2)
    g.features[:] = 0.0
    c = CA.CacheState(np.full(2, -1, np.int32), 1)
    tr = T.Trainer(g, c, T.ModelSpec(2, 3, 2), [4, 4], max_seeds=2)
    tr.step([0], lr=0.0)
    assert np.all(tr.last_forward(4)["logits"][:2] == 0.0)


def _grad_case(orc, g, cache, seeds, fanouts, gamma, kind, rs, H=16, Cc=4, feat_dtype=0, tol=TOL):
    tr = T.Trainer(g, cache, T.ModelSpec(g.feat_dim, H, Cc), fanouts, max_seeds=len(seeds), feat_dtype=feat_dtype)
    w1, w2 = T.init_model(T.ModelSpec(g.feat_dim, H, Cc), 1)
    loss, (gw1, gw2) = tr.grad_on_batch(seeds, gamma, kind, rs)
    fwd = tr.last_forward(int(len(seeds) * (1 + fanouts[0])))
    b = orc.sample_khop(g, seeds, fanouts, gamma, kind, rs, cache.device_map)
    feats = g.features[b.unique_nodes]
    if feat_dtype == 1:  # oracle consumes the same bf16-rounded features
        u = feats.view(np.uint32).astype(np.uint64)
        feats = (((u + 0x7fff + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32).view(np.float32)
    ref = orc.grad_on_edges(g.feat_dim, H, Cc, w1, w2, len(b.unique_nodes), b.num_seed_unique, b.layers, feats,
                            g.labels[b.unique_nodes[:b.num_seed_unique]])
    ns = b.num_seed_unique
    assert abs(loss - ref["loss"]) <= tol * abs(ref["loss"])
    assert rel_err(fwd["logits"][:ns * Cc], ref["logits"]) < tol
    assert rel_err(gw1, ref["gw1"]) < tol, rel_err(gw1, ref["gw1"])
    assert rel_err(gw2, ref["gw2"]) < tol, rel_err(gw2, ref["gw2"])
    return tr


@pytest.mark.parametrize("name", ["pl500", "pl3000"])
def test_grads_golden_graphs(orc, name):
    rec = load_golden(name)
    g = golden_graph(rec)
    c = CA.CacheState(rec["train_device_map"], 1)
    seeds = np.flatnonzero(rec["train_mask"])[:64].astype(np.uint32)
    _grad_case(orc, g, c, seeds, [10, 5], 8.0, 0, 5, H=8)


@pytest.fixture(scope="module")
def c1():
    return G.generate_power_law(100_000, 3, 2.5, 128, 1)


@pytest.mark.parametrize("fanouts,gamma,kind,H", [([10, 5], 1.0, 0, 16), ([10, 5], 8.0, 0, 16),
                                                  ([10, 5], 1.0, 1, 16), ([15, 10, 5], 4.0, 0, 32),
                                                  ([10], 8.0, 0, 16), ([10, 5], 8.0, 0, 5)])
def test_grads_c1_vs_oracle(orc, c1, fanouts, gamma, kind, H):
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    batches = T.plan_epoch_batches(g.train_nodes, 0, 1024, orc.hash2(1, 0))
    _grad_case(orc, g, cache, batches[3], fanouts, gamma, kind, T.sampling_seed(1, 0, 3, 0), H=H)


def test_wide_feature_rows(orc):
    """Rows wider than k_agg1's 24-warp ring (F = 1500 f32, 6 KB) stream
    through the 8-warp configuration instead of being refused."""
    g = G.generate_power_law(20_000, 3, 2.5, 1500, 3)
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    seeds = np.arange(0, 12_000, 23, dtype=np.uint32)
    _grad_case(orc, g, cache, seeds, [10, 5], 8.0, 0, 17, H=16)
    _grad_case(orc, g, cache, seeds, [10, 5], 8.0, 0, 17, H=64)


@pytest.mark.parametrize("F,feat_dtype,H", [(300, 0, 16), (602, 0, 16), (600, 1, 16), (300, 0, 64)])
def test_long_rows_tma_gather(orc, F, feat_dtype, H):
    """Rows of more than 32 16-byte chunks take k_agg1_tma (one TMA bulk copy
    per source row, per-slot mbarriers; H <= 16 with the fused h1 epilogue,
    H = 64 without): loss and gradients within the same 1e-3 of the oracle,
    f32 and bf16 rows."""
    g = G.generate_power_law(40_000, 4, 2.5, F, 5)
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    batches = T.plan_epoch_batches(g.train_nodes, 0, 1024, orc.hash2(1, 0))
    _grad_case(orc, g, cache, batches[1], [15, 10], 8.0, 0, T.sampling_seed(1, 0, 1, 0), H=H,
               feat_dtype=feat_dtype)


def test_long_rows_tma_matches_ldgsts_bitwise():
    """The TMA gather sums the same rows in the same order as the per-lane
    LDGSTS kernel (A3G_AGG_TMA=0): losses and weights after 4 steps are
    bit-identical (separate processes: the switch is read once)."""
    import json
    import os
    import subprocess
    import sys
    code = (
        "import json, numpy as np\n"
        "from paper_2511_07421_b200 import cache as CA, graph as G, train as T\n"
        "g = G.generate_power_law(40_000, 4, 2.5, 602, 5)\n"
        "c = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))\n"
        "tr = T.Trainer(g, c, T.ModelSpec(602, 16, 4), [15, 10, 5], max_seeds=1024)\n"
        "b = T.plan_epoch_batches(g.train_nodes, 0, 1024, 77)[:4]\n"
        "off = np.cumsum([0] + [len(x) for x in b]).astype(np.uint64)\n"
        "l = tr.steps_v(np.concatenate(b), off, [T.sampling_seed(1, 0, s, 0) for s in range(4)], 8.0, 0)\n"
        "w1, w2 = tr.get_weights()\n"
        "print(json.dumps([np.asarray(l).tobytes().hex(), np.asarray(w1).tobytes().hex(), np.asarray(w2).tobytes().hex()]))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                           env=dict(os.environ, A3G_AGG_TMA=v))
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]


@pytest.mark.parametrize("H", [48, 64, 128, 256])
def test_wide_hidden_on_tcgen05(orc, c1, H):
    """Realistic hidden widths (e.g. 256): h1 and dW1 run
    on tcgen05 with N = H (64 / 128 / 256 TMEM columns), k_outer strides the
    hidden units over the warp; loss and gradients within the same 1e-3."""
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    batches = T.plan_epoch_batches(g.train_nodes, 0, 1024, orc.hash2(1, 0))
    _grad_case(orc, g, cache, batches[4], [10, 5], 8.0, 0, T.sampling_seed(1, 0, 4, 0), H=H)


def test_tcgen05_gemm_path(orc, c1, monkeypatch):
    """A3G_TC_GEMMS=1: h1 and dW1 from the tcgen05 GEMMs instead of k_agg1's
    epilogue and the CUDA-core dW1 -- the same oracle tolerance (both paths
    are fp32-class)."""
    monkeypatch.setenv("A3G_TC_GEMMS", "1")
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    batches = T.plan_epoch_batches(g.train_nodes, 0, 1024, orc.hash2(1, 0))
    _grad_case(orc, g, cache, batches[2], [10, 5], 8.0, 0, T.sampling_seed(1, 0, 2, 0), H=16)


def test_intermediates_c1(orc, c1):
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    seeds = np.arange(0, 60_000, 61, dtype=np.uint32)
    tr = _grad_case(orc, g, cache, seeds, [10, 5], 8.0, 0, 9)
    fwd = tr.last_forward(len(seeds) * 11)
    b = orc.sample_khop(g, seeds, [10, 5], 8.0, 0, 9, cache.device_map)
    w1, w2 = T.init_model(T.ModelSpec(128, 16, 4), 1)
    U = len(b.unique_nodes)
    ref = orc.L  # intermediates via orc_grad_on_batch
    import ctypes as C
    F, H = 128, 16
    ni = C.c_uint64()
    agg_inner = np.empty(U * F)
    h1 = np.empty(U * H)
    agg_outer = np.empty(b.num_seed_unique * H)
    logits = np.empty(b.num_seed_unique * 4)
    gw1, gw2 = np.empty(F * H), np.empty(H * 4)
    # rebuild the oracle batch handle to get intermediates
    err = C.c_int()
    s = np.ascontiguousarray(seeds)
    f = np.array([10, 5], np.uint32)
    h = ref.orc_sample_khop(g.num_nodes, g.row_offsets.ctypes.data_as(oracle.u64p),
                            g.col_indices.ctypes.data_as(oracle.u32p), s.ctypes.data_as(oracle.u32p), len(s),
                            f.ctypes.data_as(oracle.u32p), 2, 8.0, 0, 9,
                            cache.device_map.ctypes.data_as(oracle.i32p), C.byref(err))
    feats = np.ascontiguousarray(g.features[b.unique_nodes])
    ref.orc_grad_on_batch(F, H, 4, w1.ctypes.data_as(oracle.f64p), w2.ctypes.data_as(oracle.f64p), h,
                          feats.ctypes.data_as(oracle.f32p), g.labels.ctypes.data_as(oracle.u32p),
                          gw1.ctypes.data_as(oracle.f64p), gw2.ctypes.data_as(oracle.f64p), C.byref(ni),
                          logits.ctypes.data_as(oracle.f64p), agg_inner.ctypes.data_as(oracle.f64p),
                          h1.ctypes.data_as(oracle.f64p), agg_outer.ctypes.data_as(oracle.f64p))
    ref.orc_batch_free(h)
    n = ni.value
    assert fwd["n_inner"] == n
    assert rel_err(fwd["agg_inner"], agg_inner[:n * F]) < 1e-5
    assert rel_err(fwd["h1"], h1[:n * H]) < TOL
    assert rel_err(fwd["agg_outer"][:b.num_seed_unique * H], agg_outer) < TOL


def test_bf16_features(orc, c1):
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    seeds = np.arange(0, 60_000, 59, dtype=np.uint32)
    _grad_case(orc, g, cache, seeds, [10, 5], 8.0, 0, 21, feat_dtype=1, tol=TOL)


@pytest.mark.parametrize("name", ["pl3000"])
def test_multi_step_training_vs_golden(name):
    """6 SGD steps of train() (u=1) vs the reference's own trajectory."""
    rec = load_golden(name)
    g = golden_graph(rec)
    c = CA.CacheState(rec["train_device_map"], 1)
    F = g.feat_dim
    tr = T.Trainer(g, c, T.ModelSpec(F, 8, 4, learning_rate=0.2), [10, 5], max_seeds=64)
    tr.set_weights(rec["init_w1"], rec["init_w2"])
    batches = T.plan_epoch_batches(g.train_nodes, 0, 64, oracle.Oracle().hash2(5, 0))
    losses = [tr.step(batches[s], 8.0, 0, T.sampling_seed(5, 0, s, 0)) for s in range(6)]
    np.testing.assert_allclose(losses, rec["train_losses"], rtol=TOL)
    w1, w2 = tr.get_weights()
    assert rel_err(w1, rec["train_w1"]) < TOL and rel_err(w2, rec["train_w2"]) < TOL


def test_pipelined_steps_match_sequential(c1):
    """The stream pipeline is a schedule, not an algorithm change
    (pipeline.hpp:107-109): same losses and weights as one-at-a-time steps."""
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    batches = T.plan_epoch_batches(g.train_nodes, 0, 1024, 77)[:8]
    rs = [T.sampling_seed(1, 0, s, 0) for s in range(8)]
    a = T.Trainer(g, cache, T.ModelSpec(128, 16, 4), [10, 5], 1024)
    la = [a.step(batches[s], 8.0, 0, rs[s]) for s in range(8)]
    b = T.Trainer(g, cache, T.ModelSpec(128, 16, 4), [10, 5], 1024)
    lb = b.steps(np.stack(batches), rs, 8.0, 0)
    np.testing.assert_allclose(lb, la, rtol=1e-5)
    assert rel_err(b.get_weights()[0], a.get_weights()[0]) < 1e-5


def test_data_parallel_shard_equivalence(c1):
    """SURVEY 8(e) / test_trainer.cpp:210-253: the n_k-weighted sum of shard
    gradients (same step seed) equals the full-batch gradient."""
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    seeds = T.plan_epoch_batches(g.train_nodes, 0, 1024, 5)[0]
    tr = T.Trainer(g, cache, T.ModelSpec(128, 16, 4), [10, 5], 1024)
    lf, (f1, f2) = tr.grad_on_batch(seeds, 8.0, 0, 1234)
    for k in (2, 4, 8):
        acc1, acc2, lsum = 0.0, 0.0, 0.0
        for sh in np.array_split(seeds, k):
            l, (a1, a2) = tr.grad_on_batch(sh, 8.0, 0, 1234)
            acc1 = acc1 + len(sh) * a1
            acc2 = acc2 + len(sh) * a2
            lsum += len(sh) * l
        assert rel_err(acc1 / len(seeds), f1) < 1e-4 and rel_err(acc2 / len(seeds), f2) < 1e-4
        assert abs(lsum / len(seeds) - lf) < 1e-5 * abs(lf)


def test_sgd_lr_zero_keeps_weights(c1):
    """test_trainer.cpp:175-188."""
    g = c1
    cache = CA.CacheState(np.full(g.num_nodes, -1, np.int32), 1)
    tr = T.Trainer(g, cache, T.ModelSpec(128, 16, 4), [10, 5], 256)
    w = tr.get_weights()
    tr.step(np.arange(256), lr=0.0)
    w2 = tr.get_weights()
    assert np.array_equal(w[0], w2[0]) and np.array_equal(w[1], w2[1])


def test_explicit_batch_model_api(orc, c1):
    """trainer.cpp:59-239 on the caller's own batch (the drop-in's forward /
    backward / grad_on_batch path, a3g_batch_model_*): the oracle's batch and
    rows in, ForwardResult index arrays identical to the oracle's, values and
    gradients within 1e-3; sgd_step / sync_gradients on the device are
    bit-identical to the reference's scalar arithmetic."""
    g = c1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * g.num_nodes) * g.feat_dim * 4, 1))
    seeds = np.arange(0, 60_000, 71, dtype=np.uint32)
    b = orc.sample_khop(g, seeds, [10, 5], 8.0, 0, 31, cache.device_map)
    feats = np.ascontiguousarray(g.features[b.unique_nodes])
    spec = T.ModelSpec(128, 16, 4)
    w1, w2 = T.init_model(spec, 1)
    labels = g.labels[b.unique_nodes[:b.num_seed_unique]]
    ref = orc.grad_on_edges(128, 16, 4, w1, w2, len(b.unique_nodes), b.num_seed_unique, b.layers, feats, labels)
    fwd = T.forward((w1, w2), b, feats, spec)
    # inner nodes: unique seeds, then first-seen layer-0 sources (trainer.cpp:76-89)
    want_inner = list(range(b.num_seed_unique))
    seen = set(want_inner)
    for s_ in b.layers[0][1]:
        if int(s_) not in seen:
            seen.add(int(s_))
            want_inner.append(int(s_))
    assert np.array_equal(fwd["inner_nodes"], np.array(want_inner, np.uint32))
    assert np.array_equal(fwd["outer_deg"], np.bincount(b.layers[0][0], minlength=b.num_seed_unique)[:b.num_seed_unique])
    assert rel_err(fwd["logits"], ref["logits"]) < TOL
    loss, (g1, g2) = T.backward((w1, w2), b, feats, labels, spec)
    assert abs(loss - ref["loss"]) <= TOL * abs(ref["loss"])
    assert rel_err(g1, ref["gw1"]) < TOL and rel_err(g2, ref["gw2"]) < TOL
    loss2, (h1, h2) = T.grad_on_batch((w1, w2), g, b, feats, spec)
    assert loss2 == loss and np.array_equal(h1, g1)
    # device sync / SGD vs the reference's scalar table: sum in order, x 1/k; w + (-lr) g
    a1, a2 = T.init_model(spec, 11)
    c1_, c2_ = T.init_model(spec, 12)
    m1, m2 = T.sync_gradients([(a1, a2), (c1_, c2_), (a1, a2)])
    assert np.array_equal(m1, ((0.0 + a1) + c1_ + a1) * (1.0 / 3.0)) and np.array_equal(m2, ((0.0 + a2) + c2_ + a2) * (1.0 / 3.0))
    w = w1.copy()
    T.sgd_step(w, m1, 0.2)
    assert np.array_equal(w, w1 + (-0.2) * m1)
    with pytest.raises(Exception):
        T.sync_gradients([])
