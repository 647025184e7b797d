"""The oracle (C restatement, oracle/a3g_oracle.c) pinned against golden vectors
produced by the compiled reference (tests/golden/make_golden.py), and against
the reference library directly where oracle/_ref exists."""
import numpy as np
import pytest

import oracle
from helpers import assert_same_batch, golden_cfgs, load_golden

GRAPHS = ["pl500", "pl3000"]


class G:  # minimal graph view over a golden record
    def __init__(self, rec):
        self.row_offsets = rec["row_offsets"]
        self.col_indices = rec["col_indices"]
        self.features = rec["features"]
        self.labels = rec["labels"]
        self.train_mask = rec["train_mask"]
        self.test_mask = rec["test_mask"]
        self.num_nodes = len(self.labels)
        self.num_edges = len(self.col_indices)
        self.feat_dim = self.features.shape[1]


@pytest.fixture(scope="module")
def orc():
    return oracle.Oracle()


@pytest.mark.parametrize("name", GRAPHS)
def test_sampler_golden(orc, name):
    rec = load_golden(name)
    g = G(rec)
    n = 0
    for i, c in enumerate(golden_cfgs(rec)):
        b = orc.sample_khop(g, c["seeds"], c["fanouts"], c["gamma"], c["kind"], c["rng_seed"], c["device_map"])
        assert_same_batch(b, c, f"{name} cfg{i}")
        n += 1
    assert n == 8


@pytest.mark.parametrize("name", GRAPHS)
def test_cache_golden(orc, name):
    rec = load_golden(name)
    g = G(rec)
    for nd in (1, 2, 4):
        dm = orc.build_static_cache(g, (g.num_nodes // 10) * g.feat_dim * 4, nd)
        assert np.array_equal(dm, rec[f"cache{nd}"])


@pytest.mark.parametrize("name", GRAPHS)
def test_trainer_golden(orc, name):
    rec = load_golden(name)
    g = G(rec)
    w1, w2 = orc.init_model(g.feat_dim, 8, 4, 1)
    assert np.array_equal(w1, rec["init_w1"]) and np.array_equal(w2, rec["init_w2"])
    out = orc.train_steps(g, [10, 5], 8.0, 0, 5, 64, 8, 4, 0.2, w1, w2, 6, rec["train_device_map"])
    # scalar-kernel order: bit-exact
    assert np.array_equal(out["losses"], rec["train_losses"])
    assert np.array_equal(out["w1"], rec["train_w1"]) and np.array_equal(out["w2"], rec["train_w2"])
    # the reference's own train() loop: epoch mean losses
    spe = (int(g.train_mask.sum()) + 63) // 64
    full = orc.train_steps(g, [10, 5], 8.0, 0, 5, 64, 8, 4, 0.2, w1, w2, 2 * spe, rec["train_device_map"])
    curve = [full["losses"][e * spe:(e + 1) * spe].sum() / spe for e in range(2)]
    np.testing.assert_allclose(curve, rec["train_curve"], rtol=1e-12)


@pytest.mark.parametrize("name", GRAPHS)
def test_plan_and_seeds_golden(orc, name):
    rec = load_golden(name)
    tn = np.flatnonzero(rec["train_mask"]).astype(np.uint32)
    assert np.array_equal(orc.plan_epoch_order(tn, 3, 99), rec["plan_e3"])
    got = [orc.sampling_seed(1, e, s, 0) for e in range(3) for s in range(4)]
    assert np.array_equal(np.array(got, dtype=np.uint64), rec["sampling_seeds"])


def test_forward_kat(orc):
    """test_trainer.cpp:71-87: logits 2.75 / 16.5 on the path fixture."""
    kat = load_golden("kat_path")
    out = orc.grad_on_edges(2, 2, 2, np.array([1.0, 0.5, -0.25, 1.0]), np.array([2.0, -1.0, 0.5, 3.0]), 3, 1,
                            [(np.array([0]), np.array([1])), (np.array([1]), np.array([2]))],
                            np.array([1, 2, 3, 4, -1, 6], np.float32), [0])
    np.testing.assert_allclose(out["logits"].ravel(), [2.75, 16.5], rtol=1e-12)
    assert np.array_equal(out["logits"].ravel(), kat["logits"].ravel())
    assert np.array_equal(out["gw1"], kat["gw1"]) and np.array_equal(out["gw2"], kat["gw2"])


def test_reservoir_semantics(orc):
    """test_sampler.cpp:57-88: keep-all, bad inputs, one draw per neighbour."""
    key = orc.hash2(1, 0)
    r, ctr = orc.weighted_reservoir([10, 20, 30], [1.0, 5.0, 0.2], 3, key)
    assert sorted(r.tolist()) == [10, 20, 30] and ctr == 3
    r, ctr = orc.weighted_reservoir([1, 2, 3, 4, 5, 6, 7], [1.0] * 7, 3, key)
    assert ctr == 7 and len(r) == 3
    with pytest.raises(oracle.SamplerError):
        orc.weighted_reservoir([1, 2], [1.0, 0.0], 1, key)
    with pytest.raises(oracle.SamplerError):
        orc.weighted_reservoir([1, 2], [1.0, 1.0], 0, key)
    r, ctr = orc.weighted_reservoir([], [], 3, key)
    assert len(r) == 0


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_oracle_vs_reference_random():
    """Direct pin against the compiled reference on fresh random inputs."""
    orc, ref = oracle.Oracle(), oracle.RefLib()
    g = ref.power_law(4000, 2, 2.5, 8, 42)
    rng = np.random.default_rng(0)
    for t in range(12):
        fan = [int(x) for x in rng.integers(1, 20, size=rng.integers(1, 4))]
        gamma = float(rng.choice([1.0, 2.0, 8.0, 32.0, 1.5]))
        kind = int(rng.integers(0, 2))
        dm = ref.build_static_cache(g, int(rng.integers(0, 4000)) * 32, int(rng.integers(1, 4)))
        seeds = rng.integers(0, 4000, size=int(rng.integers(1, 300))).astype(np.uint32)
        rs = int(rng.integers(0, 2**63))
        a = orc.sample_khop(g, seeds, fan, gamma, kind, rs, dm)
        b = ref.sample_khop(g, seeds, fan, gamma, kind, rs, dm)
        assert_same_batch(a, b, f"trial {t}")
    for t in range(20):  # explicit-weight reservoirs incl. arbitrary weights
        n = int(rng.integers(0, 200))
        nb = rng.integers(0, 10**6, size=n).astype(np.uint32)
        w = rng.choice([1.0, 9.0, 0.2, 4.0], size=n)
        m = int(rng.integers(1, 40))
        seed, stream = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**63))
        key = orc.hash2(seed, stream)
        assert np.array_equal(orc.weighted_reservoir(nb, w, m, key)[0], ref.weighted_reservoir(nb, w, m, seed, stream))
        assert np.array_equal(orc.uniform_reservoir(nb, m, key)[0], ref.uniform_reservoir(nb, m, seed, stream))


@pytest.mark.parametrize("name,seed", [("pl500", 3), ("pl3000", 1)])
def test_feature_rows_golden(orc, name, seed):
    """orc_feature_rows (generators.cpp:12-24 for an explicit node list, the
    papers-scale row checker) reproduces the reference generator's feature
    table bit for bit, in any node order."""
    rec = load_golden(name)
    n, F = rec["features"].shape
    ids = np.random.default_rng(0).permutation(n).astype(np.uint32)
    rows = orc.feature_rows(seed, F, ids, rec["labels"])
    assert np.array_equal(rows.view(np.uint32), rec["features"][ids].view(np.uint32))
