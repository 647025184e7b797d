"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes front-ends for
  * ``Oracle``  -- the plain-C restatement of the reference hot path
                   (oracle/a3g_oracle.c -> oracle/_build/liba3g_oracle.so), and
  * ``RefLib``  -- the UNMODIFIED reference library compiled in place
                   (oracle/ref_shim.cpp + /root/reference/proj/src -> oracle/_ref/).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this package; the product path
(paper_2511_07421_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liba3g_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_a3gnn.so")
REF_SRC = "/root/reference/proj"

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)

WEIGHTED, UNIFORM = 0, 1


def build(ref: bool = True) -> None:
    """Compile the C restatement (always) and the reference shim (only where
    /root/reference exists; on the GPU box the prebuilt oracle/_ref travels)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@dataclass
class Batch:
    """Mirror of sampling::SampleBatch (sampler.hpp:30-46) as numpy arrays."""
    seeds: np.ndarray
    unique_nodes: np.ndarray
    num_seed_unique: int
    num_duplicates_removed: int
    layers: list = field(default_factory=list)  # list of (dst_idx u32[E], src_idx u32[E])
    keys_scanned: int = 0

    def total_edges(self) -> int:
        return int(sum(len(d) for d, _ in self.layers))


class SamplerError(Exception):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"sampler error {code}: {msg}")
        self.code = code


# --------------------------------------------------------------------------
class Oracle:
    """The plain-C restatement (a3g_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.L = C.CDLL(path)
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_hash2.restype = C.c_uint64
        L.orc_hash2.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_hash3.restype = C.c_uint64
        L.orc_hash3.argtypes = [C.c_uint64] * 3
        L.orc_sampling_seed.restype = C.c_uint64
        L.orc_sampling_seed.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.orc_plan_epoch_order.argtypes = [u32p, C.c_uint64, C.c_uint32, C.c_uint64, u32p]
        L.orc_weighted_reservoir.restype = C.c_int64
        L.orc_weighted_reservoir.argtypes = [u32p, f64p, C.c_uint64, C.c_uint32, C.c_uint64, u64p, u32p]
        L.orc_uniform_reservoir.restype = C.c_int64
        L.orc_uniform_reservoir.argtypes = [u32p, C.c_uint64, C.c_uint32, C.c_uint64, u64p, u32p]
        L.orc_sample_khop.restype = C.c_void_p
        L.orc_sample_khop.argtypes = [C.c_uint64, u64p, u32p, u32p, C.c_uint64, u32p, C.c_uint32,
                                      C.c_double, C.c_int, C.c_uint64, i32p, C.POINTER(C.c_int)]
        for name, rt in [("orc_batch_num_unique", C.c_uint64), ("orc_batch_num_seed_unique", C.c_uint64),
                         ("orc_batch_dups", C.c_uint64), ("orc_batch_keys_scanned", C.c_uint64),
                         ("orc_batch_unique", u32p)]:
            getattr(L, name).restype = rt
            getattr(L, name).argtypes = [C.c_void_p]
        for name, rt in [("orc_batch_layer_ne", C.c_uint64), ("orc_batch_layer_dst", u32p),
                         ("orc_batch_layer_src", u32p)]:
            getattr(L, name).restype = rt
            getattr(L, name).argtypes = [C.c_void_p, C.c_uint32]
        L.orc_batch_free.argtypes = [C.c_void_p]
        L.orc_build_static_cache.restype = C.c_int64
        L.orc_build_static_cache.argtypes = [C.c_uint64, u64p, C.c_uint32, C.c_uint64, C.c_uint32, i32p]
        L.orc_retrieve_features.restype = C.c_uint64
        L.orc_retrieve_features.argtypes = [f32p, C.c_uint32, i32p, C.c_void_p, f32p, u64p, u64p]
        L.orc_init_model.restype = C.c_int
        L.orc_init_model.argtypes = [C.c_uint32] * 3 + [C.c_uint64, f64p, f64p]
        L.orc_grad_on_batch.restype = C.c_double
        L.orc_grad_on_batch.argtypes = [C.c_uint32] * 3 + [f64p, f64p, C.c_void_p, f32p, u32p, f64p, f64p,
                                                           u64p, f64p, f64p, f64p, f64p]
        L.orc_grad_on_edges.restype = C.c_double
        L.orc_grad_on_edges.argtypes = [C.c_uint32] * 3 + [f64p, f64p, C.c_uint64, C.c_uint64, C.c_uint32,
                                                           u64p, C.POINTER(u32p), C.POINTER(u32p), f32p, u32p,
                                                           f64p, f64p, f64p]
        L.orc_sgd_step.argtypes = [f64p, f64p, C.c_uint64, C.c_double]
        L.orc_feature_rows.argtypes = [C.c_uint64, C.c_uint32, u32p, C.c_uint64, u32p, f32p]
        L.orc_train_steps.restype = C.c_int64
        L.orc_train_steps.argtypes = [C.c_uint64, u64p, u32p, f32p, C.c_uint32, u32p, u8p, i32p, u32p,
                                      C.c_uint32, C.c_double, C.c_int, C.c_uint64, C.c_uint32, C.c_uint32,
                                      C.c_uint32, C.c_double, f64p, f64p, C.c_uint64, f64p, u64p, u64p]

    def feature_rows(self, seed, F, ids, labels) -> np.ndarray:
        """generators.cpp:12-24 rows of the power-law generator (seed, F) for `ids`."""
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        labels = np.ascontiguousarray(labels, dtype=np.uint32)
        out = np.empty((len(ids), F), np.float32)
        self.L.orc_feature_rows(seed, F, _p(ids, u32p), len(ids), _p(labels, u32p), _p(out, f32p))
        return out

    # -- rng ---------------------------------------------------------------
    def mix64(self, z): return self.L.orc_mix64(z)
    def hash2(self, a, b): return self.L.orc_hash2(a, b)
    def hash3(self, a, b, c): return self.L.orc_hash3(a, b, c)
    def sampling_seed(self, base, epoch, step, worker=0):
        return self.L.orc_sampling_seed(base, epoch, step, worker)

    def plan_epoch_order(self, train_nodes: np.ndarray, epoch: int, seed: int) -> np.ndarray:
        t = np.ascontiguousarray(train_nodes, dtype=np.uint32)
        out = np.empty_like(t)
        self.L.orc_plan_epoch_order(_p(t, u32p), len(t), epoch, seed, _p(out, u32p))
        return out

    def plan_epoch_batches(self, train_nodes, epoch, batch_size, seed):
        o = self.plan_epoch_order(train_nodes, epoch, seed)
        return [o[i:i + batch_size] for i in range(0, len(o), batch_size)]

    # -- reservoirs ---------------------------------------------------------
    def weighted_reservoir(self, nbrs, weights, m, key, ctr=0):
        n = np.ascontiguousarray(nbrs, dtype=np.uint32)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = np.zeros(max(1, min(len(n), max(m, 1))), dtype=np.uint32)
        c = C.c_uint64(ctr)
        r = self.L.orc_weighted_reservoir(_p(n, u32p), _p(w, f64p), len(n), m, key, C.byref(c), _p(out, u32p))
        if r < 0:
            raise SamplerError(int(r))
        return out[:r], c.value

    def uniform_reservoir(self, nbrs, m, key, ctr=0):
        n = np.ascontiguousarray(nbrs, dtype=np.uint32)
        out = np.zeros(max(1, min(len(n), max(m, 1))), dtype=np.uint32)
        c = C.c_uint64(ctr)
        r = self.L.orc_uniform_reservoir(_p(n, u32p), len(n), m, key, C.byref(c), _p(out, u32p))
        if r < 0:
            raise SamplerError(int(r))
        return out[:r], c.value

    # -- k-hop ---------------------------------------------------------------
    def _batch_from(self, h, seeds) -> Batch:
        L = self.L
        U = L.orc_batch_num_unique(h)
        uniq = np.ctypeslib.as_array(L.orc_batch_unique(h), shape=(max(U, 1),))[:U].copy()
        b = Batch(np.asarray(seeds, dtype=np.uint32).copy(), uniq, int(L.orc_batch_num_seed_unique(h)),
                  int(L.orc_batch_dups(h)), [], int(L.orc_batch_keys_scanned(h)))
        return b

    def sample_khop(self, g, seeds, fanouts, gamma=1.0, kind=WEIGHTED, rng_seed=0, device_map=None) -> Batch:
        s = np.ascontiguousarray(seeds, dtype=np.uint32)
        f = np.ascontiguousarray(fanouts, dtype=np.uint32)
        dm = None if device_map is None else np.ascontiguousarray(device_map, dtype=np.int32)
        err = C.c_int(0)
        h = self.L.orc_sample_khop(g.num_nodes, _p(g.row_offsets, u64p), _p(g.col_indices, u32p), _p(s, u32p),
                                   len(s), _p(f, u32p), len(f), gamma, kind, rng_seed,
                                   None if dm is None else _p(dm, i32p), C.byref(err))
        if not h:
            raise SamplerError(err.value)
        try:
            b = self._batch_from(h, s)
            for l in range(len(f)):
                ne = self.L.orc_batch_layer_ne(h, l)
                if ne:
                    d = np.ctypeslib.as_array(self.L.orc_batch_layer_dst(h, l), shape=(ne,)).copy()
                    sr = np.ctypeslib.as_array(self.L.orc_batch_layer_src(h, l), shape=(ne,)).copy()
                else:
                    d = np.zeros(0, np.uint32)
                    sr = np.zeros(0, np.uint32)
                b.layers.append((d, sr))
        finally:
            self.L.orc_batch_free(h)
        return b

    # -- cache ---------------------------------------------------------------
    def build_static_cache(self, g, volume_bytes, num_devices=1) -> np.ndarray:
        dm = np.empty(g.num_nodes, dtype=np.int32)
        r = self.L.orc_build_static_cache(g.num_nodes, _p(g.row_offsets, u64p), g.feat_dim, volume_bytes,
                                          num_devices, _p(dm, i32p))
        if r < 0:
            raise SamplerError(int(r), "num_devices < 1")
        return dm

    @staticmethod
    def retrieve_features(g, b: Batch, device_map=None):
        """cache.cpp:70-87 semantics in numpy (rows, hits, misses, B)."""
        rows = g.features[b.unique_nodes]
        if device_map is None:
            hits = 0
        else:
            hits = int((device_map[b.unique_nodes] != -1).sum())
        misses = len(b.unique_nodes) - hits
        B = len(b.unique_nodes) * g.feat_dim * 4 + b.total_edges() * 8
        return rows, hits, misses, B

    # -- trainer -------------------------------------------------------------
    def init_model(self, F, H, Cc, seed):
        w1 = np.empty(F * H, np.float64)
        w2 = np.empty(H * Cc, np.float64)
        if self.L.orc_init_model(F, H, Cc, seed, _p(w1, f64p), _p(w2, f64p)) != 0:
            raise SamplerError(-1, "init_model: dims must be >= 1")
        return w1, w2

    def _edges_args(self, layers):
        L = len(layers)
        ne = np.array([len(d) for d, _ in layers] + [0], dtype=np.uint64)
        keep = []
        D = (u32p * max(L, 1))()
        S = (u32p * max(L, 1))()
        for i, (d, s) in enumerate(layers):
            d = np.ascontiguousarray(d, dtype=np.uint32)
            s = np.ascontiguousarray(s, dtype=np.uint32)
            keep += [d, s]
            D[i] = _p(d, u32p)
            S[i] = _p(s, u32p)
        return ne, D, S, keep

    def grad_on_batch(self, g, b: Batch, feats, w1, w2, H, Cc, want_intermediates=False):
        """forward+backward (trainer.cpp:231-239). Returns dict."""
        F = g.feat_dim
        ns = b.num_seed_unique
        ne, D, S, keep = self._edges_args(b.layers)
        U = len(b.unique_nodes)
        feats = np.ascontiguousarray(feats, dtype=np.float32)
        gw1 = np.empty(F * H)
        gw2 = np.empty(H * Cc)
        logits = np.empty(ns * Cc)
        # n_inner <= U
        agg_inner = np.empty(U * F) if want_intermediates else None
        h1 = np.empty(U * H) if want_intermediates else None
        agg_outer = np.empty(ns * H) if want_intermediates else None
        labels = np.zeros(ns, np.uint32)
        seed_labels = g.labels[b.unique_nodes[:ns]].astype(np.uint32)
        loss = self.L.orc_grad_on_edges(F, H, Cc, _p(w1, f64p), _p(w2, f64p), U, ns, len(b.layers),
                                        _p(ne, u64p), D, S, _p(feats, f32p), _p(seed_labels, u32p),
                                        _p(gw1, f64p), _p(gw2, f64p), _p(logits, f64p))
        out = dict(loss=loss, gw1=gw1, gw2=gw2, logits=logits.reshape(ns, Cc))
        del labels, keep
        return out

    def grad_on_edges(self, F, H, Cc, w1, w2, n_unique, n_seeds, layers, feats, seed_labels):
        ne, D, S, keep = self._edges_args(layers)
        feats = np.ascontiguousarray(feats, dtype=np.float32)
        seed_labels = np.ascontiguousarray(seed_labels, dtype=np.uint32)
        gw1 = np.empty(F * H)
        gw2 = np.empty(H * Cc)
        logits = np.empty(n_seeds * Cc)
        loss = self.L.orc_grad_on_edges(F, H, Cc, _p(w1, f64p), _p(w2, f64p), n_unique, n_seeds, len(layers),
                                        _p(ne, u64p), D, S, _p(feats, f32p), _p(seed_labels, u32p),
                                        _p(gw1, f64p), _p(gw2, f64p), _p(logits, f64p))
        return dict(loss=loss, gw1=gw1, gw2=gw2, logits=logits.reshape(n_seeds, Cc))

    def train_steps(self, g, fanouts, gamma, kind, rng_seed, batch_size, H, Cc, lr, w1, w2, max_steps,
                    device_map=None):
        f = np.ascontiguousarray(fanouts, dtype=np.uint32)
        w1 = np.array(w1, dtype=np.float64)
        w2 = np.array(w2, dtype=np.float64)
        losses = np.zeros(max_steps)
        hits = C.c_uint64(0)
        misses = C.c_uint64(0)
        dm = None if device_map is None else np.ascontiguousarray(device_map, dtype=np.int32)
        feats = np.ascontiguousarray(g.features, dtype=np.float32)
        r = self.L.orc_train_steps(g.num_nodes, _p(g.row_offsets, u64p), _p(g.col_indices, u32p),
                                   _p(feats, f32p), g.feat_dim, _p(g.labels, u32p), _p(g.train_mask, u8p),
                                   None if dm is None else _p(dm, i32p), _p(f, u32p), len(f), gamma, kind,
                                   rng_seed, batch_size, H, Cc, lr, _p(w1, f64p), _p(w2, f64p), max_steps,
                                   _p(losses, f64p), C.byref(hits), C.byref(misses))
        if r < 0:
            raise SamplerError(int(r))
        return dict(losses=losses[:r], w1=w1, w2=w2, hits=hits.value, misses=misses.value)


# --------------------------------------------------------------------------
@dataclass
class RefGraph:
    """A graph owned by the reference library (graph.hpp:14-36) with numpy
    views over its vectors (valid while the handle lives)."""
    lib: object
    h: int
    num_nodes: int
    num_edges: int
    feat_dim: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    features: np.ndarray
    labels: np.ndarray
    train_mask: np.ndarray
    test_mask: np.ndarray

    def __del__(self):
        try:
            self.lib.L.ref_graph_free(self.h)
        except Exception:
            pass


class RefLib:
    """The compiled, unmodified reference (through oracle/ref_shim.cpp)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_backend.restype = C.c_int
        L.ref_set_backend.argtypes = [C.c_int]
        L.ref_graph_power_law.restype = C.c_void_p
        L.ref_graph_power_law.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_uint32, C.c_uint64]
        L.ref_graph_sbm.restype = C.c_void_p
        L.ref_graph_sbm.argtypes = [C.c_uint64, C.c_uint32, C.c_double, C.c_double, C.c_uint32, C.c_uint64]
        L.ref_graph_from_edges.restype = C.c_void_p
        L.ref_graph_from_edges.argtypes = [C.c_uint64, u32p, u32p, C.c_uint64, C.c_uint32]
        L.ref_graph_load.restype = C.c_void_p
        L.ref_graph_load.argtypes = [C.c_char_p]
        L.ref_graph_save.restype = C.c_int
        L.ref_graph_save.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_graph_info.argtypes = [C.c_void_p, u64p, u64p, u32p]
        L.ref_graph_arrays.argtypes = [C.c_void_p] + [C.c_void_p] * 6
        L.ref_build_static_cache.restype = C.c_int64
        L.ref_build_static_cache.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, i32p]
        L.ref_sample_khop.restype = C.c_void_p
        L.ref_sample_khop.argtypes = [C.c_void_p, i32p, C.c_uint32, u32p, C.c_uint64, u32p, C.c_uint32,
                                      C.c_double, C.c_int, C.c_uint64, C.POINTER(C.c_int)]
        for name, rt in [("ref_batch_num_unique", C.c_uint64), ("ref_batch_num_seed_unique", C.c_uint64),
                         ("ref_batch_dups", C.c_uint64), ("ref_batch_unique", u32p)]:
            getattr(L, name).restype = rt
            getattr(L, name).argtypes = [C.c_void_p]
        for name, rt in [("ref_batch_layer_ne", C.c_uint64), ("ref_batch_layer_dst", u32p),
                         ("ref_batch_layer_src", u32p)]:
            getattr(L, name).restype = rt
            getattr(L, name).argtypes = [C.c_void_p, C.c_uint32]
        L.ref_batch_free.argtypes = [C.c_void_p]
        L.ref_weighted_reservoir.restype = C.c_int64
        L.ref_weighted_reservoir.argtypes = [u32p, f64p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, u32p]
        L.ref_uniform_reservoir.restype = C.c_int64
        L.ref_uniform_reservoir.argtypes = [u32p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, u32p]
        L.ref_retrieve_features.restype = C.c_uint64
        L.ref_retrieve_features.argtypes = [C.c_void_p, i32p, C.c_uint32, C.c_void_p, f32p, u64p, u64p]
        L.ref_init_model.restype = C.c_int
        L.ref_init_model.argtypes = [C.c_uint32] * 3 + [C.c_uint64, f64p, f64p]
        L.ref_grad_on_batch.restype = C.c_double
        L.ref_grad_on_batch.argtypes = [C.c_void_p, C.c_void_p, f32p, C.c_uint32, C.c_uint32, f64p, f64p, f64p,
                                        f64p, u64p, f64p, f64p, f64p, f64p]
        L.ref_grad_on_edges.restype = C.c_double
        L.ref_grad_on_edges.argtypes = [C.c_uint32] * 3 + [f64p, f64p, C.c_uint64, C.c_uint64, C.c_uint32,
                                                           u64p, C.POINTER(u32p), C.POINTER(u32p), f32p, u32p,
                                                           f64p, f64p, f64p]
        L.ref_sampling_seed.restype = C.c_uint64
        L.ref_sampling_seed.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.ref_plan_epoch_order.argtypes = [u32p, C.c_uint64, C.c_uint32, C.c_uint64, u32p]
        L.ref_train.restype = C.c_int
        L.ref_train.argtypes = [C.c_void_p, i32p, u32p, C.c_uint32, C.c_double, C.c_int, C.c_uint64,
                                C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                                f64p, f64p, f64p]
        L.ref_train_steps.restype = C.c_int64
        L.ref_train_steps.argtypes = [C.c_void_p, i32p, u32p, C.c_uint32, C.c_double, C.c_int, C.c_uint64,
                                      C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, f64p, f64p, C.c_uint64,
                                      f64p]
        L.ref_bench_steps.restype = C.c_double
        L.ref_bench_steps.argtypes = [C.c_void_p, i32p, u32p, C.c_uint32, C.c_double, C.c_uint64, C.c_uint32,
                                      C.c_uint32, C.c_uint32, C.c_double, C.c_uint32, C.c_uint32, C.c_int,
                                      C.c_uint32, C.c_uint32, u64p]

    def err(self):
        return self.L.ref_last_error().decode()

    def _wrap(self, h) -> RefGraph:
        if not h:
            raise SamplerError(-1, self.err())
        n, m, f = C.c_uint64(), C.c_uint64(), C.c_uint32()
        self.L.ref_graph_info(h, C.byref(n), C.byref(m), C.byref(f))
        ptrs = [C.c_void_p() for _ in range(6)]
        self.L.ref_graph_arrays(h, *[C.byref(p) for p in ptrs])
        n, m, f = n.value, m.value, f.value

        def arr(p, t, cnt):
            if cnt == 0:
                return np.zeros(0, dtype=t)
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(np.ctypeslib.as_ctypes_type(t))), shape=(cnt,))

        return RefGraph(self, h, n, m, f, arr(ptrs[0], np.uint64, n + 1), arr(ptrs[1], np.uint32, m),
                        arr(ptrs[2], np.float32, n * f).reshape(n, f), arr(ptrs[3], np.uint32, n),
                        arr(ptrs[4], np.uint8, n), arr(ptrs[5], np.uint8, n))

    def power_law(self, n, m, exponent, f, seed) -> RefGraph:
        return self._wrap(self.L.ref_graph_power_law(n, m, exponent, f, seed))

    def sbm(self, n, blocks, p_in, p_out, f, seed) -> RefGraph:
        return self._wrap(self.L.ref_graph_sbm(n, blocks, p_in, p_out, f, seed))

    def from_edges(self, n, src, dst, f) -> RefGraph:
        s = np.ascontiguousarray(src, dtype=np.uint32)
        d = np.ascontiguousarray(dst, dtype=np.uint32)
        return self._wrap(self.L.ref_graph_from_edges(n, _p(s, u32p), _p(d, u32p), len(s), f))

    def load(self, path) -> RefGraph:
        return self._wrap(self.L.ref_graph_load(path.encode()))

    def save(self, g: RefGraph, path):
        if self.L.ref_graph_save(g.h, path.encode()) != 0:
            raise IOError(self.err())

    def build_static_cache(self, g: RefGraph, volume_bytes, num_devices=1):
        dm = np.empty(g.num_nodes, dtype=np.int32)
        r = self.L.ref_build_static_cache(g.h, volume_bytes, num_devices, _p(dm, i32p))
        if r < 0:
            raise SamplerError(int(r), self.err())
        return dm

    def sample_khop(self, g: RefGraph, seeds, fanouts, gamma=1.0, kind=WEIGHTED, rng_seed=0, device_map=None,
                    num_devices=1, keep_handle=False):
        s = np.ascontiguousarray(seeds, dtype=np.uint32)
        f = np.ascontiguousarray(fanouts, dtype=np.uint32)
        dm = None if device_map is None else np.ascontiguousarray(device_map, dtype=np.int32)
        err = C.c_int(0)
        h = self.L.ref_sample_khop(g.h, None if dm is None else _p(dm, i32p), num_devices, _p(s, u32p), len(s),
                                   _p(f, u32p), len(f), gamma, kind, rng_seed, C.byref(err))
        if not h:
            raise SamplerError(err.value, self.err())
        L = self.L
        U = L.ref_batch_num_unique(h)
        uniq = np.ctypeslib.as_array(L.ref_batch_unique(h), shape=(max(U, 1),))[:U].copy()
        b = Batch(s.copy(), uniq, int(L.ref_batch_num_seed_unique(h)), int(L.ref_batch_dups(h)), [])
        for l in range(len(f)):
            ne = L.ref_batch_layer_ne(h, l)
            if ne:
                d = np.ctypeslib.as_array(L.ref_batch_layer_dst(h, l), shape=(ne,)).copy()
                sr = np.ctypeslib.as_array(L.ref_batch_layer_src(h, l), shape=(ne,)).copy()
            else:
                d = np.zeros(0, np.uint32)
                sr = np.zeros(0, np.uint32)
            b.layers.append((d, sr))
        if keep_handle:
            return b, h
        L.ref_batch_free(h)
        return b

    def weighted_reservoir(self, nbrs, weights, m, seed, stream):
        n = np.ascontiguousarray(nbrs, dtype=np.uint32)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = np.zeros(max(1, len(n)), dtype=np.uint32)
        r = self.L.ref_weighted_reservoir(_p(n, u32p), _p(w, f64p), len(n), m, seed, stream, _p(out, u32p))
        if r < 0:
            raise SamplerError(int(r), self.err())
        return out[:r]

    def uniform_reservoir(self, nbrs, m, seed, stream):
        n = np.ascontiguousarray(nbrs, dtype=np.uint32)
        out = np.zeros(max(1, len(n)), dtype=np.uint32)
        r = self.L.ref_uniform_reservoir(_p(n, u32p), len(n), m, seed, stream, _p(out, u32p))
        if r < 0:
            raise SamplerError(int(r), self.err())
        return out[:r]

    def init_model(self, F, H, Cc, seed):
        w1 = np.empty(F * H)
        w2 = np.empty(H * Cc)
        if self.L.ref_init_model(F, H, Cc, seed, _p(w1, f64p), _p(w2, f64p)) != 0:
            raise SamplerError(-1, self.err())
        return w1, w2

    def grad_on_edges(self, F, H, Cc, w1, w2, n_unique, n_seeds, layers, feats, seed_labels):
        ne = np.array([len(d) for d, _ in layers] + [0], dtype=np.uint64)
        keep = []
        D = (u32p * max(len(layers), 1))()
        S = (u32p * max(len(layers), 1))()
        for i, (d, s) in enumerate(layers):
            d = np.ascontiguousarray(d, dtype=np.uint32)
            s = np.ascontiguousarray(s, dtype=np.uint32)
            keep += [d, s]
            D[i] = _p(d, u32p)
            S[i] = _p(s, u32p)
        feats = np.ascontiguousarray(feats, dtype=np.float32)
        seed_labels = np.ascontiguousarray(seed_labels, dtype=np.uint32)
        gw1 = np.empty(F * H)
        gw2 = np.empty(H * Cc)
        logits = np.empty(n_seeds * Cc)
        loss = self.L.ref_grad_on_edges(F, H, Cc, _p(w1, f64p), _p(w2, f64p), n_unique, n_seeds, len(layers),
                                        _p(ne, u64p), D, S, _p(feats, f32p), _p(seed_labels, u32p),
                                        _p(gw1, f64p), _p(gw2, f64p), _p(logits, f64p))
        return dict(loss=loss, gw1=gw1, gw2=gw2, logits=logits.reshape(n_seeds, Cc))

    def sampling_seed(self, base, epoch, step, worker=0):
        return self.L.ref_sampling_seed(base, epoch, step, worker)

    def plan_epoch_order(self, train_nodes, epoch, seed):
        t = np.ascontiguousarray(train_nodes, dtype=np.uint32)
        out = np.empty_like(t)
        self.L.ref_plan_epoch_order(_p(t, u32p), len(t), epoch, seed, _p(out, u32p))
        return out

    def train(self, g, device_map, fanouts, gamma, kind, rng_seed, batch_size, epochs, H, Cc, lr, model_seed):
        f = np.ascontiguousarray(fanouts, dtype=np.uint32)
        dm = None if device_map is None else np.ascontiguousarray(device_map, dtype=np.int32)
        lc = np.zeros(epochs)
        hr = np.zeros(epochs)
        acc = C.c_double()
        r = self.L.ref_train(g.h, None if dm is None else _p(dm, i32p), _p(f, u32p), len(f), gamma, kind,
                             rng_seed, batch_size, epochs, H, Cc, lr, model_seed, _p(lc, f64p), _p(hr, f64p),
                             C.byref(acc))
        if r != 0:
            raise SamplerError(r, self.err())
        return dict(loss_curve=lc, hit_rates=hr, accuracy=acc.value)

    def train_steps(self, g, device_map, fanouts, gamma, kind, rng_seed, batch_size, H, Cc, lr, w1, w2,
                    max_steps):
        f = np.ascontiguousarray(fanouts, dtype=np.uint32)
        dm = None if device_map is None else np.ascontiguousarray(device_map, dtype=np.int32)
        w1 = np.array(w1, dtype=np.float64)
        w2 = np.array(w2, dtype=np.float64)
        losses = np.zeros(max_steps)
        r = self.L.ref_train_steps(g.h, None if dm is None else _p(dm, i32p), _p(f, u32p), len(f), gamma, kind,
                                   rng_seed, batch_size, H, Cc, lr, _p(w1, f64p), _p(w2, f64p), max_steps,
                                   _p(losses, f64p))
        if r < 0:
            raise SamplerError(int(r), self.err())
        return dict(losses=losses[:r], w1=w1, w2=w2)

    def bench_steps(self, g, device_map, fanouts, gamma, rng_seed, batch_size, H, Cc, lr, units, producers,
                    queue_capacity=8, warmup=0, mode=1):
        """Seconds for `units` steps (after `warmup` untimed ones) of the
        executor schedule `mode` (0 sequential, 1 pmode1, 2 pmode2) over the
        reference's own per-batch functions; returns (seconds, seeds)."""
        f = np.ascontiguousarray(fanouts, dtype=np.uint32)
        dm = None if device_map is None else np.ascontiguousarray(device_map, dtype=np.int32)
        seeds = C.c_uint64()
        t = self.L.ref_bench_steps(g.h, None if dm is None else _p(dm, i32p), _p(f, u32p), len(f), gamma,
                                   rng_seed, batch_size, H, Cc, lr, warmup, units, mode, producers,
                                   queue_capacity, C.byref(seeds))
        return t, seeds.value


def ref_available() -> bool:
    return os.path.exists(REF_SO)
