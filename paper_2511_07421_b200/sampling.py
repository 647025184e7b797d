"""a3gnn::sampling mirror (proj/include/a3gnn/sampler.hpp) over the sm_100a sampler.

``sample_khop`` runs the whole k-hop sample on the GPU (sampler.cu) and copies
the SampleBatch back in the reference's exact layout and order.
``DeviceSampler`` keeps the batch resident for the training path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from ._lib import ParameterError, check, f64p, lib, ptr, u32p, u64p, vp
from .cache import CacheState
from .graph import Graph


class SamplerKind(enum.IntEnum):
    """sampler.hpp:18-21."""
    weighted_reservoir = 0
    uniform_baseline = 1


@dataclass
class SamplerConfig:
    """sampler.hpp:23-28."""
    fanouts: list = field(default_factory=list)  # outermost first
    bias_rate: float = 1.0                       # gamma >= 1
    rng_seed: int = 0
    kind: SamplerKind = SamplerKind.weighted_reservoir


@dataclass
class SampleBatch:
    """sampler.hpp:30-46; layers[l] = (dst_idx u32[E], src_idx u32[E])."""
    seeds: np.ndarray
    unique_nodes: np.ndarray
    num_seed_unique: int = 0
    layers: list = field(default_factory=list)
    num_duplicates_removed: int = 0

    def total_edges(self) -> int:
        return int(sum(len(d) for d, _ in self.layers))

    def edges(self, l: int):
        d, s = self.layers[l]
        return list(zip(d.tolist(), s.tolist()))


class DeviceSampler:
    """An ``a3g_sampler*`` arena: device-resident k-hop batches."""

    def __init__(self, g: Graph, cache: CacheState, max_seeds: int, fanouts, device: int = 0):
        self.g = g
        self.cache = cache
        self.fanouts = [int(f) for f in fanouts]
        f = np.asarray(self.fanouts, dtype=np.uint32)
        if any(x < 1 for x in self.fanouts):
            raise ParameterError("sample_khop: fanout must be >= 1")
        dg = g.device(device)
        h = vp()
        check(lib().a3g_sampler_create(dg.h, cache.device(g, device), max_seeds, ptr(f, u32p), len(f), C.byref(h)))
        self.h = h
        self.max_seeds = max_seeds

    def __del__(self):
        try:
            if self.h:
                lib().a3g_sampler_destroy(self.h)
        except Exception:
            pass

    def sample(self, seeds, bias_rate=1.0, kind=SamplerKind.weighted_reservoir, rng_seed=0):
        s = np.ascontiguousarray(seeds, dtype=np.uint32)
        check(lib().a3g_sample_khop(self.h, ptr(s, u32p), len(s), 0, float(bias_rate), int(kind), int(rng_seed),
                                    None))
        self._seeds = s

    def sizes(self):
        L = len(self.fanouts)
        nu, ns, dups = C.c_uint64(), C.c_uint64(), C.c_uint64()
        le = np.zeros(max(L, 1), dtype=np.uint64)
        check(lib().a3g_batch_sizes(self.h, C.byref(nu), C.byref(ns), C.byref(dups), ptr(le, u64p)))
        return nu.value, ns.value, dups.value, le[:L]

    def batch(self) -> SampleBatch:
        nu, ns, dups, le = self.sizes()
        L = len(self.fanouts)
        uniq = np.empty(max(nu, 1), dtype=np.uint32)
        ds = [np.empty(max(int(e), 1), dtype=np.uint32) for e in le]
        ss = [np.empty(max(int(e), 1), dtype=np.uint32) for e in le]
        D = (u32p * max(L, 1))(*[ptr(x, u32p) for x in ds])
        S = (u32p * max(L, 1))(*[ptr(x, u32p) for x in ss])
        check(lib().a3g_batch_copy(self.h, ptr(uniq, u32p), D, S))
        layers = [(ds[l][:int(le[l])].copy(), ss[l][:int(le[l])].copy()) for l in range(L)]
        return SampleBatch(self._seeds.copy(), uniq[:nu].copy(), int(ns), layers, int(dups))

    def retrieve_features(self):
        """Gather the last batch's unique rows (device) -> host f32[U, F], hits, misses, B."""
        nu = self.sizes()[0]
        out = np.empty(max(nu, 1) * self.g.feat_dim, dtype=np.float32)
        h, m, B = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().a3g_retrieve_features(self.h, ptr(out, C.POINTER(C.c_float)), 0, C.byref(h), C.byref(m),
                                          C.byref(B), None))
        return out[:nu * self.g.feat_dim].reshape(nu, self.g.feat_dim), h.value, m.value, B.value


_SAMPLERS: dict = {}


def _sampler_for(g: Graph, cache: CacheState, n_seeds: int, fanouts) -> DeviceSampler:
    key = (id(g), id(cache), tuple(int(f) for f in fanouts))
    s = _SAMPLERS.get(key)
    if s is None or s.max_seeds < n_seeds or s.g is not g or s.cache is not cache:
        cap = max(n_seeds, 1024 if s is None else 2 * s.max_seeds)
        s = DeviceSampler(g, cache, cap, fanouts)
        _SAMPLERS[key] = s
    return s


def clear_sampler_cache():
    _SAMPLERS.clear()


def sample_khop(g: Graph, seeds, cfg: SamplerConfig, cache: CacheState) -> SampleBatch:
    """sampler.hpp:62-63, on the GPU; same errors as sampler.cpp:91-94,110."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint32)
    if len(seeds) == 0:
        raise ParameterError("sample_khop: seeds must be non-empty")
    if any(int(f) < 1 for f in cfg.fanouts):
        # the reference throws at the layer's start; seeds are validated first
        if np.any(seeds >= g.num_nodes):
            raise ParameterError("sample_khop: seed out of range")
        raise ParameterError("sample_khop: fanout must be >= 1")
    s = _sampler_for(g, cache, len(seeds), cfg.fanouts)
    s.sample(seeds, cfg.bias_rate, cfg.kind, cfg.rng_seed)
    return s.batch()


def weighted_reservoir_sample(neighbors, weights, m: int, key: int, ctr: int = 0):
    """sampler.hpp:50-53 on the device (one warp). The RNG stream is given as
    (key, counter) -- RngStream(seed, stream).key == hash2(seed, stream).
    Returns (reservoir, new counter)."""
    n = np.ascontiguousarray(neighbors, dtype=np.uint32)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    if len(n) != len(w):
        raise ParameterError("weighted_reservoir_sample: |neighbors| != |weights|")
    out = np.zeros(max(1, min(len(n), max(m, 1))), dtype=np.uint32)
    cnt = C.c_uint64()
    check(lib().a3g_weighted_reservoir(ptr(n, u32p), ptr(w, f64p), len(n), m, key, ctr, ptr(out, u32p),
                                       C.byref(cnt)))
    return out[:cnt.value], ctr + len(n)


def uniform_reservoir_sample(neighbors, m: int, key: int, ctr: int = 0):
    """sampler.hpp:55-57 on the device. Returns (reservoir, new counter)."""
    n = np.ascontiguousarray(neighbors, dtype=np.uint32)
    out = np.zeros(max(1, min(len(n), max(m, 1))), dtype=np.uint32)
    cnt = C.c_uint64()
    check(lib().a3g_uniform_reservoir(ptr(n, u32p), len(n), m, key, ctr, ptr(out, u32p), C.byref(cnt)))
    return out[:cnt.value], ctr + max(0, len(n) - m)


def assign_weights(neighbors, cache: CacheState, gamma: float) -> np.ndarray:
    """sampler.cpp:60-68."""
    if gamma < 1.0:
        raise ParameterError("assign_weights: gamma must be >= 1")
    n = np.asarray(neighbors, dtype=np.int64)
    cached = np.array([cache.is_cached(int(v)) for v in n], dtype=bool)
    return np.where(cached, float(gamma), 1.0)


def dedup_ratio(b: SampleBatch) -> float:
    """sampler.cpp:139-142."""
    d = float(b.num_duplicates_removed)
    return d / (d + float(len(b.unique_nodes)))


def validate_batch(g: Graph, b: SampleBatch) -> None:
    """sampler.cpp:144-165 (vectorised)."""
    U = len(b.unique_nodes)
    for d, s in b.layers:
        if len(d) and (int(d.max()) >= U or int(s.max()) >= U):
            raise ParameterError("validate_batch: edge index out of range")
        for di, si in zip(b.unique_nodes[d], b.unique_nodes[s]):
            nb = g.out_neighbors(int(di))
            k = np.searchsorted(nb, si)
            if k >= len(nb) or nb[k] != si:
                raise ParameterError("validate_batch: sampled edge not in CSR")
    if len(np.unique(b.unique_nodes)) != U:
        raise ParameterError("validate_batch: unique_nodes has repeats")
