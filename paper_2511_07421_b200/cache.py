"""a3gnn::cache mirror (proj/include/a3gnn/cache.hpp).

The static out-degree hotness cache (cache.cpp:12-46) is built by the C-ABI;
``CacheState.device(dev)`` holds the device bitmap the sampler's locality bias
reads. ``retrieve_features`` gathers rows on the GPU (cache.cpp:70-87).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from ._lib import ParameterError, check, i32p, lib, ptr, u32p, f32p, u64p, vp
from .graph import Graph

KCACHE_MISS = -1


@dataclass
class CacheConfig:
    """cache.hpp:26-30: Theta per device (bytes), device count."""
    volume_bytes: int = 0
    num_devices: int = 1


class _DeviceCache:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            lib().a3g_cache_destroy(self.h)
        except Exception:
            pass


@dataclass(eq=False)
class CacheState:
    """cache.hpp:34-52."""
    device_map: np.ndarray                     # i32[n], -1 = miss
    num_devices: int = 1
    volume_bytes: int = 0
    _dev: dict = field(default_factory=dict, repr=False)
    _graph: object = field(default=None, repr=False)  # the graph it was last placed on (lookup)

    def is_cached(self, v: int) -> bool:
        return 0 <= v < len(self.device_map) and self.device_map[v] != KCACHE_MISS

    def device_of(self, v: int) -> int:
        return int(self.device_map[v]) if 0 <= v < len(self.device_map) else KCACHE_MISS

    @property
    def cached_per_device(self):
        return [np.flatnonzero(self.device_map == d).astype(np.uint32) for d in range(self.num_devices)]

    def total_cached(self) -> int:
        return int((self.device_map != KCACHE_MISS).sum())

    def device(self, g: Graph, device: int = 0, feat_dtype: int = 0):
        self._graph = g
        key = (id(g), device, feat_dtype)
        if key not in self._dev:
            dg = g.device(device, feat_dtype)
            h = vp()
            dm = np.ascontiguousarray(self.device_map, dtype=np.int32)
            check(lib().a3g_cache_from_map(dg.h, ptr(dm, i32p), self.num_devices, C.byref(h)))
            self._dev[key] = _DeviceCache(h)
        return self._dev[key].h


class CacheAccounting:
    """cache.hpp:54-63 (hits / misses / per-device hits; thread-safe)."""

    def __init__(self, num_devices: int = 1):
        self.hits = 0
        self.misses = 0
        self.per_device_hits = [0] * num_devices
        self._mu = threading.Lock()

    def total(self) -> int:
        return self.hits + self.misses

    def add(self, hits, misses):
        with self._mu:
            self.hits += int(hits)
            self.misses += int(misses)


@dataclass
class BatchStats:
    batch_bytes: int = 0
    num_nodes: int = 0
    num_edges: int = 0


def build_static_cache(g: Graph, cfg: CacheConfig, device: int = 0) -> CacheState:
    """cache.cpp:12-46 (degree desc, id asc; round-robin over devices)."""
    if cfg.num_devices < 1:
        raise ParameterError("build_static_cache: num_devices >= 1")
    dg = g.device(device)
    dm = np.empty(g.num_nodes, dtype=np.int32)
    h = vp()
    check(lib().a3g_cache_build(dg.h, cfg.volume_bytes, cfg.num_devices, ptr(dm, i32p), C.byref(h)))
    st = CacheState(dm, cfg.num_devices, cfg.volume_bytes)
    st._dev[(id(g), device, 0)] = _DeviceCache(h)
    st._graph = g
    return st


def lookup(c: CacheState, ids, acc: CacheAccounting, g: Graph | None = None, device: int = 0) -> np.ndarray:
    """cache.cpp:48-68 on the device (a3g_cache_lookup): per-id device
    (-1 = miss) and the hit / miss / per-device accounting. `g` names the graph
    the cache was built over (default: the one it was last placed on)."""
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    g = g if g is not None else c._graph
    if g is None:
        raise ParameterError("lookup: the cache has no graph (pass g)")
    out = np.empty(max(len(ids), 1), dtype=np.int32)
    h, m = C.c_uint64(), C.c_uint64()
    pd = np.zeros(max(c.num_devices, 1), dtype=np.uint64)
    check(lib().a3g_cache_lookup(c.device(g, device), ptr(ids, u32p), len(ids), ptr(out, i32p), C.byref(h),
                                 C.byref(m), ptr(pd, u64p)))
    acc.add(h.value, m.value)
    for dev in range(min(len(acc.per_device_hits), c.num_devices)):
        acc.per_device_hits[dev] += int(pd[dev])
    return out[:len(ids)]


def retrieve_features(b, c: CacheState, g: Graph, acc: CacheAccounting, device: int = 0):
    """cache.cpp:70-87: gather f32 rows of b.unique_nodes on the GPU; B bytes.

    Returns (feats f32[U*F], BatchStats)."""
    uniq = np.ascontiguousarray(b.unique_nodes, dtype=np.uint32)
    dg = g.device(device)
    ch = c.device(g, device)
    out = np.empty(len(uniq) * g.feat_dim, dtype=np.float32)
    hits, misses = C.c_uint64(), C.c_uint64()
    check(lib().a3g_gather_rows(dg.h, ch, ptr(uniq, u32p), len(uniq), ptr(out, f32p), C.byref(hits),
                                C.byref(misses)))
    acc.add(hits.value, misses.value)
    if c.num_devices > 1 and len(uniq):  # per-device hits from the device lookup
        pd = np.zeros(c.num_devices, dtype=np.uint64)
        check(lib().a3g_cache_lookup(ch, ptr(uniq, u32p), len(uniq), None, None, None, ptr(pd, u64p)))
        for dev in range(min(len(acc.per_device_hits), c.num_devices)):
            acc.per_device_hits[dev] += int(pd[dev])
    elif acc.per_device_hits:
        acc.per_device_hits[0] += hits.value
    ne = b.total_edges()
    st = BatchStats(len(uniq) * g.feat_dim * 4 + ne * 2 * 4, len(uniq), ne)
    return out, st


def hit_rate(acc: CacheAccounting) -> float:
    """cache.cpp:89-93."""
    t = acc.total()
    if t == 0:
        raise ParameterError("hit_rate: no lookups issued")
    return acc.hits / t
