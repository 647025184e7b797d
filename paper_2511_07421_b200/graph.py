"""a3gnn::graph mirror (proj/include/a3gnn/graph.hpp, generators.hpp, graph_io.hpp).

``Graph`` is the host CSR + dense feature store (graph.hpp:14-36) with numpy
arrays; ``Graph.device(dev)`` uploads it once into HBM (pitched rows, f32 or
bf16) and returns the C-ABI handle shared by caches, samplers and trainers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, f32p, i32p, lib, ptr, u32p, u64p, vp

FEAT_F32, FEAT_BF16 = 0, 1


@dataclass
class GraphStats:
    density: float = 0.0
    degree_mean: float = 0.0
    degree_max: int = 0
    num_nodes: int = 0
    num_edges: int = 0


class DeviceGraph:
    """Owns an ``a3g_graph*`` (device CSR + feature store)."""

    def __init__(self, g: "Graph", device: int, feat_dtype: int, upload_features: bool = True):
        h = vp()
        feats = g.features if upload_features and g.features is not None and g.features.size else None
        check(lib().a3g_graph_create(device, g.num_nodes, g.num_edges, g.feat_dim, ptr(g.row_offsets, u64p),
                                     ptr(g.col_indices, u32p), None if feats is None else ptr(feats, f32p),
                                     feat_dtype, ptr(g.labels, u32p), C.byref(h)))
        self.h = h
        self.device = device
        self.feat_dtype = feat_dtype
        self.graph = g

    def __del__(self):
        try:
            if self.h:
                lib().a3g_graph_destroy(self.h)
        except Exception:
            pass


STORE_HBM, STORE_CACHE, STORE_SHARDED = 0, 1, 2


class Store:
    """Tiered feature store (a3g_store_*) attached to a
    DeviceGraph: the B200 placement of the reference's static cache
    (cache.cpp:12-46). Policies: STORE_HBM (all rows in HBM), STORE_CACHE
    (cached rows in HBM, misses in mapped pinned host memory), STORE_SHARDED
    (rank r holds device_map == r, peers over NVLink, misses on the host)."""

    def __init__(self, dg: DeviceGraph, features: np.ndarray, device_map=None, policy: int = STORE_HBM,
                 rank: int = 0, nranks: int = 1):
        # features None: the rows come from the graph's own device table (synthesized)
        f = None if features is None else np.ascontiguousarray(features, dtype=np.float32)
        dm = None if device_map is None else np.ascontiguousarray(device_map, dtype=np.int32)
        h = vp()
        check(lib().a3g_store_create(dg.h, None if f is None else ptr(f, f32p), None if dm is None else ptr(dm, i32p), policy, rank,
                                     nranks, C.byref(h)))
        self.h, self.dg, self.policy, self.rank, self.nranks = h, dg, policy, rank, nranks

    def info(self):
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().a3g_store_info(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return dict(local_rows=a.value, host_rows=b.value, remote_rows=c.value)

    def local_ptr(self) -> int:
        p = vp()
        check(lib().a3g_store_local_ptr(self.h, C.byref(p)))
        return p.value or 0

    def set_peer(self, rank: int, dev_ptr: int) -> None:
        check(lib().a3g_store_set_peer(self.h, rank, vp(dev_ptr)))

    def ipc_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        check(lib().a3g_store_ipc_handle(self.h, buf))
        return bytes(buf)

    def open_peer(self, rank: int, handle: bytes) -> None:
        buf = (C.c_uint8 * 64).from_buffer_copy(handle)
        check(lib().a3g_store_open_peer(self.h, rank, buf))

    def __del__(self):
        try:
            if self.h and self.dg.h:
                lib().a3g_store_destroy(self.h)
        except Exception:
            pass


@dataclass(eq=False)
class Graph:
    """graph::Graph (graph.hpp:14-36)."""
    num_nodes: int
    num_edges: int
    feat_dim: int
    row_offsets: np.ndarray          # u64[n+1]
    col_indices: np.ndarray          # u32[m]
    features: np.ndarray             # f32[n, F]
    labels: np.ndarray               # u32[n]
    train_mask: np.ndarray           # u8[n]
    test_mask: np.ndarray            # u8[n]
    _owner: object = field(default=None, repr=False)
    _dev: dict = field(default_factory=dict, repr=False)

    def out_neighbors(self, v: int) -> np.ndarray:
        return self.col_indices[self.row_offsets[v]:self.row_offsets[v + 1]]

    def out_degree(self, v=None):
        d = np.diff(self.row_offsets)
        return d if v is None else int(d[v])

    def feature_row(self, v: int) -> np.ndarray:
        return self.features[v]

    def num_classes(self) -> int:
        return int(self.labels.max()) + 1 if self.num_nodes else 0

    def device(self, device: int = 0, feat_dtype: int = FEAT_F32) -> DeviceGraph:
        key = (device, feat_dtype)
        if key not in self._dev:
            self._dev[key] = DeviceGraph(self, device, feat_dtype)
        return self._dev[key]

    def release_device(self):
        self._dev.clear()

    @property
    def train_nodes(self) -> np.ndarray:
        return np.flatnonzero(self.train_mask).astype(np.uint32)


class _HostOwner:
    def __init__(self, p):
        self.p = p

    def __del__(self):
        try:
            lib().a3g_host_graph_free(self.p)
        except Exception:
            pass


def _wrap_host(p) -> Graph:
    hg = p.contents
    n, m, f = hg.num_nodes, hg.num_edges, hg.feat_dim

    def arr(ptr_, dtype, count):
        if count == 0:
            return np.zeros(0, dtype=dtype)
        return np.ctypeslib.as_array(ptr_, shape=(count,)).view(dtype)

    return Graph(n, m, f, arr(hg.row_offsets, np.uint64, n + 1), arr(hg.col_indices, np.uint32, m),
                 arr(hg.features, np.float32, n * f).reshape(n, f), arr(hg.labels, np.uint32, n),
                 arr(hg.train_mask, np.uint8, n), arr(hg.test_mask, np.uint8, n), _HostOwner(p))


def generate_power_law(n_nodes: int, min_degree: int, exponent: float, feat_dim: int, seed: int,
                       threads: int = 0) -> Graph:
    """generators.hpp:15-20; bit-identical to the reference, multithreaded."""
    p = C.POINTER(_lib.HostGraph)()
    check(lib().a3g_host_graph_power_law(n_nodes, min_degree, exponent, feat_dim, seed, threads, C.byref(p)))
    return _wrap_host(p)


def load_graph(path: str) -> Graph:
    """graph_io.hpp:13 (A3G1)."""
    p = C.POINTER(_lib.HostGraph)()
    check(lib().a3g_host_graph_load(path.encode(), C.byref(p)))
    return _wrap_host(p)


def save_graph(g: Graph, path: str) -> None:
    """graph_io.hpp:12 (A3G1)."""
    hg = _lib.HostGraph(g.num_nodes, g.num_edges, g.feat_dim, ptr(g.row_offsets, u64p), ptr(g.col_indices, u32p),
                        ptr(np.ascontiguousarray(g.features, np.float32), f32p), ptr(g.labels, u32p),
                        ptr(g.train_mask, _lib.u8p), ptr(g.test_mask, _lib.u8p))
    check(lib().a3g_host_graph_save(C.byref(hg), path.encode()))


def from_edges(num_nodes: int, edges, feat_dim: int) -> Graph:
    """graph.hpp:51-53 (sorts (src,dst); zero features/labels/masks)."""
    e = np.asarray(edges, dtype=np.uint32).reshape(-1, 2)
    src = np.ascontiguousarray(e[:, 0])
    dst = np.ascontiguousarray(e[:, 1])
    p = C.POINTER(_lib.HostGraph)()
    check(lib().a3g_host_graph_from_edges(num_nodes, ptr(src, u32p), ptr(dst, u32p), len(src), feat_dim,
                                          C.byref(p)))
    return _wrap_host(p)


def from_arrays(row_offsets, col_indices, features, labels=None, train_mask=None, test_mask=None) -> Graph:
    ro = np.ascontiguousarray(row_offsets, dtype=np.uint64)
    n = len(ro) - 1
    col = np.ascontiguousarray(col_indices, dtype=np.uint32)
    feats = np.ascontiguousarray(features, dtype=np.float32).reshape(n, -1)
    z = np.zeros(n, np.uint8)
    return Graph(n, len(col), feats.shape[1], ro, col, feats,
                 np.ascontiguousarray(labels if labels is not None else np.zeros(n), dtype=np.uint32),
                 np.ascontiguousarray(train_mask if train_mask is not None else z, dtype=np.uint8),
                 np.ascontiguousarray(test_mask if test_mask is not None else z, dtype=np.uint8))


def graph_stats(g: Graph) -> GraphStats:
    """graph.cpp:42-57."""
    s = GraphStats(num_nodes=g.num_nodes, num_edges=g.num_edges)
    if g.num_nodes > 1:
        s.density = g.num_edges / (g.num_nodes * (g.num_nodes - 1))
    if g.num_nodes > 0:
        s.degree_mean = g.num_edges / g.num_nodes
        s.degree_max = int(np.diff(g.row_offsets).max())
    return s


def validate(g: Graph) -> None:
    """graph.cpp:13-40 (raises ParameterError)."""
    P = _lib.ParameterError
    if g.feat_dim < 1:
        raise P("graph: feat_dim must be >= 1")
    if len(g.row_offsets) != g.num_nodes + 1:
        raise P("graph: row_offsets length mismatch")
    if g.row_offsets[0] != 0:
        raise P("graph: row_offsets[0] != 0")
    if g.row_offsets[-1] != g.num_edges:
        raise P("graph: row_offsets[last] != num_edges")
    if np.any(np.diff(g.row_offsets.astype(np.int64)) < 0):
        raise P("graph: row_offsets not non-decreasing")
    if len(g.col_indices) != g.num_edges:
        raise P("graph: col_indices length mismatch")
    if g.num_edges and int(g.col_indices.max()) >= g.num_nodes:
        raise P("graph: col_index out of range")
    if g.features.size != g.num_nodes * g.feat_dim:
        raise P("graph: feature matrix size mismatch")
    if len(g.labels) != g.num_nodes or len(g.train_mask) != g.num_nodes or len(g.test_mask) != g.num_nodes:
        raise P("graph: per-node array size mismatch")
