"""a3gnn::train mirror (proj/include/a3gnn/trainer.hpp) over the sm_100a step.

``Trainer`` owns the device model (fp32 W1/W2), two sampler arenas and the
compute/sampling streams. ``step`` is one batch (sample -> gather+aggregate ->
forward -> backward -> [allreduce] -> sgd, trainer.cpp:385-406); ``steps``
runs K batches through the depth-2 CUDA-stream pipeline.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import ConfigError, ParameterError, check, f64p, i32p, lib, ptr, u8p, u32p, u64p, vp
from .cache import CacheState
from .graph import STORE_HBM, DeviceGraph, Graph, Store
from .sampling import SamplerKind


STAT_UNIQUE, STAT_EDGES, STAT_INNER, STAT_SEEDS, STAT_HITS, STAT_MISSES, STAT_BAD_SEEDS, STAT_POSITIONS = range(8)
STEP_STATS = 8


@dataclass
class ModelSpec:
    """trainer.hpp:24-36."""
    feat_dim: int = 0
    hidden_dim: int = 0
    num_classes: int = 0
    num_layers: int = 2
    learning_rate: float = 0.2

    def param_bytes(self) -> int:
        return (self.feat_dim * self.hidden_dim + self.hidden_dim * self.num_classes) * 4


def init_model(spec: ModelSpec, seed: int):
    """trainer.cpp:12-28 -> (w1 f64[F*H], w2 f64[H*C])."""
    w1 = np.empty(spec.feat_dim * spec.hidden_dim, dtype=np.float64)
    w2 = np.empty(spec.hidden_dim * spec.num_classes, dtype=np.float64)
    check(lib().a3g_init_model(spec.feat_dim, spec.hidden_dim, spec.num_classes, seed, ptr(w1, f64p),
                               ptr(w2, f64p)))
    return w1, w2


_M64 = (1 << 64) - 1


def mix64(z: int) -> int:
    """rng.hpp:15-22 (host integer arithmetic, for seeds and plans)."""
    z &= _M64
    z ^= z >> 30
    z = (z * 0xbf58476d1ce4e5b9) & _M64
    z ^= z >> 27
    z = (z * 0x94d049bb133111eb) & _M64
    return z ^ (z >> 31)


def hash2(a: int, b: int) -> int:
    """rng.hpp:24-27."""
    return mix64((a & _M64) ^ mix64((b + 0x9e3779b97f4a7c15) & _M64))


def sampling_seed(base: int, epoch: int, step: int, worker: int = 0) -> int:
    """trainer.cpp:345-348."""
    return int(lib().a3g_sampling_seed(base, epoch, step, worker))


def plan_epoch_order(train_nodes, epoch: int, seed: int) -> np.ndarray:
    t = np.ascontiguousarray(train_nodes, dtype=np.uint32)
    out = np.empty_like(t)
    lib().a3g_plan_epoch_order(ptr(t, u32p), len(t), epoch, seed, ptr(out, u32p))
    return out


def plan_epoch_batches(train_nodes, epoch: int, batch_size: int, seed: int):
    """trainer.cpp:330-343."""
    o = plan_epoch_order(train_nodes, epoch, seed)
    return [o[i:i + batch_size] for i in range(0, len(o), batch_size)]


def sgd_step(w: np.ndarray, g: np.ndarray, lr: float, fused: int = 0) -> None:
    """trainer.cpp:208-211 on the device (a3g_sgd_step): w += (-lr) * g in
    place, f64; the first `fused` elements as one fused multiply-add (the
    reference's AVX2 kernel table fuses n - n % 4), the rest rounded
    separately (its scalar table)."""
    w = np.asarray(w)
    if w.dtype != np.float64 or not w.flags.c_contiguous:
        raise ParameterError("sgd_step: weights must be a contiguous f64 array")
    gg = np.ascontiguousarray(g, dtype=np.float64)
    if gg.size != w.size:
        raise ParameterError("sgd_step: shape mismatch")
    check(lib().a3g_sgd_step(0, ptr(w, f64p), ptr(gg, f64p), w.size, int(fused), float(lr)))


def sync_gradients(grads):
    """trainer.cpp:213-229 on the device (a3g_mean_gradients): element-wise
    mean of a list of (gw1, gw2), summed in list order then x (1/k)."""
    if not grads:
        raise ParameterError("sync_gradients: empty gradient list")
    out = []
    for part in (0, 1):
        arrs = [np.ascontiguousarray(gr[part], dtype=np.float64) for gr in grads]
        if any(a.shape != arrs[0].shape for a in arrs):
            raise ParameterError("sync_gradients: shape mismatch")
        res = np.empty_like(arrs[0])
        ptrs = (f64p * len(arrs))(*[ptr(a, f64p) for a in arrs])
        check(lib().a3g_mean_gradients(0, ptrs, len(arrs), res.size, ptr(res, f64p)))
        out.append(res)
    return out[0], out[1]


class BatchModel:
    """trainer.cpp:34-239 on an explicit batch (a3g_batch_model_*): the
    reference's SampleBatch + the feats the caller gathered, through the
    pipeline's own device kernels."""

    def __init__(self, spec: ModelSpec, device: int = 0):
        h = vp()
        check(lib().a3g_batch_model_create(device, spec.feat_dim, spec.hidden_dim, spec.num_classes, C.byref(h)))
        self.h, self.spec = h, spec

    def __del__(self):
        try:
            if self.h:
                lib().a3g_batch_model_destroy(self.h)
        except Exception:
            pass

    def load(self, batch, feats, seed_labels=None) -> int:
        layers = list(batch.layers)[:2]
        L = len(layers)
        keep = []
        ne = np.array([len(d) for d, _ in layers] + [0], dtype=np.uint64)
        D = (u32p * max(L, 1))()
        S = (u32p * max(L, 1))()
        for i, (d, s_) in enumerate(layers):
            d = np.ascontiguousarray(d, dtype=np.uint32)
            s_ = np.ascontiguousarray(s_, dtype=np.uint32)
            keep += [d, s_]
            D[i], S[i] = ptr(d, u32p), ptr(s_, u32p)
        f = np.ascontiguousarray(feats, dtype=np.float32)
        lab = None if seed_labels is None else np.ascontiguousarray(seed_labels, dtype=np.uint32)
        ni = C.c_uint64()
        check(lib().a3g_batch_model_load(self.h, len(batch.unique_nodes), batch.num_seed_unique, L, ptr(ne, u64p), D,
                                         S, ptr(f, C.POINTER(C.c_float)), None if lab is None else ptr(lab, u32p),
                                         C.byref(ni)))
        return ni.value

    def run(self, w1, w2):
        a = np.ascontiguousarray(w1, dtype=np.float64)
        b = np.ascontiguousarray(w2, dtype=np.float64)
        loss = C.c_double()
        g1, g2 = np.empty_like(a), np.empty_like(b)
        check(lib().a3g_batch_model_run(self.h, ptr(a, f64p), ptr(b, f64p), C.byref(loss), ptr(g1, f64p),
                                        ptr(g2, f64p)))
        return loss.value, (g1, g2)


def forward(model, batch, feats, spec: ModelSpec, device: int = 0) -> dict:
    """trainer.cpp:59-137 on the device: the ForwardResult arrays (inner_nodes,
    inner_pos, inner_deg, outer_deg, agg_inner, h1, agg_outer, logits)."""
    bm = BatchModel(spec, device)
    ni = bm.load(batch, feats)
    bm.run(*model)
    F, H, Cc = spec.feat_dim, spec.hidden_dim, spec.num_classes
    ns, U = batch.num_seed_unique, len(batch.unique_nodes)
    out = dict(inner_nodes=np.empty(ni, np.uint32), inner_pos=np.empty(U, np.int32), inner_deg=np.empty(ni, np.uint32),
               outer_deg=np.empty(ns, np.uint32), agg_inner=np.empty(ni * F), h1=np.empty(ni * H),
               agg_outer=np.empty(ns * H), logits=np.empty(ns * Cc))
    check(lib().a3g_batch_model_forward(bm.h, ptr(out["inner_nodes"], u32p), ptr(out["inner_pos"], i32p),
                                        ptr(out["inner_deg"], u32p), ptr(out["outer_deg"], u32p),
                                        ptr(out["agg_inner"], f64p), ptr(out["h1"], f64p),
                                        ptr(out["agg_outer"], f64p), ptr(out["logits"], f64p)))
    return out


def backward(model, batch, feats, seed_labels, spec: ModelSpec, device: int = 0):
    """trainer.cpp:139-206 on the device (the forward is recomputed there):
    (loss, (gw1, gw2))."""
    if len(seed_labels) != batch.num_seed_unique:
        raise ParameterError("backward: seed_labels size mismatch")
    bm = BatchModel(spec, device)
    bm.load(batch, feats, seed_labels)
    return bm.run(*model)


def grad_on_batch(model, g: Graph, batch, feats, spec: ModelSpec, device: int = 0):
    """trainer.cpp:231-239: labels of the unique seeds from the graph, then backward."""
    labels = g.labels[np.asarray(batch.unique_nodes[:batch.num_seed_unique], dtype=np.int64)]
    return backward(model, batch, feats, labels, spec, device)


class Trainer:
    """Device-resident 2-layer mean-GCN trainer (trainer.hpp:24-60, 63-83)."""

    def __init__(self, g: Graph, cache: CacheState, spec: ModelSpec, fanouts, max_seeds: int,
                 model_seed: int = 1, device: int = 0, feat_dtype: int = 0, placement=None, synth_seed=None):
        """placement: None (whole feature table in HBM) or dict(policy=STORE_*,
        rank=0, nranks=1) -- feature rows placed by the tiered store from the
        cache's device_map (graph.Store). synth_seed: papers-scale inputs --
        the host graph carries topology/labels only (feat_dim 1) and the
        spec.feat_dim features are synthesized on the device
        (a3g_graph_synthesize_features, the generator's formula)."""
        if synth_seed is None and spec.feat_dim != g.feat_dim:
            raise ParameterError("trainer: spec.feat_dim != graph feat_dim")
        self.g, self.cache, self.spec = g, cache, spec
        self.fanouts = [int(x) for x in fanouts]
        if any(x < 1 for x in self.fanouts):
            raise ParameterError("sample_khop: fanout must be >= 1")
        f = np.asarray(self.fanouts, dtype=np.uint32)
        self.store = None
        if synth_seed is not None:
            dg = DeviceGraph(g, device, feat_dtype, upload_features=False)
            check(lib().a3g_graph_synthesize_features(dg.h, spec.feat_dim, feat_dtype, int(synth_seed)))
            if placement is not None:  # tiered store placed from the synthesized device table
                self.store = Store(dg, None, cache.device_map, placement.get("policy", STORE_HBM),
                                   placement.get("rank", 0), placement.get("nranks", 1))
            from .cache import _DeviceCache
            hc = vp()
            dm = np.ascontiguousarray(cache.device_map, dtype=np.int32)
            check(lib().a3g_cache_from_map(dg.h, ptr(dm, i32p), cache.num_devices, C.byref(hc)))
            dc = _DeviceCache(hc)
            ch = dc.h
            keep = [dc, self.store, dg]
        elif placement is None:
            dg = g.device(device, feat_dtype)
            ch = cache.device(g, device, feat_dtype)
            keep = [dg]
        else:
            dg = DeviceGraph(g, device, feat_dtype, upload_features=False)
            self.store = Store(dg, g.features, cache.device_map, placement.get("policy", STORE_HBM),
                               placement.get("rank", 0), placement.get("nranks", 1))
            from .cache import _DeviceCache
            hc = vp()
            dm = np.ascontiguousarray(cache.device_map, dtype=np.int32)
            check(lib().a3g_cache_from_map(dg.h, ptr(dm, i32p), cache.num_devices, C.byref(hc)))
            dc = _DeviceCache(hc)
            ch = dc.h
            keep = [dc, self.store, dg]
        h = vp()
        check(lib().a3g_trainer_create(dg.h, ch, max_seeds, ptr(f, u32p), len(f),
                                       spec.hidden_dim, spec.num_classes, spec.learning_rate, model_seed,
                                       C.byref(h)))
        self.h = h
        self.max_seeds = max_seeds
        self._keep = keep

    def __del__(self):
        try:
            if self.h:
                lib().a3g_trainer_destroy(self.h)
        except Exception:
            pass
        self._keep = None

    # -- weights ---------------------------------------------------------------
    def get_weights(self):
        w1 = np.empty(self.spec.feat_dim * self.spec.hidden_dim)
        w2 = np.empty(self.spec.hidden_dim * self.spec.num_classes)
        check(lib().a3g_trainer_get_weights(self.h, ptr(w1, f64p), ptr(w2, f64p)))
        return w1, w2

    def set_weights(self, w1, w2):
        a = np.ascontiguousarray(w1, dtype=np.float64)
        b = np.ascontiguousarray(w2, dtype=np.float64)
        check(lib().a3g_trainer_set_weights(self.h, ptr(a, f64p), ptr(b, f64p)))

    def set_pipeline(self, sampling_streams: int):
        """0 = sequential (Mode::sequential), 1..12 concurrent sampling streams (default: 12 for
        batches of <= 2048 seeds, else 8)."""
        check(lib().a3g_trainer_set_pipeline(self.h, int(sampling_streams)))

    def set_comm(self, comm):
        check(lib().a3g_trainer_set_comm(self.h, comm.h if comm is not None else None))

    # -- steps -----------------------------------------------------------------
    def step(self, seeds, bias_rate=1.0, kind=SamplerKind.weighted_reservoir, rng_seed=0, lr=None,
             sync_loss=True):
        s = np.ascontiguousarray(seeds, dtype=np.uint32)
        loss = C.c_double(float("nan"))
        check(lib().a3g_train_step(self.h, ptr(s, u32p), len(s), 0, float(bias_rate), int(kind), int(rng_seed),
                                   -1.0 if lr is None else float(lr), C.byref(loss) if sync_loss else None))
        return loss.value

    def grad_on_batch(self, seeds, bias_rate=1.0, kind=SamplerKind.weighted_reservoir, rng_seed=0):
        """trainer.cpp:231-239 on the device: loss and (gw1, gw2), weights untouched."""
        loss = self.step(seeds, bias_rate, kind, rng_seed, lr=0.0)
        return loss, self.last_grads()

    def steps(self, seed_batches: np.ndarray, rng_seeds, bias_rate=1.0, kind=SamplerKind.weighted_reservoir):
        """K pipelined steps; seed_batches u32[K, B] (host), rng_seeds u64[K]."""
        sb = np.ascontiguousarray(seed_batches, dtype=np.uint32)
        K, B = sb.shape
        rs = np.ascontiguousarray(rng_seeds, dtype=np.uint64)
        losses = np.empty(K, dtype=np.float64)
        check(lib().a3g_train_steps(self.h, ptr(sb, u32p), B, K, ptr(rs, u64p), float(bias_rate), int(kind), 0,
                                    ptr(losses, f64p)))
        return losses

    def steps_v(self, seeds, offsets, rng_seeds, bias_rate=1.0, kind=SamplerKind.weighted_reservoir):
        """Pipelined steps with per-step batch sizes: batch i = seeds[offsets[i]:offsets[i+1]]."""
        s = np.ascontiguousarray(seeds, dtype=np.uint32)
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        K = len(off) - 1
        rs = np.ascontiguousarray(rng_seeds, dtype=np.uint64)
        losses = np.empty(max(K, 0), dtype=np.float64)
        check(lib().a3g_train_steps_v(self.h, ptr(s, u32p), ptr(off, u64p), K, ptr(rs, u64p), float(bias_rate),
                                      int(kind), 0, ptr(losses, f64p)))
        return losses

    def step_stats(self, K: int) -> np.ndarray:
        """u64[K, 8] rows (STAT_UNIQUE, EDGES, INNER, SEEDS, HITS, MISSES, BAD_SEEDS, POSITIONS) of the
        last steps call."""
        out = np.zeros((K, STEP_STATS), dtype=np.uint64)
        check(lib().a3g_trainer_step_stats(self.h, ptr(out, u64p), K))
        return out

    def evaluate_full_graph(self) -> float:
        """trainer.cpp:241-303 on the device with the current weights."""
        m = np.ascontiguousarray(self.g.test_mask, dtype=np.uint8)
        acc = C.c_double()
        check(lib().a3g_evaluate_full_graph(self.h, ptr(m, u8p), C.byref(acc)))
        return acc.value

    def last_grads(self):
        gw1 = np.empty(self.spec.feat_dim * self.spec.hidden_dim)
        gw2 = np.empty(self.spec.hidden_dim * self.spec.num_classes)
        check(lib().a3g_trainer_last_grads(self.h, ptr(gw1, f64p), ptr(gw2, f64p)))
        return gw1, gw2

    def last_forward(self, max_inner: int):
        F, H, Cc = self.spec.feat_dim, self.spec.hidden_dim, self.spec.num_classes
        ni = C.c_uint64()
        logits = np.empty(self.max_seeds * Cc)
        agg_inner = np.empty(max_inner * F)
        h1 = np.empty(max_inner * H)
        agg_outer = np.empty(self.max_seeds * H)
        check(lib().a3g_trainer_last_forward(self.h, C.byref(ni), ptr(logits, f64p), ptr(agg_inner, f64p),
                                             ptr(h1, f64p), ptr(agg_outer, f64p)))
        n = ni.value
        return dict(n_inner=n, logits=logits, agg_inner=agg_inner[:n * F].reshape(n, F),
                    h1=h1[:n * H].reshape(n, H), agg_outer=agg_outer)

    def set_tier_accounting(self, on: bool):
        check(lib().a3g_trainer_set_tier_accounting(self.h, 1 if on else 0))

    def tier_rows(self) -> np.ndarray:
        """u64[16]: distinct rows the fused gather read per store tier over the
        last steps call (tier r < 15: HBM shard of rank r; 15: pinned host)."""
        out = np.zeros(16, dtype=np.uint64)
        check(lib().a3g_trainer_tier_rows(self.h, ptr(out, u64p)))
        return out

    def gemm_timing(self):
        """Average ms of the tcgen05 h1 / dW1 GEMMs of the last steps call."""
        a, b, n = C.c_double(), C.c_double(), C.c_uint64()
        check(lib().a3g_trainer_gemm_timing(self.h, C.byref(a), C.byref(b), C.byref(n)))
        return dict(h1_ms=a.value, dw1_ms=b.value, launches=n.value)

    def timing(self):
        t, a, b, l = C.c_double(), C.c_double(), C.c_double(), C.c_uint64()
        check(lib().a3g_trainer_timing(self.h, C.byref(t), C.byref(a), C.byref(b), C.byref(l)))
        return dict(total_ms=t.value, agg_ms=a.value, agg_bytes=b.value, launches_per_step=l.value)


class Comm:
    """NCCL communicator for the data-parallel gradient sum."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int, device: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = vp()
        check(lib().a3g_comm_create(buf, nranks, rank, device, C.byref(h)))
        self.h = h

    @classmethod
    def host(cls, nranks: int, rank: int, allreduce) -> "Comm":
        """Host-transport communicator (a3g_comm_create_host): `allreduce(buf)`
        receives the packed f32 gradient buffer as a numpy view over pinned
        host memory and must sum it in place over all ranks (gloo, MPI, ...)."""
        self = cls.__new__(cls)
        proto = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_float), C.c_size_t, C.c_void_p)

        def _cb(buf, count, _user):
            try:
                allreduce(np.ctypeslib.as_array(buf, shape=(count,)))
                return 0
            except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
                import traceback
                traceback.print_exc()
                return 1

        self._cb = proto(_cb)  # kept alive with the communicator
        h = vp()
        check(lib().a3g_comm_create_host(nranks, rank, C.cast(self._cb, vp), None, C.byref(h)))
        self.h = h
        return self

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().a3g_comm_unique_id(buf))
        return bytes(buf)

    def __del__(self):
        try:
            if self.h:
                lib().a3g_comm_destroy(self.h)
        except Exception:
            pass


@dataclass
class TrainOptions:
    """trainer.hpp:85-92 (u = 1: the B200 path is the single-worker algorithm;
    data parallelism is across GPUs)."""
    batch_size: int = 64
    epochs: int = 10
    u: int = 1
    model_seed: int = 1
    reference_accuracy: float = None


@dataclass
class TrainReport:
    """trainer.hpp:94-103."""
    test_accuracy: float = 0.0
    epochs_run: int = 0
    loss_curve: list = None
    accuracy_drop: float = float("nan")
    epoch_hit_rates: list = None
    max_batch_bytes: int = 0
    max_activation_bytes: int = 0
    param_bytes: int = 0


def train(g: Graph, spec: ModelSpec, sampler_cfg, cache: CacheState, opts: TrainOptions, device: int = 0,
          placement=None, feat_dtype: int = 0) -> TrainReport:
    """train::train (trainer.cpp:350-424) with every step on the device: per
    epoch the reference's batch plan (plan seed hash2(rng_seed, 0)) and step
    seeds sampling_seed(rng_seed, epoch, step, 0) run through the CUDA-stream
    pipeline; loss curve, epoch hit rates, max batch/activation bytes and the
    final full-graph accuracy as the reference reports them."""
    if opts.batch_size < 1:
        raise ParameterError("train: batch_size must be >= 1")
    if opts.u != 1:
        raise ConfigError("train: partitioned workers (u > 1) are not part of the B200 path; "
                          "use data parallelism across GPUs")
    tn = g.train_nodes
    if len(tn) == 0:
        raise ConfigError("train: a worker has no train nodes")
    spec = ModelSpec(spec.feat_dim, spec.hidden_dim, spec.num_classes, spec.num_layers, spec.learning_rate)
    tr = Trainer(g, cache, spec, sampler_cfg.fanouts, max_seeds=min(opts.batch_size, len(tn)),
                 model_seed=opts.model_seed, device=device, feat_dtype=feat_dtype, placement=placement)
    rep = TrainReport(loss_curve=[], epoch_hit_rates=[], param_bytes=spec.param_bytes(), epochs_run=opts.epochs)
    F, H, Cc = spec.feat_dim, spec.hidden_dim, spec.num_classes
    for epoch in range(opts.epochs):
        order = plan_epoch_order(tn, epoch, hash2(sampler_cfg.rng_seed, 0))  # trainer.cpp:378-379
        steps = (len(order) + opts.batch_size - 1) // opts.batch_size
        off = np.minimum(np.arange(steps + 1, dtype=np.uint64) * opts.batch_size, len(order)).astype(np.uint64)
        rs = [sampling_seed(sampler_cfg.rng_seed, epoch, s, 0) for s in range(steps)]
        losses = tr.steps_v(order, off, rs, sampler_cfg.bias_rate, sampler_cfg.kind)
        st = tr.step_stats(steps).astype(np.int64)
        rep.loss_curve.append(float(losses.mean()) if steps else 0.0)
        h, m = int(st[:, STAT_HITS].sum()), int(st[:, STAT_MISSES].sum())
        rep.epoch_hit_rates.append(h / (h + m) if h + m else 0.0)
        bb = st[:, STAT_UNIQUE] * F * 4 + st[:, STAT_EDGES] * 8   # cache.cpp:84
        ab = (st[:, STAT_INNER] * (F + H) + st[:, STAT_SEEDS] * (H + Cc)) * 4  # trainer.cpp:134-135
        rep.max_batch_bytes = max(rep.max_batch_bytes, int(bb.max()))
        rep.max_activation_bytes = max(rep.max_activation_bytes, int(ab.max()))
    rep.test_accuracy = tr.evaluate_full_graph()
    if opts.reference_accuracy is not None:
        rep.accuracy_drop = opts.reference_accuracy - rep.test_accuracy
    return rep
