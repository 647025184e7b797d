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

from ._lib import ParameterError, check, f64p, lib, ptr, u32p, u64p, vp
from .cache import CacheState
from .graph import Graph
from .sampling import SamplerKind


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


def sgd_step(w: np.ndarray, g: np.ndarray, lr: float) -> None:
    """trainer.cpp:208-211 (host arrays)."""
    w += (-lr) * g


def sync_gradients(grads):
    """trainer.cpp:213-229: element-wise mean of a list of (gw1, gw2)."""
    if not grads:
        raise ParameterError("sync_gradients: empty gradient list")
    s1 = np.zeros_like(grads[0][0])
    s2 = np.zeros_like(grads[0][1])
    for a, b in grads:
        if a.shape != s1.shape or b.shape != s2.shape:
            raise ParameterError("sync_gradients: shape mismatch")
        s1 += a
        s2 += b
    inv = 1.0 / len(grads)
    return s1 * inv, s2 * inv


class Trainer:
    """Device-resident 2-layer mean-GCN trainer (trainer.hpp:24-60, 63-83)."""

    def __init__(self, g: Graph, cache: CacheState, spec: ModelSpec, fanouts, max_seeds: int,
                 model_seed: int = 1, device: int = 0, feat_dtype: int = 0):
        if spec.feat_dim != g.feat_dim:
            raise ParameterError("trainer: spec.feat_dim != graph feat_dim")
        self.g, self.cache, self.spec = g, cache, spec
        self.fanouts = [int(x) for x in fanouts]
        if any(x < 1 for x in self.fanouts):
            raise ParameterError("sample_khop: fanout must be >= 1")
        f = np.asarray(self.fanouts, dtype=np.uint32)
        dg = g.device(device, feat_dtype)
        h = vp()
        check(lib().a3g_trainer_create(dg.h, cache.device(g, device, feat_dtype), max_seeds, ptr(f, u32p), len(f),
                                       spec.hidden_dim, spec.num_classes, spec.learning_rate, model_seed,
                                       C.byref(h)))
        self.h = h
        self.max_seeds = max_seeds
        self._keep = [dg]

    def __del__(self):
        try:
            if self.h:
                lib().a3g_trainer_destroy(self.h)
        except Exception:
            pass

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
