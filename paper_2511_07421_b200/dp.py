"""Data parallelism across GPUs.

One process per GPU. Every rank holds the full CSR; rank r trains the
contiguous shard [r*B, (r+1)*B) of each global batch of N*B seeds, with the
step seed sampling_seed(base, epoch, step, 0) shared by all ranks. The only
exchange per step is an allreduce(sum) of [n_k*dW1 | n_k*dW2 | n_k | n_k*loss]
followed by division by sum(n_k) -- on the device that is k_scale_for_sync ->
ncclAllReduce -> k_sgd (train.cu, comm.cpp). Because the reference's forward
is separable per seed and its scatter / dW1 are linear (test_trainer.cpp:210-
253), the result equals the reference's single-worker step on the union batch.

The reference's own train(u > 1) partitions the graph and re-keys the RNG
with partition-local ids (trainer.cpp:356-359) -- a different algorithm,
out of scope.
"""
from __future__ import annotations

import numpy as np

from . import train as T


def shard_of(global_seeds, rank: int, world: int) -> np.ndarray:
    """Rank's contiguous shard of one global batch (equal shards; the last
    ranks get the remainder short, like np.array_split)."""
    return np.array_split(np.asarray(global_seeds, dtype=np.uint32), world)[rank]


def global_batches(train_nodes, batch_per_rank: int, world: int, steps: int, base_seed: int = 1, offset: int = 0):
    """Global batches of world * batch_per_rank seeds over consecutive steps:
    the reference's epoch plan (trainer.cpp:330-343, plan seed
    hash2(base, 0)) re-cut at the global batch size, plus the step seeds
    sampling_seed(base, epoch, step, 0) (trainer.cpp:345-348)."""
    gb = batch_per_rank * world
    per_epoch = len(train_nodes) // gb
    if per_epoch < 1:
        raise ValueError("global batch larger than the train set")
    plans, out, seeds = {}, [], []
    for i in range(offset, offset + steps):
        e, s = divmod(i, per_epoch)
        if e not in plans:
            plans[e] = T.plan_epoch_order(train_nodes, e, T.hash2(base_seed, 0))
        out.append(plans[e][s * gb:(s + 1) * gb])
        seeds.append(T.sampling_seed(base_seed, e, s, 0))
    return np.stack(out), np.array(seeds, dtype=np.uint64)


def pack(gw1, gw2, n_k: int, loss: float) -> np.ndarray:
    """The allreduce buffer of one rank: n_k-weighted gradients, n_k, n_k*loss
    (the layout of the device's d_gw, trainer.cuh)."""
    return np.concatenate([n_k * np.asarray(gw1, np.float64).ravel(), n_k * np.asarray(gw2, np.float64).ravel(),
                           [float(n_k), n_k * float(loss)]])


def unpack(buf: np.ndarray, n1: int):
    """Summed buffer -> (dW1, dW2, loss) of the union batch."""
    n = buf[-2]
    return buf[:n1] / n, buf[n1:-2] / n, buf[-1] / n
