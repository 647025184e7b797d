"""Data-parallel host logic over torch.distributed gloo, world_size 2, on CPU
(the multi-GPU path of DESIGN.md section 6 with the device step replaced by
the oracle): each rank samples and differentiates its shard of the global
batch with the same step seed, packs [n_k dW1 | n_k dW2 | n_k | n_k loss],
all-reduces with gloo and unpacks -- the result must equal the oracle's
single-worker step on the union batch (test_trainer.cpp:210-253)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from helpers import golden_graph, load_golden  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_grads(orc, g, dm, seeds, step_seed, w1, w2, H, C):
    b = orc.sample_khop(g, seeds, [10, 5], 8.0, 0, step_seed, dm)
    ref = orc.grad_on_edges(g.feat_dim, H, C, w1, w2, len(b.unique_nodes), b.num_seed_unique, b.layers,
                            g.features[b.unique_nodes], g.labels[b.unique_nodes[:b.num_seed_unique]])
    return ref, b.num_seed_unique


def _worker(rank, world, port, out_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import oracle
    from helpers import golden_graph, load_golden
    from paper_2511_07421_b200 import dp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.Oracle()
    rec = load_golden("pl3000")
    g = golden_graph(rec)
    dm = rec["train_device_map"]
    H, C = 8, 4
    w1, w2 = orc.init_model(g.feat_dim, H, C, 1)
    gbatch, sseeds = dp.global_batches(g.train_nodes, 64, world, 3)
    res = []
    for step in range(len(gbatch)):
        mine = dp.shard_of(gbatch[step], rank, world)
        ref, n_k = _rank_grads(orc, g, dm, mine, int(sseeds[step]), w1, w2, H, C)
        buf = torch.from_numpy(dp.pack(ref["gw1"], ref["gw2"], n_k, ref["loss"]))
        dist.all_reduce(buf, op=dist.ReduceOp.SUM)
        gw1, gw2, loss = dp.unpack(buf.numpy(), len(ref["gw1"]))
        res.append((gw1, gw2, loss))
    if rank == 0:
        np.save(out_path, np.array([np.concatenate([a, b, [l]]) for a, b, l in res]))
    dist.barrier()
    dist.destroy_process_group()


def test_dp_gloo_world2_equals_union_batch(tmp_path):
    import oracle
    from paper_2511_07421_b200 import dp
    out = str(tmp_path / "dp.npy")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn", join=True)
    got = np.load(out)
    orc = oracle.Oracle()
    rec = load_golden("pl3000")
    g = golden_graph(rec)
    w1, w2 = orc.init_model(g.feat_dim, 8, 4, 1)
    gbatch, sseeds = dp.global_batches(g.train_nodes, 64, 2, 3)
    for step in range(len(gbatch)):
        ref, _ = _rank_grads(orc, g, rec["train_device_map"], gbatch[step], int(sseeds[step]), w1, w2, 8, 4)
        want = np.concatenate([ref["gw1"], ref["gw2"], [ref["loss"]]])
        np.testing.assert_allclose(got[step], want, rtol=1e-10, atol=1e-15)


def test_shards_partition_the_global_batch():
    from paper_2511_07421_b200 import dp
    gb = np.arange(1000, dtype=np.uint32)
    for world in (1, 2, 4, 8):
        parts = [dp.shard_of(gb, r, world) for r in range(world)]
        assert np.array_equal(np.concatenate(parts), gb)
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
