"""Multi-GPU data plane, exercised on ONE B200 with two processes
(trainer.cpp:213-229, test_trainer.cpp:210-253):

* device data parallelism at world 2: each rank runs the whole device step
  on its shard of the global batch (same step seed), the packed
  [n_k dW1 | n_k dW2 | n_k | n_k loss] buffer is summed across the ranks
  through the host-transport communicator (a3g_comm_create_host over
  torch.distributed gloo -- NCCL refuses two ranks on one GPU) and k_sgd
  applies the union-batch step. The trajectory must equal one process
  training on the union batch (fp32 reassociation only), and the oracle's
  single-worker union-batch trajectory within 1e-3;
* the cross-process NVLink-peer feature store: two processes each own a
  rank%2 shard of the cached rows (A3G_STORE_SHARDED), exchange cudaIpc
  handles (a3g_store_ipc_handle / a3g_store_open_peer) and train
  BIT-identically to a single process with the whole table in HBM.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu
N, F, B, K, H = 100_000, 128, 1024, 4, 16


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(rank, world, port):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _graph():
    from paper_2511_07421_b200 import cache as CA, graph as G
    g = G.generate_power_law(N, 3, 2.5, F, 1)
    cache = CA.build_static_cache(g, CA.CacheConfig(int(0.2 * N) * F * 4, 2))
    return g, cache


def _dp_worker(rank, world, port, out):
    _setup(rank, world, port)
    from paper_2511_07421_b200 import dp, train as T
    g, cache = _graph()
    gb, gs = dp.global_batches(g.train_nodes, B // world, world, K)
    tr = T.Trainer(g, cache, T.ModelSpec(F, H, 4), [10, 5], max_seeds=B // world)

    def allreduce(buf):
        t = torch.from_numpy(buf)  # shares the pinned host buffer
        dist.all_reduce(t, op=dist.ReduceOp.SUM)

    comm = T.Comm.host(world, rank, allreduce)
    tr.set_comm(comm)
    mine = np.stack([dp.shard_of(b, rank, world) for b in gb])
    losses = tr.steps(mine, gs, 8.0, 0)
    w1, w2 = tr.get_weights()
    if rank == 0:
        np.savez(out, losses=losses, w1=w1, w2=w2)
    dist.barrier()
    tr.set_comm(None)
    dist.destroy_process_group()


def test_device_dp_world2_equals_union_batch(tmp_path):
    import oracle
    from paper_2511_07421_b200 import dp, train as T
    out = str(tmp_path / "dp.npz")
    mp.start_processes(_dp_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn", join=True)
    got = np.load(out)
    g, cache = _graph()
    gb, gs = dp.global_batches(g.train_nodes, B // 2, 2, K)
    one = T.Trainer(g, cache, T.ModelSpec(F, H, 4), [10, 5], max_seeds=B)
    la = one.steps(gb, gs, 8.0, 0)
    w1, w2 = one.get_weights()
    np.testing.assert_allclose(got["losses"], la, rtol=1e-5)
    for a, b in ((got["w1"], w1), (got["w2"], w2)):
        assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b)
    # the oracle's single-worker trajectory on the union batches (fp64)
    orc = oracle.Oracle()
    ow1, ow2 = T.init_model(T.ModelSpec(F, H, 4), 1)
    ref = orc.train_steps(g, [10, 5], 8.0, 0, 1, B, H, 4, 0.2, ow1, ow2, K, cache.device_map)
    np.testing.assert_allclose(got["losses"], ref["losses"], rtol=1e-3)
    assert np.linalg.norm(got["w1"] - ref["w1"]) <= 1e-3 * np.linalg.norm(ref["w1"])


def _ipc_worker(rank, world, port, out):
    _setup(rank, world, port)
    from paper_2511_07421_b200 import dp, graph as G, train as T
    g, cache = _graph()
    tr = T.Trainer(g, cache, T.ModelSpec(F, H, 4), [10, 5], max_seeds=B,
                   placement=dict(policy=G.STORE_SHARDED, rank=rank, nranks=world))
    handles = [None] * world
    dist.all_gather_object(handles, tr.store.ipc_handle())
    for r in range(world):
        if r != rank:
            tr.store.open_peer(r, handles[r])
    info = tr.store.info()
    dist.barrier()  # every peer mapped before anyone reads
    gb, gs = dp.global_batches(g.train_nodes, B, 1, K)
    losses = tr.steps(gb, gs, 8.0, 0)
    w1, w2 = tr.get_weights()
    dist.barrier()  # nobody frees a shard another rank still reads
    if rank == 0:
        np.savez(out, losses=losses, w1=w1, w2=w2, info=np.array([info["local_rows"], info["remote_rows"],
                                                                   info["host_rows"]]))
    dist.barrier()
    dist.destroy_process_group()


def test_ipc_peer_store_two_processes_bit_identical(tmp_path):
    from paper_2511_07421_b200 import dp, train as T
    out = str(tmp_path / "ipc.npz")
    mp.start_processes(_ipc_worker, args=(2, _free_port(), out), nprocs=2, start_method="spawn", join=True)
    got = np.load(out)
    g, cache = _graph()
    local, remote, host = got["info"]
    assert local > 0 and remote > 0 and local + remote == cache.total_cached() and host == N - local - remote
    gb, gs = dp.global_batches(g.train_nodes, B, 1, K)
    one = T.Trainer(g, cache, T.ModelSpec(F, H, 4), [10, 5], max_seeds=B)
    la = one.steps(gb, gs, 8.0, 0)
    w1, w2 = one.get_weights()
    assert np.array_equal(got["losses"], la)
    assert np.array_equal(got["w1"], w1) and np.array_equal(got["w2"], w2)
