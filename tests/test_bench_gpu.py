"""bench.py end to end on the B200: the one-GPU JSON line carries the contract
keys, and the N > 1 path (torchrun, sharded feature store over cudaIpc, the
gradient allreduce) runs with two ranks sharing the one GPU through the
host-transport communicator (NCCL refuses two ranks on one device) -- a
functional check of the multi-process bench, not a scaling number."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _json_line(out):
    lines = [l for l in out.strip().splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_one_gpu_contract_keys():
    r = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "5", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _json_line(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.5


def test_bench_two_ranks_sharded_store_host_comm():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--config", "c1", "--steps",
           "5", "--warmup", "3", "--no-cpu-baseline", "--comm", "host", "--share-device", "--store", "sharded"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    d = _json_line(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["store"] == "sharded" and d["config"]["parallelism"] == "dp2"
    assert d["config"]["global_batch"] == 2 * d["config"]["batch_per_gpu"]
    res = d["roofline"]["resources"]
    assert "hbm_local" in res and "nvlink_peer" in res  # the other rank's shard is read through the peer path


def test_bench_two_ranks_default_placement_replicates():
    """--store auto at N > 1: the table fits one GPU, so every rank holds it (weak scaling moves
    only the gradient allreduce between GPUs)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--config", "c1", "--steps",
           "5", "--warmup", "3", "--no-cpu-baseline", "--comm", "host", "--share-device"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    d = _json_line(r.stdout)
    assert d["n_gpus"] == 2 and d["config"]["store"] == "hbm" and d["value"] > 0
