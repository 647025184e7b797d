"""bench.py -- trained seed nodes/sec of the A3GNN data-parallel mini-batch hot
path on B200 (BASELINE.json metric), one JSON line on rank 0.

A step = one batch of the workload through the whole path:
  k-hop locality-aware sampling -> cached feature gather + mean aggregation ->
  2-layer mean-GCN forward/backward -> [NCCL allreduce] -> SGD.
Default workload = BASELINE.json configs[1] (Reddit-shaped synthetic graph,
233K nodes / 112.8M edges, 602-d f32 features, fanout [15,10,5], batch 1024
per GPU, full feature cache), generated bit-identically to the reference's
generate_power_law(233000, 165, 2.5, 602, seed 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
For N>1 launch under torchrun (one rank per GPU, NCCL).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

# nine CUDA streams drive the pipeline: more hardware work queues than the
# default 8 keep them from serialising behind each other (set before any CUDA
# context exists; liba3g_b200.so asks for the same when it loads first)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, min_degree, feat_dim, fanouts, batch, cache_frac, description)
    "c2": (233_000, 165, 602, [15, 10, 5], 1024, 1.0,
           "reddit-shaped synthetic 233K nodes / 112.8M edges, 602-d f32, fanout [15,10,5], batch 1024/GPU, "
           "full feature cache"),
    "c1": (100_000, 3, 128, [10, 5], 1024, 0.2,
           "power-law synthetic 100K nodes / 0.9M edges, 128-d f32, fanout [10,5], batch 1024/GPU, 20% cache "
           "(the sampling bias set; feature placement per --store)"),
    "c3": (2_450_000, 9, 100, [15, 10, 5], 4096, 0.2,
           "ogbn-products-shaped synthetic 2.45M nodes / 65M edges, 100-d f32, fanout [15,10,5], batch 4096/GPU, "
           "20% cache (the sampling bias set; feature placement per --store)"),
    # papers-scale: topology from the host generator at feat_dim 1, the 128-d
    # features synthesized on the device in bf16 (a3g_graph_synthesize_features)
    "c5": (111_000_000, 5, 128, [15, 10, 5], 8192, 0.2,
           "ogbn-papers100M-shaped synthetic 111M nodes / 1.6B edges, 128-d bf16 (device-synthesized), "
           "fanout [15,10,5], batch 8192/GPU, 20% cache (the sampling bias set; feature placement per --store: "
           "--store cache = the stated 20% in HBM with pinned-host spill)"),
}
SYNTH = {"c5"}  # configs whose features are synthesized on the device (bf16)
HIDDEN, CLASSES, LR, BASE_SEED = 16, 4, 0.2, 1


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)  # ~35 ms at C2: past the 8-deep pipeline ramp
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=list(CONFIGS), default="c2")
    p.add_argument("--gamma", type=float, default=8.0)
    p.add_argument("--hidden", type=int, default=HIDDEN,
                   help="hidden width H (reference default 16, config.hpp:51; > 16 puts h1 and dW1 on tcgen05)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-units", type=int, default=3, help="batches in the bounded cpu_baseline sample")
    p.add_argument("--pipeline", type=int, default=None, help="sampling streams (0 = sequential; default: library's)")
    p.add_argument("--comm", choices=["nccl", "host"], default="nccl",
                   help="gradient allreduce at N>1: NCCL over NVLink (default), or the host-transport "
                        "communicator over gloo (a3g_comm_create_host) -- with --share-device, N ranks on one GPU "
                        "exercise the multi-process path where NCCL cannot (functional check, not a scaling number)")
    p.add_argument("--share-device", action="store_true",
                   help="every rank uses cuda:0 (multi-process functional check on a one-GPU box)")
    p.add_argument("--store", choices=["auto", "hbm", "cache", "sharded"], default="auto",
                   help="feature placement (DESIGN.md 5): hbm = whole table replicated in each GPU's HBM; cache = "
                        "cached rows in HBM, misses in pinned host memory (zero-copy PCIe); sharded = rank r holds "
                        "the rows the cache places on device r, peers read over NVLink (cudaIpc), misses on the "
                        "host. auto: hbm (replicated) whenever the table fits in a quarter of one GPU's HBM -- "
                        "every BASELINE config does, even C5's 28 GB of bf16 rows -- so weak scaling moves no "
                        "feature bytes over NVLink; sharded otherwise")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_tflops():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f).get("bf16_tflops", 1590.0))
    return 1590.0


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML polled
    every ~2 ms from a thread (the timed region of a short run is tens of ms,
    below nvidia-smi's sampling period); nvidia-smi is the fallback."""
    NAMES = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.sm, self.mx, self.reasons = [], None, set()
        self.stop = threading.Event()
        self.t = None

    def _poll(self):
        import pynvml
        h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
        get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        self.mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while True:
            self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            r = get_r(h)
            for name, bit in self.NAMES.items():
                if r & bit:
                    self.reasons.add(name)
            if self.stop.wait(0.002):
                break

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def _smi(self):  # fallback without NVML bindings: nvidia-smi at its fastest period
        try:
            self._smi_loop()
        except Exception:
            pass

    def _smi_loop(self):
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits", "-lms", "20"],
                                     stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 6 and p[0].replace(".", "").isdigit():
                self.sm.append(float(p[0]))
                self.mx = float(p[1]) if p[1].replace(".", "").isdigit() else self.mx
                self.reasons.update(n for n, v in zip(names, p[2:6]) if v.lower() == "active")

    def __enter__(self):
        self.proc = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.t = threading.Thread(target=self._poll, daemon=True)
        except Exception:
            self.t = threading.Thread(target=self._smi, daemon=True)
        self.t.start()
        time.sleep(0.005)  # first sample lands inside the region
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml"}


def make_graph(cfg_name):
    from paper_2511_07421_b200 import graph as G
    n, m, F, fan, B, frac, _ = CONFIGS[cfg_name]
    return G.generate_power_law(n, m, 2.5, 1 if cfg_name in SYNTH else F, BASE_SEED)


NVLINK_PEER_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md; 900 nominal)


def measure_pcie_h2d_gbs(device: int) -> float:
    """Pinned host -> device copy bandwidth on this box (best of 5, 256 MiB,
    CUDA events): the ceiling of the zero-copy miss path."""
    import torch
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def host_cpu():
    """nproc and the CPU model of this host (printed beside the CPU numbers)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return n, model


def cpu_reference_run(rg, cfg_name, gamma, units, mode, producers, warmup=1, hidden=HIDDEN):
    """Time the reference's own CPU path (oracle/_ref: the unmodified reference
    compiled in place) on `units` batches of the workload after `warmup`
    untimed ones, scheduled as the executor's `mode` (0 sequential, 1 pmode1,
    2 pmode2; pipeline_exec.cpp:219-276) over the reference's per-batch
    functions. `rg` is a graph held by the reference library."""
    import oracle
    n, m, F, fan, B, frac, _ = CONFIGS[cfg_name]
    ref = oracle.RefLib()
    dm = ref.build_static_cache(rg, int(frac * n) * F * 4, 1)
    secs, seeds = ref.bench_steps(rg, dm, fan, gamma, BASE_SEED, B, hidden, CLASSES, LR, units, producers, 8,
                                  warmup=warmup, mode=mode)
    return dict(seconds=secs, seeds=seeds, seeds_per_s=seeds / secs if secs > 0 else 0.0, units=units,
                mode=["sequential", "pmode1", "pmode2"][mode], threads=1 if mode == 0 else producers + 1)


def run_reference(args):
    """The reference arm: the reference's own CPU implementation (oracle/_ref,
    compiled in place from /root/reference's sources), on its OWN generator's
    graph -- this process never imports or loads the B200 package."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    n, m, F, fan, B, frac, desc = CONFIGS[args.config]
    import oracle
    cores, cpu_model = host_cpu()
    base = {"metric": "trained seed nodes/sec", "unit": "seeds/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "dtype": "f64", "data": "synthetic (the reference's generate_power_law, seed 1)", "vs_baseline": None,
            "config": {"workload": args.config, "description": desc, "global_batch": B, "fanouts": fan,
                       "gamma": args.gamma, "hidden": args.hidden, "classes": CLASSES}}
    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (reference compiled in place) not built"}))
        return 0
    if args.config in SYNTH:
        print(json.dumps({"impl": "reference", "unavailable": "papers-scale config: the reference generator needs "
                          "~30 min and 22.6 GB at F=1 (SURVEY 8(c)(iv)); not a bounded sample"}))
        return 0
    ref = oracle.RefLib()
    t0 = time.time()
    rg = ref.power_law(n, m, 2.5, F, BASE_SEED)  # generators.cpp:79-149, the reference's own
    gen_s = time.time() - t0
    producers = max(1, cores - 1)
    K, W = max(1, args.steps), max(0, args.warmup)
    # headline: the executor's pmode1 schedule, nproc-1 producers + the trainer thread, queue 8
    r1 = cpu_reference_run(rg, args.config, args.gamma, K, 1, producers, warmup=W, hidden=args.hidden)
    # beside it (bounded): pmode2 and the 1-thread sequential train() loop
    r2 = cpu_reference_run(rg, args.config, args.gamma, max(1, min(K, 8)), 2, producers, warmup=1, hidden=args.hidden)
    r0 = cpu_reference_run(rg, args.config, args.gamma, max(1, min(K, 3)), 0, 0, warmup=1, hidden=args.hidden)
    v = r1["seeds_per_s"]
    base.update({"value": v, "ms_per_step": 1e3 * r1["seconds"] / max(1, r1["units"]),
                 "cpu_baseline": {"value": v, "unit": "seeds/s", "cores": cores, "cpu_model": cpu_model,
                                  "kind": "reference",
                                  "sample": f"{K} consecutive batches of epoch 0 after {W} untimed, executor pmode1 "
                                            f"schedule (pipeline_exec.cpp:229-276) over the reference's sample_khop/"
                                            f"retrieve_features/forward/backward/sync_gradients/sgd_step, "
                                            f"{producers} producer threads + 1 trainer thread, queue 8"},
                 "cpu_modes": {k: {"seeds_per_s": r["seeds_per_s"], "batches": r["units"], "threads": r["threads"]}
                               for k, r in (("pmode1", r1), ("pmode2", r2), ("sequential_1thread", r0))},
                 "graph_gen_s": round(gen_s, 1),
                 "e2e": {"value": v, "unit": "seeds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(base))
    return 0


def run_ours(args):
    rank, world, local = dist_env()
    import torch
    if args.share_device:
        local = 0
    torch.cuda.set_device(local)
    host_comm = world > 1 and args.comm == "host"
    if world > 1:
        import torch.distributed as dist
        if host_comm:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2511_07421_b200 import cache as CA, train as T
    n, m, F, fan, B, frac, desc = CONFIGS[args.config]
    t0 = time.time()
    g = make_graph(args.config)
    gen_s = time.time() - t0
    synth = args.config in SYNTH
    Fh = 1 if synth else F  # host feat_dim (the cache's node_cost, cache.cpp:20, scales the same set)
    table_bytes = n * F * (2 if synth else 4)
    hbm_bytes = torch.cuda.get_device_properties(local).total_memory
    store = args.store if args.store != "auto" else ("hbm" if world == 1 or table_bytes * 4 <= hbm_bytes
                                                     else "sharded")
    from paper_2511_07421_b200 import graph as Gm
    # Appendix B: the ratio is the aggregate cached fraction; per-device volume
    # ratio*n*F*4/N over N devices caches the same set for every N
    ndev = world if store == "sharded" else 1
    cache = CA.build_static_cache(g, CA.CacheConfig(int(frac * n) * Fh * 4 // ndev, ndev), device=local)
    placement = None
    if store == "cache":
        placement = dict(policy=Gm.STORE_CACHE)
    elif store == "sharded":
        placement = dict(policy=Gm.STORE_SHARDED, rank=rank, nranks=world)
    H = args.hidden
    tr = T.Trainer(g, cache, T.ModelSpec(F, H, CLASSES, learning_rate=LR), fan, max_seeds=B, device=local,
                   feat_dtype=1 if synth else 0, synth_seed=BASE_SEED if synth else None, placement=placement)
    if store == "sharded" and world > 1:  # peer shards over NVLink: exchange cudaIpc handles
        import torch.distributed as dist
        handles = [None] * world
        dist.all_gather_object(handles, tr.store.ipc_handle())
        for r in range(world):
            if r != rank:
                tr.store.open_peer(r, handles[r])
        dist.barrier()
    comm = None
    if host_comm:
        import torch.distributed as dist

        def _allreduce(buf):
            dist.all_reduce(torch.from_numpy(buf), op=dist.ReduceOp.SUM)

        comm = T.Comm.host(world, rank, _allreduce)
        tr.set_comm(comm)
    elif world > 1:
        import torch.distributed as dist
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(T.Comm.unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        comm = T.Comm(bytes(uid.cpu().numpy().tobytes()), world, rank, local)
        tr.set_comm(comm)
    W, K = args.warmup, args.steps
    # the library's default depth (trainer.cuh): 12 sampling streams for batches of <= 2048 seeds, else 8
    pipe = args.pipeline if args.pipeline is not None else (12 if B <= 2048 else 8)
    tr.set_pipeline(pipe)
    from paper_2511_07421_b200 import dp
    gbatches, gseeds = dp.global_batches(g.train_nodes, B, world, W + 3 * K, BASE_SEED)
    mine = np.ascontiguousarray(np.stack([dp.shard_of(gb, rank, world) for gb in gbatches]))
    # ---- warmup (untimed)
    tr.steps(mine[:W], gseeds[:W], args.gamma, 0)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # ---- timed: inputs resident in HBM (device seeds), device time via events
    dev_seeds = torch.from_numpy(mine[W:W + K].astype(np.int32)).cuda()
    barrier()
    with ClockSampler(local) as clk:
        losses = _steps_device(tr, dev_seeds, gseeds[W:W + K], args.gamma)
        barrier()
    tm = tr.timing()
    dev_ms = tm["total_ms"]
    st_dev = tr.step_stats(K)
    # ---- e2e: host seeds through the C-ABI (H2D in the region, losses D2H)
    barrier()
    t1 = time.perf_counter()
    losses_e2e = tr.steps(mine[W + K:W + 2 * K], gseeds[W + K:W + 2 * K], args.gamma, 0)
    barrier()
    e2e_s = time.perf_counter() - t1
    tm2 = tr.timing()
    # ---- roofline leg: the same K-step call in sequential mode (one stream, the
    # reference's Mode::sequential), so k_agg1's event window holds k_agg1 alone;
    # the pipelined run's k_agg1 shares the SMs with the concurrent sampling streams.
    barrier()
    tr.set_pipeline(0)
    tr.set_tier_accounting(True)  # distinct rows per store tier, counted after k_agg1's events
    dev_seq = torch.from_numpy(mine[W + 2 * K:W + 3 * K].astype(np.int32)).cuda()
    _steps_device(tr, dev_seq, gseeds[W + 2 * K:W + 3 * K], args.gamma)
    barrier()
    tm3 = tr.timing()
    gt3 = tr.gemm_timing()
    st3 = tr.step_stats(K)
    tiers = tr.tier_rows()
    tr.set_tier_accounting(False)
    tr.set_pipeline(pipe)
    if world > 1:
        import torch.distributed as dist
        x = torch.tensor([dev_ms, e2e_s], dtype=torch.float64, device="cpu" if host_comm else "cuda")
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        dev_ms, e2e_s = float(x[0]), float(x[1])
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0
    seeds_total = world * B * K
    value = seeds_total / (dev_ms / 1e3)
    e2e = seeds_total / e2e_s
    hbm, peak_kind = measured_peaks()
    agg_ms, agg_bytes = tm3["agg_ms"], tm3["agg_bytes"]
    achieved = agg_bytes / (agg_ms * 1e-3) / 1e9 if agg_ms > 0 else 0.0
    pipe_ms = tm["agg_ms"]
    pipe_gbs = tm["agg_bytes"] / (pipe_ms * 1e-3) / 1e9 if pipe_ms > 0 else 0.0
    # per-resource roofline of the gather: distinct rows per tier
    # x row bytes per launch, over the same k_agg1 launch time
    esz = 2 if args.config in SYNTH else 4
    rows_local = int(tiers[rank if store == "sharded" else 0])
    rows_host = int(tiers[15])
    rows_peer = int(tiers[:15].sum()) - rows_local
    res = {}
    pcie = measure_pcie_h2d_gbs(local) if rows_host else None
    for name, rows, peak, kind in (("hbm_local", rows_local, hbm, peak_kind),
                                   ("nvlink_peer", rows_peer, NVLINK_PEER_GBS, "guide-measured peer copy"),
                                   ("pcie_host", rows_host, pcie, "measured pinned H2D on this box")):
        if rows == 0:
            continue
        b = rows * F * esz / K
        a = b / (agg_ms * 1e-3) / 1e9 if agg_ms > 0 else 0.0
        res[name] = {"bytes_per_launch": b, "achieved": a, "peak": peak, "peak_kind": kind,
                     "frac": a / peak if peak else None}
    bound = max(res, key=lambda k: res[k]["frac"] or 0.0) if res else None
    # the sampler's work: neighbour positions drawn per step (sum of frontier
    # degrees, one draw per neighbour, sampler.cpp:22-27) over the step time,
    # against the hash prefilter's measured ALU ceiling
    pos = float(st_dev[:, T.STAT_POSITIONS].mean())
    tpos = pos / (dev_ms / K * 1e-3) / 1e12 if dev_ms > 0 else 0.0
    sampler = {"positions_per_step": pos, "achieved_tpos_s": tpos, "ceiling_tpos_s": 1.37,
               "ceiling_kind": "measured hash-prefilter throughput, one B200 (tools/microbench/hash_pipes.cu)",
               "frac": tpos / 1.37,
               "note": "positions over the whole pipelined step time: the sampler shares the GPU with the gather "
                       "and the dense update"}
    # the dense update on the tensor cores (H > 16): algorithmic flops of
    # h1 = agg W1 and dW1 = agg^T G (2 n_inner F H each) over their launch time
    tensor = None
    if gt3["launches"]:
        n_inner = float(st3[:, T.STAT_INNER].mean())
        fl = 2 * 2.0 * n_inner * F * H
        ms = gt3["h1_ms"] + gt3["dw1_ms"]
        tf = fl / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
        peak_tf = measured_tflops()
        tensor = {"kernels": "k_h1_tc + k_dw1_tc (tcgen05.mma kind::f16, fp32 TMEM accumulators)", "bound": "tensor",
                  "flops_per_step": fl, "ms_per_step": ms, "h1_ms": gt3["h1_ms"], "dw1_ms": gt3["dw1_ms"],
                  "achieved": tf, "peak": peak_tf, "unit": "TFLOP/s", "frac": tf / peak_tf if peak_tf else None,
                  "mma_flops_issued_per_step": 6 * fl,
                  "note": "fp32 operands as 3 bf16 terms, 6 MMAs per product (fp32-class accuracy); the issued "
                          "tensor work is 6x the algorithmic flops"}
    traffic = None
    prof = os.path.join(ROOT, "profiles", "agg_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get(args.config)
    out = {
        "metric": "trained seed nodes/sec", "value": value, "unit": "seeds/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": dev_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if args.config in SYNTH else "f32", "data": "synthetic (generate_power_law, bit-identical to the reference generator)",
        "config": {"workload": args.config, "description": desc, "global_batch": world * B, "batch_per_gpu": B,
                   "fanouts": fan, "gamma": args.gamma, "model": f"2-layer mean-GCN (reference trainer), H={H}, C=4",
                   "hidden": H, "classes": CLASSES, "parallelism": f"dp{world}", "sampling_streams": pipe,
                   "store": store, "comm": ("host (gloo)" if host_comm else "nccl") if world > 1 else None,
                   "shared_device": bool(args.share_device),
                   "l2": "inputs larger than L2 (CSR %.0f MB + features %.0f MB)" % (
                       g.num_edges * 4 / 1e6, n * F * (2 if args.config in SYNTH else 4) / 1e6),
                   "graph_gen_s": round(gen_s, 1)},
        "roofline": {"kernel": "k_agg1 (fused feature gather + mean aggregation + h1 = relu(agg W1) epilogue)", "bound": "hbm",
                     "achieved": achieved, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "bytes_per_launch": agg_bytes,
                     "ms_per_launch": agg_ms,
                     "timed_in": f"{K} sequential-mode steps (k_agg1 alone on the device), CUDA events on the compute stream",
                     "pipelined": {"ms_per_launch": pipe_ms, "achieved": pipe_gbs, "frac": pipe_gbs / hbm,
                                   "note": "same kernel inside the timed pipelined region, sharing SMs/HBM with the concurrent sampling streams"},
                     "sequential_ms_per_step": tm3["total_ms"] / K,
                     "resources": res, "bound_resource": bound,
                     "resource_note": "feature rows the gather reads, split by where the store placed them; "
                                      "achieved = those bytes / the k_agg1 launch time; the path's fraction is "
                                      "the max over resources"},
        "e2e": {"value": e2e, "unit": "seeds/s", "h2d_bytes_per_step": B * 4, "d2h_bytes_per_step": 8},
        "tensor_roofline": tensor,
        "sampler": sampler,
        "gpu_launches": int(tm["launches_per_step"]) * K,
        "clocks": clk.summary(),
        "loss_first_last": [float(losses[0]), float(losses_e2e[-1])],
    }
    if not args.no_cpu_baseline and world == 1 and args.config not in SYNTH:
        import oracle
        if oracle.ref_available():
            # the same graph handed to the reference through its own A3G1 loader
            # (graph_io.cpp:60-87); our generator is bit-identical to its
            # generate_power_law (tests/test_host.py)
            from paper_2511_07421_b200 import graph as G
            path = os.path.join("/tmp", f"a3g_bench_{args.config}_{os.getpid()}.a3g")
            G.save_graph(g, path)
            rg = oracle.RefLib().load(path)
            os.remove(path)
            cores, cpu_model = host_cpu()
            r = cpu_reference_run(rg, args.config, args.gamma, args.cpu_units, 0, 0, warmup=1, hidden=args.hidden)
            out["cpu_baseline"] = {"value": r["seeds_per_s"], "unit": "seeds/s", "cores": 1, "kind": "reference",
                                   "cpu_model": cpu_model, "host_nproc": cores,
                                   "sample": f"{args.cpu_units} batches of epoch 0 (B={B}) after 1 untimed, "
                                             f"sequential 1-thread schedule, {r['seconds']:.1f} s"}
    print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def _steps_device(tr, dev_seeds, rng_seeds, gamma):
    """a3g_train_steps with seeds already resident in HBM (seeds_on_device=1)."""
    import ctypes as C
    from paper_2511_07421_b200._lib import check, f64p, lib, ptr, u64p
    K, B = dev_seeds.shape
    rs = np.ascontiguousarray(rng_seeds, dtype=np.uint64)
    losses = np.empty(K, dtype=np.float64)
    check(lib().a3g_train_steps(tr.h, C.cast(C.c_void_p(dev_seeds.data_ptr()), C.POINTER(C.c_uint32)), B, K,
                                ptr(rs, u64p), float(gamma), 0, 1, ptr(losses, f64p)))
    return losses


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
