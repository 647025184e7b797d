"""paper_2511_07421_b200 -- B200-native A3GNN data-parallel mini-batch hot path.

Host-side mirror of the reference's ``proj/include/a3gnn`` sampler /
feature-cache / trainer interfaces over the C-ABI library liba3g_b200.so
(include/a3g.h), whose kernels are hand-written for sm_100a:

    graph     -> graph::Graph, generate_power_law, A3G1 load/save
    cache     -> cache::build_static_cache, retrieve_features, hit_rate
    sampling  -> sampling::sample_khop (GPU), reservoirs, dedup_ratio
    train     -> train::Trainer (GPU step / pipelined steps), init_model, ...
"""
from ._lib import (A3gError, ConfigError, CudaError, IoError, LookupError_, NcclError, OutOfMemory,  # noqa: F401
                   ParameterError, LIB_PATH, lib)

__all__ = ["graph", "cache", "sampling", "train", "lib", "LIB_PATH", "ParameterError", "IoError", "ConfigError",
           "CudaError"]


def __getattr__(name):
    if name in ("graph", "cache", "sampling", "train"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
