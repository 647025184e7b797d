// dropin.hpp -- shared plumbing of the C++ drop-in (a3gnn:: declarations of
// proj/include/a3gnn implemented over the C-ABI include/a3g.h).
//
// The drop-in sources compile against the reference's OWN headers
// (-I <reference>/proj/include) and define the reference's functions, so a
// maintainer swaps them in for proj/src/{sampler,cache}.cpp and the train /
// evaluate_full_graph entry points of trainer.cpp. Device
// copies of a Graph / CacheState are made on first use and reused while the
// object lives (the reference treats both as immutable and shared,
// graph.hpp:3-4, cache.hpp:3-5).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "a3g.h"
#include "a3gnn/cache.hpp"
#include "a3gnn/common.hpp"
#include "a3gnn/graph.hpp"
#include "a3gnn/partition.hpp"
#include "a3gnn/trainer.hpp"

namespace a3gnn::b200 {

// a3g_status -> the reference's exception types (common.hpp:14-40).
[[noreturn]] void raise_status(a3g_status st);
inline void check(a3g_status st) {
  if (st != A3G_OK) raise_status(st);
}

// CUDA device used by the drop-in: $A3GNN_B200_DEVICE, default 0.
int device();

// Device CSR + f32 feature store + labels of g (uploaded once per Graph).
a3g_graph* device_graph(const graph::Graph& g);
// Device cache state (cached bitmap) of c over g.
a3g_cache* device_cache(const graph::Graph& g, const cache::CacheState& c);
// The device cache of c when only the CacheState is known (lookup(),
// cache.hpp:75): a registered cache with the same content, else one over a
// topology-only graph of device_map.size() nodes.
a3g_cache* device_cache_of(const cache::CacheState& c);
// This thread's sampler arena for (g, c) with capacity >= n_seeds and the
// given fanouts (the reference's producers call sample_khop concurrently,
// pipeline_exec.cpp:235-256: one arena per thread).
a3g_sampler* thread_sampler(a3g_graph* g, a3g_cache* c, std::uint32_t n_seeds,
                            const std::vector<std::uint32_t>& fanouts);
// Drop the device copies of g (and of caches over it).
void release(const graph::Graph& g);

// train() with u > 1 partition-local workers on the device (trainer_b200.cpp);
// also behind execute_pipeline with partitions > 1.
struct PartitionedRun {
  train::TrainReport rep;
  std::uint64_t hits = 0, misses = 0;
  train::Model model;
};
PartitionedRun train_partitioned(const graph::Graph& g, const train::ModelSpec& spec,
                                 const sampling::SamplerConfig& sampler_cfg, const cache::CacheState& cache_global,
                                 std::uint32_t u, graph::PartitionMethod method, std::uint32_t batch_size,
                                 std::uint32_t epochs, std::uint64_t model_seed);

}  // namespace a3gnn::b200
