// a3gnn_b200.hpp -- public additions of the B200 drop-in for reference code
// (compile against proj/include; link liba3gnn_b200.so).
//
// make_device_evaluator: a surrogate::Evaluator (surrogate.hpp:19) backed by
// the device executor, for the reference's host-side RL tuner
// (tuner::tune / grid_search, tuner.cpp:29-120) and its L4 dataset
// collection (collect_profile_dataset). The tuner keeps its seven knobs and
// its fixed state length (design_space.hpp:30-41, tuner.hpp:56); on the B200
// path they mean:
//
//   knob 0 batch_size        as is
//   knob 1 partitions        FANOUT LEVEL: index i selects fanout_levels[i]
//                            (the B200 tuner selects cache ratio, fanout and
//                            pipeline depth only -- scaling is data
//                            parallelism across GPUs -- so this slot carries
//                            the fanout knob the reference lacks; the
//                            partitioned mode itself still runs through
//                            train / execute_pipeline); empty fanout_levels =
//                            the sampler_base fanouts
//   knob 2 bias_rate         as is (gamma)
//   knob 3 sampling_device   no effect: sampling always runs on the GPU
//                            (the reference's knob only scales sampling time)
//   knob 4 workers           PIPELINE DEPTH: sampling streams (1..8) ahead of
//                            the compute stream in pmode1 / pmode2
//   knob 5 cache_volume      CACHE RATIO: volume / (n * F * 4) of the nodes,
//                            by out-degree hotness (cache.cpp:12-46)
//   knob 6 mode              sequential = depth 0 (one stream)
//
// Metrics are execute_pipeline's (pipeline_exec.cpp:279-290): epochs per
// second of the device run, the reference's analytic memory estimate, and the
// device full-graph test accuracy.
#pragma once

#include <cstdint>
#include <vector>

#include "a3gnn/surrogate.hpp"

namespace a3gnn::b200 {

struct DeviceEvalOptions {
  std::uint32_t epochs = 1;
  std::uint32_t queue_capacity = 4;
  std::uint64_t model_seed = 1;
  // fanouts per level of the space's partitions grid (outermost first)
  std::vector<std::vector<std::uint32_t>> fanout_levels;
};

// The resolved design the device evaluator runs for point p (knob mapping above).
struct DeviceDesign {
  ResolvedDesign design;  // partitions forced to 1
  std::vector<std::uint32_t> fanouts;
  int sampling_streams = 0;  // 0 = sequential
  double cache_ratio = 0.0;
};
DeviceDesign resolve_device_design(const graph::Graph& g, const DesignSpace& space, const DesignPoint& p,
                                   const sampling::SamplerConfig& sampler_base, const DeviceEvalOptions& opts);

surrogate::Evaluator make_device_evaluator(const graph::Graph& g, const DesignSpace& space,
                                           const pipeline::PlatformSpec& platform, const train::ModelSpec& spec,
                                           const sampling::SamplerConfig& sampler_base,
                                           const DeviceEvalOptions& opts);

}  // namespace a3gnn::b200
