// evaluator_b200.cpp -- the tuner's ground-truth Evaluator on the device
// executor (surrogate.hpp:79-88 make_execute_evaluator, with the knob mapping
// of a3gnn_b200.hpp). The tuner itself (PPO walk, rewards, Pareto front) stays
// the reference's host code.
#include <algorithm>

#include "a3gnn_b200.hpp"
#include "dropin.hpp"

namespace a3gnn::b200 {

DeviceDesign resolve_device_design(const graph::Graph& g, const DesignSpace& space, const DesignPoint& p,
                                   const sampling::SamplerConfig& sampler_base, const DeviceEvalOptions& opts) {
  DeviceDesign dd;
  dd.design = resolve(space, p);  // bounds-checked (ParameterError)
  const std::uint32_t level = p.idx[1];
  if (!opts.fanout_levels.empty()) {
    if (opts.fanout_levels.size() != space.partitions.size())
      throw ParameterError("device evaluator: one fanout level per partitions grid entry");
    dd.fanouts = opts.fanout_levels[level];
  } else {
    dd.fanouts = sampler_base.fanouts;
  }
  dd.design.partitions = 1;
  dd.sampling_streams =
      dd.design.mode == Mode::sequential ? 0 : static_cast<int>(std::clamp<std::uint32_t>(dd.design.workers, 1, 8));
  const double table = static_cast<double>(g.num_nodes) * g.feat_dim * 4.0;
  dd.cache_ratio = table > 0 ? std::min(1.0, static_cast<double>(dd.design.cache_volume) / table) : 0.0;
  return dd;
}

surrogate::Evaluator make_device_evaluator(const graph::Graph& g, const DesignSpace& space,
                                           const pipeline::PlatformSpec& platform, const train::ModelSpec& spec,
                                           const sampling::SamplerConfig& sampler_base,
                                           const DeviceEvalOptions& opts) {
  space.validate();
  return [&g, space, platform, spec, sampler_base, opts](const DesignPoint& p) -> Metrics {
    const DeviceDesign dd = resolve_device_design(g, space, p, sampler_base, opts);
    sampling::SamplerConfig cfg = sampler_base;
    cfg.fanouts = dd.fanouts;
    pipeline::ExecOptions eo;
    eo.epochs = opts.epochs;
    eo.queue_capacity = opts.queue_capacity;
    eo.model_seed = opts.model_seed;
    // the drop-in's execute_pipeline: the CUDA-stream pipeline (pipeline_b200.cpp)
    return pipeline::execute_pipeline(g, dd.design, platform, spec, cfg, eo).metrics;
  };
}

}  // namespace a3gnn::b200
