// tuner_check.cpp -- TEST DRIVER of the device Evaluator (a3gnn_b200.hpp).
// Built twice (paper_2511_07421_b200/build.py):
//   tuner_check        the reference alone: surrogate::make_execute_evaluator
//                      (the CPU executor) on design points at fanout level 0
//   tuner_check_b200   linked with liba3gnn_b200.so: b200::make_device_evaluator
//                      on the same points, then the reference's own PPO tuner
//                      (tuner::tune) and grid search driving it
// and prints one line per result (tests/test_tuner_gpu.py compares them).
#include <cstdio>

#include "a3gnn/generators.hpp"
#include "a3gnn/tuner.hpp"
#ifdef A3G_DEVICE_EVAL
#include "a3gnn_b200.hpp"
#endif

using namespace a3gnn;

int main(int argc, char** argv) {
  const std::uint64_t n = argc > 1 ? std::stoull(argv[1]) : 20000;
  const graph::Graph g = graph::generate_power_law(n, 3, 2.5, 32, 1);
  DesignSpace space;
  space.batch_sizes = {256, 512};
  space.partitions = {1, 2};  // device evaluator: fanout levels {10,5}, {15,10}
  space.bias_rates = {1, 8};
  space.sampling_devices = {Device::gpu};
  space.workers = {1, 4};
  space.cache_volumes = {0, (n / 5) * g.feat_dim * 4};
  space.modes = {Mode::sequential, Mode::pmode1, Mode::pmode2};
  train::ModelSpec spec;
  spec.feat_dim = g.feat_dim;
  spec.hidden_dim = 16;
  spec.num_classes = 4;
  sampling::SamplerConfig base;
  base.fanouts = {10, 5};
  base.rng_seed = 3;
  pipeline::PlatformSpec plat;
#ifdef A3G_DEVICE_EVAL
  b200::DeviceEvalOptions o;
  o.epochs = 1;
  o.fanout_levels = {{10, 5}, {15, 10}};
  const surrogate::Evaluator eval = b200::make_device_evaluator(g, space, plat, spec, base, o);
#else
  pipeline::ExecOptions eo;
  eo.epochs = 1;
  const surrogate::Evaluator eval = surrogate::make_execute_evaluator(g, space, plat, spec, base, eo);
#endif
  // knob order: batch, partitions (fanout level), bias, device, workers, cache, mode
  const std::vector<DesignPoint> pts = {{{0, 0, 0, 0, 0, 0, 0}}, {{1, 0, 1, 0, 1, 1, 1}}, {{0, 0, 1, 0, 1, 1, 2}},
                                        {{1, 0, 0, 0, 0, 1, 0}}};
  for (std::size_t i = 0; i < pts.size(); ++i) {
    const Metrics m = eval(pts[i]);
    std::printf("point %zu accuracy %.17g mem %.17g thr_positive %d\n", i, m.accuracy, m.memory_bytes,
                m.throughput_eps > 0 ? 1 : 0);
  }
#ifdef A3G_DEVICE_EVAL
  {  // the knob mapping itself
    const auto dd = b200::resolve_device_design(g, space, {{1, 1, 1, 0, 1, 1, 1}}, base, o);
    std::printf("mapping fanouts %u,%u streams %d ratio %.3f partitions %u\n", dd.fanouts[0], dd.fanouts[1],
                dd.sampling_streams, dd.cache_ratio, dd.design.partitions);
  }
  tuner::TunerConfig cfg;
  cfg.weights = {1.0, 0.0, 1.0};
  cfg.budget = 8;
  cfg.thr_hi = 50.0;
  cfg.acc_lo = 0.2;
  cfg.acc_hi = 0.35;
  const auto r = tuner::tune(space, eval, cfg, 7);
  std::printf("tune evaluations %llu feasible %d best_fanout_level %u best_acc %.4f pareto %zu\n",
              (unsigned long long)r.evaluations_used, r.found_feasible ? 1 : 0, r.best_point.idx[1],
              r.best_metrics.accuracy, r.pareto.size());
#endif
  return 0;
}
