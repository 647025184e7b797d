// trainer_b200.cpp -- drop-in for train::train and train::evaluate_full_graph
// (trainer.hpp:81-117, trainer.cpp:241-303, 350-424): every step -- sampling,
// fused gather + mean aggregation, forward, backward, SGD -- runs on the
// device through the CUDA-stream pipeline (a3g_train_steps_v); the host plans
// the epoch's batches and seeds exactly as the reference.
#include <algorithm>
#include <cmath>
#include <limits>
#include <memory>

#include "a3gnn/rng.hpp"
#include "a3gnn/trainer.hpp"
#include "dropin.hpp"

namespace a3gnn::train {
namespace {

struct TrainerHandle {
  a3g_trainer* h = nullptr;
  ~TrainerHandle() {
    if (h) a3g_trainer_destroy(h);
  }
};

std::unique_ptr<TrainerHandle> make_trainer(const Graph& g, const CacheState& c, const ModelSpec& spec,
                                            const std::vector<std::uint32_t>& fanouts, std::uint32_t max_seeds,
                                            std::uint64_t model_seed) {
  if (spec.feat_dim != g.feat_dim) throw ParameterError("train: spec.feat_dim != graph feat_dim");
  auto t = std::make_unique<TrainerHandle>();
  b200::check(a3g_trainer_create(b200::device_graph(g), b200::device_cache(g, c), max_seeds, fanouts.data(),
                                 static_cast<std::uint32_t>(fanouts.size()), spec.hidden_dim, spec.num_classes,
                                 spec.learning_rate, model_seed, &t->h));
  return t;
}

}  // namespace

double evaluate_full_graph(const Model& m, const Graph& g) {
  const ModelSpec& spec = m.spec;
  const CacheState none;  // placement is irrelevant to the full-graph pass
  const std::vector<std::uint32_t> fan{1};
  auto t = make_trainer(g, none, spec, fan, 1, m.init_seed);
  b200::check(a3g_trainer_set_weights(t->h, m.w1.data(), m.w2.data()));
  double acc = 0.0;
  b200::check(a3g_evaluate_full_graph(t->h, g.test_mask.data(), &acc));
  return acc;
}

TrainReport train(const Graph& g, const ModelSpec& spec, const SamplerConfig& sampler_cfg,
                  const CacheState& cache_global, const TrainOptions& opts) {
  if (opts.batch_size < 1) throw ParameterError("train: batch_size must be >= 1");
  if (opts.u > 1)
    throw ConfigError("train: partitioned workers (u > 1) are not part of the B200 path "
                      "(data parallelism runs across GPUs)");
  std::vector<NodeId> train_nodes;
  for (std::uint64_t v = 0; v < g.num_nodes; ++v)
    if (g.train_mask[v]) train_nodes.push_back(static_cast<NodeId>(v));
  if (train_nodes.empty()) throw ConfigError("train: a worker has no train nodes");
  const std::uint32_t max_seeds =
      static_cast<std::uint32_t>(std::min<std::size_t>(opts.batch_size, train_nodes.size()));
  auto t = make_trainer(g, cache_global, spec, sampler_cfg.fanouts, max_seeds, opts.model_seed);
  const int kind = sampler_cfg.kind == sampling::SamplerKind::uniform_baseline ? A3G_SAMPLER_UNIFORM
                                                                               : A3G_SAMPLER_WEIGHTED;
  TrainReport rep;
  rep.param_bytes = spec.param_bytes();
  const std::uint64_t F = spec.feat_dim, H = spec.hidden_dim, C = spec.num_classes;
  std::vector<NodeId> order(train_nodes.size());
  for (std::uint32_t epoch = 0; epoch < opts.epochs; ++epoch) {
    // plan_epoch_batches(train_nodes, epoch, B, hash2(rng_seed, 0)) (trainer.cpp:378-379)
    a3g_plan_epoch_order(train_nodes.data(), train_nodes.size(), epoch, hash2(sampler_cfg.rng_seed, 0),
                         order.data());
    const std::uint32_t steps =
        static_cast<std::uint32_t>((order.size() + opts.batch_size - 1) / opts.batch_size);
    std::vector<std::uint64_t> off(steps + 1), seeds(steps);
    for (std::uint32_t s = 0; s <= steps; ++s)
      off[s] = std::min<std::uint64_t>(static_cast<std::uint64_t>(s) * opts.batch_size, order.size());
    for (std::uint32_t s = 0; s < steps; ++s) seeds[s] = a3g_sampling_seed(sampler_cfg.rng_seed, epoch, s, 0);
    std::vector<double> losses(steps);
    b200::check(a3g_train_steps_v(t->h, order.data(), off.data(), steps, seeds.data(), sampler_cfg.bias_rate, kind,
                                  0, losses.data()));
    std::vector<std::uint64_t> st(static_cast<std::size_t>(steps) * A3G_STEP_STATS);
    b200::check(a3g_trainer_step_stats(t->h, st.data(), steps));
    double loss = 0.0;
    std::uint64_t hits = 0, misses = 0;
    for (std::uint32_t s = 0; s < steps; ++s) {
      const std::uint64_t* r = st.data() + static_cast<std::size_t>(s) * A3G_STEP_STATS;
      loss += losses[s];
      hits += r[A3G_STAT_HITS];
      misses += r[A3G_STAT_MISSES];
      rep.max_batch_bytes = std::max(rep.max_batch_bytes, r[A3G_STAT_UNIQUE] * F * 4 + r[A3G_STAT_EDGES] * 8);
      rep.max_activation_bytes = std::max(
          rep.max_activation_bytes, (r[A3G_STAT_INNER] * (F + H) + r[A3G_STAT_SEEDS] * (H + C)) * 4);
    }
    rep.loss_curve.push_back(steps ? loss / steps : 0.0);
    rep.epoch_hit_rates.push_back(hits + misses ? static_cast<double>(hits) / static_cast<double>(hits + misses)
                                                : 0.0);
  }
  rep.epochs_run = opts.epochs;
  b200::check(a3g_evaluate_full_graph(t->h, g.test_mask.data(), &rep.test_accuracy));
  rep.accuracy_drop = opts.reference_accuracy ? *opts.reference_accuracy - rep.test_accuracy
                                              : std::numeric_limits<double>::quiet_NaN();
  return rep;
}

}  // namespace a3gnn::train
