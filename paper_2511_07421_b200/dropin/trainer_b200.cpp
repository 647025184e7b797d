// trainer_b200.cpp -- drop-in for the trainer entry points of trainer.hpp:
//  * forward / backward / grad_on_batch (trainer.cpp:59-239) on the caller's
//    explicit SampleBatch + feats: one device model per host thread
//    (a3g_batch_model_*, the pipeline's own kernels);
//  * sgd_step / sync_gradients (trainer.cpp:208-229) on the device
//    (a3g_sgd_step, a3g_mean_gradients);
//  * train (trainer.cpp:350-424) and evaluate_full_graph (:241-303): every
//    step -- sampling, fused gather + mean aggregation, forward, backward,
//    SGD -- runs on the device through the CUDA-stream pipeline
//    (a3g_train_steps_v); the host plans the epoch's batches and seeds exactly
//    as the reference.
#include <algorithm>
#include <cmath>
#include <limits>
#include <memory>

#include "a3gnn/kernels.hpp"
#include "a3gnn/partition.hpp"
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

// This thread's device model for explicit batches of (F, H, C).
a3g_batch_model* thread_model(const ModelSpec& spec) {
  struct Slot {
    a3g_batch_model* m = nullptr;
    std::uint32_t F = 0, H = 0, C = 0;
    ~Slot() { a3g_batch_model_destroy(m); }
  };
  thread_local Slot slot;
  if (!slot.m || slot.F != spec.feat_dim || slot.H != spec.hidden_dim || slot.C != spec.num_classes) {
    a3g_batch_model_destroy(slot.m);
    slot.m = nullptr;
    b200::check(a3g_batch_model_create(b200::device(), spec.feat_dim, spec.hidden_dim, spec.num_classes, &slot.m));
    slot.F = spec.feat_dim;
    slot.H = spec.hidden_dim;
    slot.C = spec.num_classes;
  }
  return slot.m;
}

// Loads (batch, feats, labels) into the thread's device model; returns n_inner.
std::uint64_t load(a3g_batch_model* dm, const SampleBatch& batch, const float* feats, const std::uint32_t* labels) {
  const std::size_t L = std::min<std::size_t>(batch.layers.size(), 2);  // trainer.cpp reads layers[0..1]
  std::vector<std::vector<std::uint32_t>> d(L), s(L);
  std::vector<const std::uint32_t*> pd(std::max<std::size_t>(L, 1)), ps(std::max<std::size_t>(L, 1));
  std::vector<std::uint64_t> ne(std::max<std::size_t>(L, 1), 0);
  for (std::size_t l = 0; l < L; ++l) {
    const auto& e = batch.layers[l].edges;
    d[l].resize(e.size());
    s[l].resize(e.size());
    for (std::size_t i = 0; i < e.size(); ++i) {
      d[l][i] = e[i].first;
      s[l][i] = e[i].second;
    }
    pd[l] = d[l].data();
    ps[l] = s[l].data();
    ne[l] = e.size();
  }
  std::uint64_t n_inner = 0;
  b200::check(a3g_batch_model_load(dm, batch.unique_nodes.size(), batch.num_seed_unique,
                                   static_cast<std::uint32_t>(L), ne.data(), pd.data(), ps.data(), feats, labels,
                                   &n_inner));
  return n_inner;
}

}  // namespace

ForwardResult forward(const Model& m, const SampleBatch& batch, const float* feats) {
  const ModelSpec& spec = m.spec;
  a3g_batch_model* dm = thread_model(spec);
  const std::uint64_t ni = load(dm, batch, feats, nullptr);
  b200::check(a3g_batch_model_run(dm, m.w1.data(), m.w2.data(), nullptr, nullptr, nullptr));
  const std::size_t ns = batch.num_seed_unique;
  ForwardResult out;
  out.inner_nodes.resize(ni);
  out.inner_pos.resize(batch.unique_nodes.size());
  out.inner_deg.resize(ni);
  out.outer_deg.resize(ns);
  out.agg_inner.resize(ni * spec.feat_dim);
  out.h1.resize(ni * spec.hidden_dim);
  out.agg_outer.resize(ns * spec.hidden_dim);
  out.logits.resize(ns * spec.num_classes);
  b200::check(a3g_batch_model_forward(dm, out.inner_nodes.data(), out.inner_pos.data(), out.inner_deg.data(),
                                      out.outer_deg.data(), out.agg_inner.data(), out.h1.data(),
                                      out.agg_outer.data(), out.logits.data()));
  // modelled as 4 bytes per value (trainer.cpp:134-135)
  out.activation_bytes = (out.agg_inner.size() + out.h1.size() + out.agg_outer.size() + out.logits.size()) * 4;
  return out;
}

// The device recomputes the forward pass it needs (fwd is the caller's cache
// of it; the kernels keep their own activations resident).
double backward(const Model& m, const SampleBatch& batch, const float* feats, const ForwardResult& fwd,
                const std::vector<std::uint32_t>& seed_labels, Gradients& grads) {
  (void)fwd;
  if (seed_labels.size() != batch.num_seed_unique) throw ParameterError("backward: seed_labels size mismatch");
  a3g_batch_model* dm = thread_model(m.spec);
  load(dm, batch, feats, seed_labels.data());
  grads.w1.assign(m.w1.size(), 0.0);
  grads.w2.assign(m.w2.size(), 0.0);
  double loss = 0.0;
  b200::check(a3g_batch_model_run(dm, m.w1.data(), m.w2.data(), &loss, grads.w1.data(), grads.w2.data()));
  return loss;
}

double grad_on_batch(const Model& m, const Graph& g, const SampleBatch& batch, const float* feats,
                     Gradients& grads) {
  std::vector<std::uint32_t> labels(batch.num_seed_unique);  // trainer.cpp:234-237
  for (std::size_t s = 0; s < batch.num_seed_unique; ++s) labels[s] = g.labels[batch.unique_nodes[s]];
  a3g_batch_model* dm = thread_model(m.spec);
  load(dm, batch, feats, labels.data());
  grads.w1.assign(m.w1.size(), 0.0);
  grads.w2.assign(m.w2.size(), 0.0);
  double loss = 0.0;
  b200::check(a3g_batch_model_run(dm, m.w1.data(), m.w2.data(), &loss, grads.w1.data(), grads.w2.data()));
  return loss;
}

void sgd_step(Model& m, const Gradients& g, double lr) {
  // the reference's axpy is fused in blocks of four under the AVX2 table
  const bool fused = kernels::active_backend() == kernels::Backend::avx2;
  auto step = [&](std::vector<double>& w, const std::vector<double>& gr) {
    const std::size_t n = std::min(w.size(), gr.size());
    b200::check(a3g_sgd_step(b200::device(), w.data(), gr.data(), n, fused ? n - n % 4 : 0, lr));
  };
  step(m.w1, g.w1);
  step(m.w2, g.w2);
}

Gradients sync_gradients(const std::vector<Gradients>& grads) {
  if (grads.empty()) throw ParameterError("sync_gradients: empty gradient list");
  for (const Gradients& g : grads)
    if (g.w1.size() != grads[0].w1.size() || g.w2.size() != grads[0].w2.size())
      throw ParameterError("sync_gradients: shape mismatch");
  Gradients out;
  out.w1.resize(grads[0].w1.size());
  out.w2.resize(grads[0].w2.size());
  std::vector<const double*> p1, p2;
  for (const Gradients& g : grads) {
    p1.push_back(g.w1.data());
    p2.push_back(g.w2.data());
  }
  const auto k = static_cast<std::uint32_t>(grads.size());
  b200::check(a3g_mean_gradients(b200::device(), p1.data(), k, out.w1.size(), out.w1.data()));
  b200::check(a3g_mean_gradients(b200::device(), p2.data(), k, out.w2.size(), out.w2.data()));
  return out;
}

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

}  // namespace a3gnn::train

namespace a3gnn::b200 {

// trainer.cpp:350-424 with u > 1 partition-local workers:
// the reference's own partitioning and worker contexts (partition_graph,
// make_worker_contexts, cache::localize -- host setup), each worker's step on
// the device over its local graph and localized cache (RNG keyed by local
// ids, as the reference), the unweighted mean of the workers' gradients
// (sync_gradients) and the SGD step (sgd_step), both on the device.
PartitionedRun train_partitioned(const graph::Graph& g, const train::ModelSpec& spec,
                                 const sampling::SamplerConfig& sampler_cfg, const cache::CacheState& cache_global,
                                 std::uint32_t u, graph::PartitionMethod method, std::uint32_t batch_size,
                                 std::uint32_t epochs, std::uint64_t model_seed) {
  using namespace a3gnn::train;
  const graph::PartitionSet parts = graph::partition_graph(g, u, method);
  const std::vector<WorkerContext> ctxs = make_worker_contexts(g, &parts, cache_global);
  const auto nw = static_cast<std::uint32_t>(ctxs.size());
  for (const auto& c : ctxs)
    if (c.train_nodes.empty()) throw ConfigError("train: a worker has no train nodes");
  PartitionedRun run;
  run.model = init_model(spec, model_seed);
  ModelSpec wspec = spec;
  wspec.learning_rate = 0.0;  // worker trainers compute gradients only
  std::vector<a3g_trainer*> tr(nw, nullptr);
  struct Guard {
    std::vector<a3g_trainer*>& t;
    ~Guard() {
      for (a3g_trainer* h : t) a3g_trainer_destroy(h);
    }
  } guard{tr};
  for (std::uint32_t w = 0; w < nw; ++w) {
    const Graph& lg = *ctxs[w].graph;
    const auto ms = static_cast<std::uint32_t>(std::min<std::size_t>(batch_size, ctxs[w].train_nodes.size()));
    b200::check(a3g_trainer_create(device_graph(lg), device_cache(lg, ctxs[w].cache), ms, sampler_cfg.fanouts.data(),
                                   static_cast<std::uint32_t>(sampler_cfg.fanouts.size()), spec.hidden_dim,
                                   spec.num_classes, 0.0, model_seed, &tr[w]));
  }
  const int kind = sampler_cfg.kind == sampling::SamplerKind::uniform_baseline ? A3G_SAMPLER_UNIFORM
                                                                               : A3G_SAMPLER_WEIGHTED;
  const std::uint64_t F = spec.feat_dim, H = spec.hidden_dim, C = spec.num_classes;
  TrainReport& rep = run.rep;
  rep.param_bytes = spec.param_bytes();
  for (std::uint32_t epoch = 0; epoch < epochs; ++epoch) {
    std::vector<std::vector<std::vector<NodeId>>> batches(nw);
    std::size_t steps = 0;
    for (std::uint32_t w = 0; w < nw; ++w) {
      batches[w] = plan_epoch_batches(ctxs[w].train_nodes, epoch, batch_size, hash2(sampler_cfg.rng_seed, w));
      steps = std::max(steps, batches[w].size());
    }
    double epoch_loss = 0.0;
    std::size_t loss_count = 0;
    std::uint64_t hits = 0, misses = 0;
    for (std::size_t step = 0; step < steps; ++step) {
      std::vector<Gradients> grads(nw);
      for (std::uint32_t w = 0; w < nw; ++w) {
        const auto& seeds = batches[w][step % batches[w].size()];
        const std::uint64_t off[2] = {0, seeds.size()};
        const std::uint64_t rs = sampling_seed(sampler_cfg.rng_seed, epoch, static_cast<std::uint32_t>(step), w);
        b200::check(a3g_trainer_set_weights(tr[w], run.model.w1.data(), run.model.w2.data()));
        double loss = 0.0;
        b200::check(a3g_train_steps_v(tr[w], seeds.data(), off, 1, &rs, sampler_cfg.bias_rate, kind, 0, &loss));
        grads[w].w1.resize(run.model.w1.size());
        grads[w].w2.resize(run.model.w2.size());
        b200::check(a3g_trainer_last_grads(tr[w], grads[w].w1.data(), grads[w].w2.data()));
        std::uint64_t st[A3G_STEP_STATS];
        b200::check(a3g_trainer_step_stats(tr[w], st, 1));
        hits += st[A3G_STAT_HITS];
        misses += st[A3G_STAT_MISSES];
        rep.max_batch_bytes = std::max(rep.max_batch_bytes, st[A3G_STAT_UNIQUE] * F * 4 + st[A3G_STAT_EDGES] * 8);
        rep.max_activation_bytes =
            std::max(rep.max_activation_bytes, (st[A3G_STAT_INNER] * (F + H) + st[A3G_STAT_SEEDS] * (H + C)) * 4);
        epoch_loss += loss;
        ++loss_count;
      }
      sgd_step(run.model, sync_gradients(grads), spec.learning_rate);
    }
    rep.loss_curve.push_back(loss_count > 0 ? epoch_loss / static_cast<double>(loss_count) : 0.0);
    rep.epoch_hit_rates.push_back(hits + misses ? static_cast<double>(hits) / static_cast<double>(hits + misses)
                                                : 0.0);
    run.hits += hits;
    run.misses += misses;
  }
  rep.epochs_run = epochs;
  rep.test_accuracy = evaluate_full_graph(run.model, g);
  return run;
}

}  // namespace a3gnn::b200

namespace a3gnn::train {

TrainReport train(const Graph& g, const ModelSpec& spec, const SamplerConfig& sampler_cfg,
                  const CacheState& cache_global, const TrainOptions& opts) {
  if (opts.batch_size < 1) throw ParameterError("train: batch_size must be >= 1");
  if (opts.u > 1) {  // partition-local workers (trainer.cpp:353-359)
    auto run = b200::train_partitioned(g, spec, sampler_cfg, cache_global, opts.u, opts.partition_method,
                                       opts.batch_size, opts.epochs, opts.model_seed);
    run.rep.accuracy_drop = opts.reference_accuracy ? *opts.reference_accuracy - run.rep.test_accuracy
                                                    : std::numeric_limits<double>::quiet_NaN();
    return run.rep;
  }
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
