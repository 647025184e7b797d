// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference library (compiled in place from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It calls only
// the reference's public API (proj/include/a3gnn/*.hpp) so that tests can
// (1) pin the plain-C restatement in oracle/a3g_oracle.c, (2) generate the
// golden fixtures under tests/golden/, and (3) time the reference's own CPU
// path as bench.py's cpu_baseline / --impl reference arm.
// No reference source is copied here.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "a3gnn/cache.hpp"
#include "a3gnn/generators.hpp"
#include "a3gnn/graph_io.hpp"
#include "a3gnn/kernels.hpp"
#include "a3gnn/sampler.hpp"
#include "a3gnn/trainer.hpp"

using namespace a3gnn;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const ParameterError*>(&e)) return 1;
  if (dynamic_cast<const LookupError*>(&e)) return 2;
  if (dynamic_cast<const ConfigError*>(&e)) return 3;
  if (dynamic_cast<const IoError*>(&e)) return 4;
  return 9;
}

cache::CacheState cache_from_map(const std::int32_t* device_map, std::uint64_t n,
                                 std::uint32_t num_devices) {
  cache::CacheState c;
  c.device_map.assign(n, cache::kCacheMiss);
  if (device_map)
    for (std::uint64_t v = 0; v < n; ++v)
      num_devices = std::max<std::uint32_t>(num_devices, static_cast<std::uint32_t>(device_map[v] + 1));
  c.cached_per_device.resize(std::max<std::uint32_t>(1, num_devices));
  c.bytes_used.assign(c.cached_per_device.size(), 0);
  if (device_map) {
    for (std::uint64_t v = 0; v < n; ++v) {
      c.device_map[v] = device_map[v];
      if (device_map[v] >= 0) c.cached_per_device[device_map[v]].push_back(static_cast<NodeId>(v));
    }
  }
  return c;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// kernels.hpp:41-44: 0 = scalar, 1 = avx2
int ref_set_backend(int b) {
  try {
    kernels::set_backend(b == 0 ? kernels::Backend::scalar : kernels::Backend::avx2);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---------------------------------------------------------------- graph ---
void* ref_graph_power_law(std::uint64_t n, std::uint32_t m, double exponent, std::uint32_t f,
                          std::uint64_t seed) {
  try {
    return new graph::Graph(graph::generate_power_law(n, m, exponent, f, seed));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void* ref_graph_sbm(std::uint64_t n, std::uint32_t blocks, double p_in, double p_out,
                    std::uint32_t f, std::uint64_t seed) {
  try {
    return new graph::Graph(graph::generate_sbm(n, blocks, p_in, p_out, f, seed));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void* ref_graph_from_edges(std::uint64_t n, const std::uint32_t* src, const std::uint32_t* dst,
                           std::uint64_t m, std::uint32_t f) {
  try {
    std::vector<std::pair<NodeId, NodeId>> e(m);
    for (std::uint64_t i = 0; i < m; ++i) e[i] = {src[i], dst[i]};
    return new graph::Graph(graph::from_edges(n, std::move(e), f));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
void* ref_graph_load(const char* path) {
  try {
    return new graph::Graph(graph::load_graph(path));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
int ref_graph_save(void* h, const char* path) {
  try {
    graph::save_graph(*static_cast<graph::Graph*>(h), path);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
void ref_graph_free(void* h) { delete static_cast<graph::Graph*>(h); }
void ref_graph_info(void* h, std::uint64_t* n, std::uint64_t* m, std::uint32_t* f) {
  auto* g = static_cast<graph::Graph*>(h);
  *n = g->num_nodes;
  *m = g->num_edges;
  *f = g->feat_dim;
}
// Pointers into the graph's vectors (valid until ref_graph_free).
void ref_graph_arrays(void* h, const std::uint64_t** ro, const std::uint32_t** col,
                      const float** feat, const std::uint32_t** labels,
                      const std::uint8_t** train_mask, const std::uint8_t** test_mask) {
  auto* g = static_cast<graph::Graph*>(h);
  *ro = g->row_offsets.data();
  *col = g->col_indices.data();
  *feat = g->features.data();
  *labels = g->labels.data();
  *train_mask = g->train_mask.data();
  *test_mask = g->test_mask.data();
}

// ---------------------------------------------------------------- cache ---
std::int64_t ref_build_static_cache(void* h, std::uint64_t volume, std::uint32_t num_devices,
                                    std::int32_t* device_map_out) {
  try {
    auto* g = static_cast<graph::Graph*>(h);
    cache::CacheConfig cfg;
    cfg.volume_bytes = volume;
    cfg.num_devices = num_devices;
    const auto c = cache::build_static_cache(*g, cfg);
    std::copy(c.device_map.begin(), c.device_map.end(), device_map_out);
    return static_cast<std::int64_t>(c.total_cached());
  } catch (const std::exception& e) {
    return -fail(e);
  }
}

// -------------------------------------------------------------- sampler ---
struct RefBatch {
  sampling::SampleBatch b;
  std::vector<std::vector<std::uint32_t>> dst, src;
};

void* ref_sample_khop(void* h, const std::int32_t* device_map, std::uint32_t num_devices,
                      const std::uint32_t* seeds, std::uint64_t n_seeds,
                      const std::uint32_t* fanouts, std::uint32_t num_layers, double gamma,
                      int kind, std::uint64_t rng_seed, int* err) {
  try {
    auto* g = static_cast<graph::Graph*>(h);
    const auto c = cache_from_map(device_map, g->num_nodes, num_devices);
    sampling::SamplerConfig cfg;
    cfg.fanouts.assign(fanouts, fanouts + num_layers);
    cfg.bias_rate = gamma;
    cfg.rng_seed = rng_seed;
    cfg.kind = kind == 1 ? sampling::SamplerKind::uniform_baseline
                         : sampling::SamplerKind::weighted_reservoir;
    auto* rb = new RefBatch;
    rb->b = sampling::sample_khop(*g, std::vector<NodeId>(seeds, seeds + n_seeds), cfg, c);
    for (const auto& l : rb->b.layers) {
      rb->dst.emplace_back();
      rb->src.emplace_back();
      for (const auto& [d, s] : l.edges) {
        rb->dst.back().push_back(d);
        rb->src.back().push_back(s);
      }
    }
    *err = 0;
    return rb;
  } catch (const std::exception& e) {
    *err = fail(e);
    return nullptr;
  }
}
void ref_batch_free(void* p) { delete static_cast<RefBatch*>(p); }
std::uint64_t ref_batch_num_unique(void* p) { return static_cast<RefBatch*>(p)->b.unique_nodes.size(); }
std::uint64_t ref_batch_num_seed_unique(void* p) { return static_cast<RefBatch*>(p)->b.num_seed_unique; }
std::uint64_t ref_batch_dups(void* p) { return static_cast<RefBatch*>(p)->b.num_duplicates_removed; }
const std::uint32_t* ref_batch_unique(void* p) { return static_cast<RefBatch*>(p)->b.unique_nodes.data(); }
std::uint64_t ref_batch_layer_ne(void* p, std::uint32_t l) { return static_cast<RefBatch*>(p)->dst[l].size(); }
const std::uint32_t* ref_batch_layer_dst(void* p, std::uint32_t l) { return static_cast<RefBatch*>(p)->dst[l].data(); }
const std::uint32_t* ref_batch_layer_src(void* p, std::uint32_t l) { return static_cast<RefBatch*>(p)->src[l].data(); }

// weighted_reservoir_sample / uniform_reservoir_sample on an explicit stream.
std::int64_t ref_weighted_reservoir(const std::uint32_t* nbrs, const double* w, std::uint64_t n,
                                    std::uint32_t m, std::uint64_t seed, std::uint64_t stream,
                                    std::uint32_t* out) {
  try {
    RngStream rng(seed, stream);
    const auto r = sampling::weighted_reservoir_sample({nbrs, n}, {w, n}, m, rng);
    std::copy(r.begin(), r.end(), out);
    return static_cast<std::int64_t>(r.size());
  } catch (const std::exception& e) {
    return -fail(e);
  }
}
std::int64_t ref_uniform_reservoir(const std::uint32_t* nbrs, std::uint64_t n, std::uint32_t m,
                                   std::uint64_t seed, std::uint64_t stream, std::uint32_t* out) {
  try {
    RngStream rng(seed, stream);
    const auto r = sampling::uniform_reservoir_sample({nbrs, n}, m, rng);
    std::copy(r.begin(), r.end(), out);
    return static_cast<std::int64_t>(r.size());
  } catch (const std::exception& e) {
    return -fail(e);
  }
}

// retrieve_features: rows + hits/misses + B
std::uint64_t ref_retrieve_features(void* h, const std::int32_t* device_map,
                                    std::uint32_t num_devices, void* p, float* out,
                                    std::uint64_t* hits, std::uint64_t* misses) {
  auto* g = static_cast<graph::Graph*>(h);
  const auto c = cache_from_map(device_map, g->num_nodes, num_devices);
  cache::CacheAccounting acc(std::max<std::uint32_t>(1, num_devices));
  auto [feats, stats] = cache::retrieve_features(static_cast<RefBatch*>(p)->b, c, *g, acc);
  std::copy(feats.begin(), feats.end(), out);
  *hits = acc.hits.load();
  *misses = acc.misses.load();
  return stats.batch_bytes;
}

// -------------------------------------------------------------- trainer ---
int ref_init_model(std::uint32_t f, std::uint32_t hdim, std::uint32_t c, std::uint64_t seed,
                   double* w1, double* w2) {
  try {
    train::ModelSpec spec;
    spec.feat_dim = f;
    spec.hidden_dim = hdim;
    spec.num_classes = c;
    const auto m = train::init_model(spec, seed);
    std::copy(m.w1.begin(), m.w1.end(), w1);
    std::copy(m.w2.begin(), m.w2.end(), w2);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// forward + backward on a sampled batch with caller weights; intermediates out.
double ref_grad_on_batch(void* h, void* p, const float* feats, std::uint32_t hdim, std::uint32_t c,
                         const double* w1, const double* w2, double* gw1, double* gw2,
                         std::uint64_t* n_inner, double* logits, double* agg_inner, double* h1,
                         double* agg_outer) {
  auto* g = static_cast<graph::Graph*>(h);
  const auto& b = static_cast<RefBatch*>(p)->b;
  train::Model m;
  m.spec.feat_dim = g->feat_dim;
  m.spec.hidden_dim = hdim;
  m.spec.num_classes = c;
  m.w1.assign(w1, w1 + static_cast<std::size_t>(g->feat_dim) * hdim);
  m.w2.assign(w2, w2 + static_cast<std::size_t>(hdim) * c);
  const auto fwd = train::forward(m, b, feats);
  std::vector<std::uint32_t> labels(b.num_seed_unique);
  for (std::size_t s = 0; s < b.num_seed_unique; ++s) labels[s] = g->labels[b.unique_nodes[s]];
  train::Gradients gr;
  const double loss = train::backward(m, b, feats, fwd, labels, gr);
  std::copy(gr.w1.begin(), gr.w1.end(), gw1);
  std::copy(gr.w2.begin(), gr.w2.end(), gw2);
  if (n_inner) *n_inner = fwd.inner_nodes.size();
  if (logits) std::copy(fwd.logits.begin(), fwd.logits.end(), logits);
  if (agg_inner) std::copy(fwd.agg_inner.begin(), fwd.agg_inner.end(), agg_inner);
  if (h1) std::copy(fwd.h1.begin(), fwd.h1.end(), h1);
  if (agg_outer) std::copy(fwd.agg_outer.begin(), fwd.agg_outer.end(), agg_outer);
  return loss;
}

// Hand-built-batch forward/backward (test_trainer.cpp:22-35 style fixtures).
double ref_grad_on_edges(std::uint32_t f, std::uint32_t hdim, std::uint32_t c, const double* w1,
                         const double* w2, std::uint64_t n_unique, std::uint64_t n_seeds,
                         std::uint32_t num_layers, const std::uint64_t* ne,
                         const std::uint32_t* const* ed, const std::uint32_t* const* es,
                         const float* feats, const std::uint32_t* seed_labels, double* gw1,
                         double* gw2, double* logits) {
  sampling::SampleBatch b;
  b.unique_nodes.resize(n_unique);
  for (std::uint64_t i = 0; i < n_unique; ++i) b.unique_nodes[i] = static_cast<NodeId>(i);
  b.seeds.assign(b.unique_nodes.begin(), b.unique_nodes.begin() + n_seeds);
  b.num_seed_unique = n_seeds;
  b.layers.resize(num_layers);
  for (std::uint32_t l = 0; l < num_layers; ++l)
    for (std::uint64_t e = 0; e < ne[l]; ++e) b.layers[l].edges.emplace_back(ed[l][e], es[l][e]);
  train::Model m;
  m.spec.feat_dim = f;
  m.spec.hidden_dim = hdim;
  m.spec.num_classes = c;
  m.w1.assign(w1, w1 + static_cast<std::size_t>(f) * hdim);
  m.w2.assign(w2, w2 + static_cast<std::size_t>(hdim) * c);
  const auto fwd = train::forward(m, b, feats);
  train::Gradients gr;
  const double loss =
      train::backward(m, b, feats, fwd, std::vector<std::uint32_t>(seed_labels, seed_labels + n_seeds), gr);
  std::copy(gr.w1.begin(), gr.w1.end(), gw1);
  std::copy(gr.w2.begin(), gr.w2.end(), gw2);
  if (logits) std::copy(fwd.logits.begin(), fwd.logits.end(), logits);
  return loss;
}

std::uint64_t ref_sampling_seed(std::uint64_t base, std::uint32_t epoch, std::uint32_t step,
                                std::uint32_t worker) {
  return train::sampling_seed(base, epoch, step, worker);
}

// plan_epoch_batches flattened (batches are consecutive chunks).
void ref_plan_epoch_order(const std::uint32_t* train_nodes, std::uint64_t n, std::uint32_t epoch,
                          std::uint64_t seed, std::uint32_t* order) {
  const auto b = train::plan_epoch_batches(std::vector<NodeId>(train_nodes, train_nodes + n),
                                           epoch, static_cast<std::uint32_t>(std::max<std::uint64_t>(n, 1)), seed);
  std::uint64_t k = 0;
  for (const auto& x : b)
    for (NodeId v : x) order[k++] = v;
}

// train() (trainer.cpp:350) at u=1: epoch loss curve, hit rates, accuracy.
int ref_train(void* h, const std::int32_t* device_map, const std::uint32_t* fanouts,
              std::uint32_t num_layers, double gamma, int kind, std::uint64_t rng_seed,
              std::uint32_t batch_size, std::uint32_t epochs, std::uint32_t hdim, std::uint32_t c,
              double lr, std::uint64_t model_seed, double* loss_curve, double* hit_rates,
              double* accuracy) {
  try {
    auto* g = static_cast<graph::Graph*>(h);
    const auto cache = cache_from_map(device_map, g->num_nodes, 1);
    train::ModelSpec spec;
    spec.feat_dim = g->feat_dim;
    spec.hidden_dim = hdim;
    spec.num_classes = c;
    spec.learning_rate = lr;
    sampling::SamplerConfig scfg;
    scfg.fanouts.assign(fanouts, fanouts + num_layers);
    scfg.bias_rate = gamma;
    scfg.rng_seed = rng_seed;
    scfg.kind = kind == 1 ? sampling::SamplerKind::uniform_baseline
                          : sampling::SamplerKind::weighted_reservoir;
    train::TrainOptions opts;
    opts.batch_size = batch_size;
    opts.epochs = epochs;
    opts.model_seed = model_seed;
    const auto r = train::train(*g, spec, scfg, cache, opts);
    std::copy(r.loss_curve.begin(), r.loss_curve.end(), loss_curve);
    std::copy(r.epoch_hit_rates.begin(), r.epoch_hit_rates.end(), hit_rates);
    *accuracy = r.test_accuracy;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The train() step loop (trainer.cpp:374-407, u=1) composed from the public
// API, bounded to max_steps and exposing the weights: per-step losses out,
// w1/w2 updated in place.
std::int64_t ref_train_steps(void* h, const std::int32_t* device_map, const std::uint32_t* fanouts,
                             std::uint32_t num_layers, double gamma, int kind,
                             std::uint64_t rng_seed, std::uint32_t batch_size, std::uint32_t hdim,
                             std::uint32_t c, double lr, double* w1, double* w2,
                             std::uint64_t max_steps, double* losses) {
  try {
    auto* g = static_cast<graph::Graph*>(h);
    const auto cache = cache_from_map(device_map, g->num_nodes, 1);
    train::Model m;
    m.spec.feat_dim = g->feat_dim;
    m.spec.hidden_dim = hdim;
    m.spec.num_classes = c;
    m.w1.assign(w1, w1 + static_cast<std::size_t>(g->feat_dim) * hdim);
    m.w2.assign(w2, w2 + static_cast<std::size_t>(hdim) * c);
    const auto ctxs = train::make_worker_contexts(*g, nullptr, cache);
    cache::CacheAccounting acc(1);
    std::uint64_t done = 0;
    for (std::uint32_t epoch = 0; done < max_steps; ++epoch) {
      const auto batches =
          train::plan_epoch_batches(ctxs[0].train_nodes, epoch, batch_size, hash2(rng_seed, 0));
      for (std::size_t step = 0; step < batches.size() && done < max_steps; ++step) {
        sampling::SamplerConfig cfg;
        cfg.fanouts.assign(fanouts, fanouts + num_layers);
        cfg.bias_rate = gamma;
        cfg.kind = kind == 1 ? sampling::SamplerKind::uniform_baseline
                             : sampling::SamplerKind::weighted_reservoir;
        cfg.rng_seed = train::sampling_seed(rng_seed, epoch, static_cast<std::uint32_t>(step), 0);
        const auto batch = sampling::sample_khop(*g, batches[step], cfg, cache);
        auto [feats, stats] = cache::retrieve_features(batch, cache, *g, acc);
        const auto fwd = train::forward(m, batch, feats.data());
        std::vector<std::uint32_t> labels(batch.num_seed_unique);
        for (std::size_t s = 0; s < batch.num_seed_unique; ++s)
          labels[s] = g->labels[batch.unique_nodes[s]];
        std::vector<train::Gradients> grads(1);
        losses[done++] = train::backward(m, batch, feats.data(), fwd, labels, grads[0]);
        train::sgd_step(m, train::sync_gradients(grads), lr);
      }
    }
    std::copy(m.w1.begin(), m.w1.end(), w1);
    std::copy(m.w2.begin(), m.w2.end(), w2);
    return static_cast<std::int64_t>(done);
  } catch (const std::exception& e) {
    return -fail(e);
  }
}

// Bounded CPU-baseline harness: the reference's own per-batch functions
// (sample_khop -> retrieve_features -> forward -> backward -> sync_gradients
// -> sgd_step) on `units` consecutive steps of epoch 0, scheduled exactly as
// execute_pipeline's three modes (pipeline_exec.cpp:219-276):
//   mode 0 sequential: one thread does everything (:219-228);
//   mode 1 pmode1: `producers` threads sample + retrieve into an ordered
//          bounded channel of `queue_capacity`, the calling thread trains;
//   mode 2 pmode2: producers only sample, the consumer retrieves + trains.
// execute_pipeline itself always runs whole epochs and ends with a full-graph
// evaluation (C2: 112.8M edges x 602 f64 = ~540 GB of row reads), which does
// not fit a bounded sample; this harness times the same schedule over a
// bounded slice. `warmup` steps (steps [0, warmup)) run untimed first; the
// timed units are steps [warmup, warmup + units). Returns wall seconds of the
// timed units; *seeds_out = seeds trained in them.
double ref_bench_steps(void* h, const std::int32_t* device_map, const std::uint32_t* fanouts,
                       std::uint32_t num_layers, double gamma, std::uint64_t rng_seed,
                       std::uint32_t batch_size, std::uint32_t hdim, std::uint32_t c, double lr,
                       std::uint32_t warmup, std::uint32_t units, int mode, std::uint32_t producers,
                       std::uint32_t queue_capacity, std::uint64_t* seeds_out) {
  auto* g = static_cast<graph::Graph*>(h);
  const auto cache = cache_from_map(device_map, g->num_nodes, 1);
  train::ModelSpec spec;
  spec.feat_dim = g->feat_dim;
  spec.hidden_dim = hdim;
  spec.num_classes = c;
  spec.learning_rate = lr;
  train::Model model = train::init_model(spec, 1);
  const auto ctxs = train::make_worker_contexts(*g, nullptr, cache);
  const auto batches = train::plan_epoch_batches(ctxs[0].train_nodes, 0, batch_size, hash2(rng_seed, 0));
  const auto nb = static_cast<std::uint32_t>(batches.size());
  warmup = std::min(warmup, nb);
  units = std::min<std::uint32_t>(units, nb - warmup);
  cache::CacheAccounting acc(1);
  auto sample_unit = [&](std::uint32_t step) {
    sampling::SamplerConfig cfg;
    cfg.fanouts.assign(fanouts, fanouts + num_layers);
    cfg.bias_rate = gamma;
    cfg.rng_seed = train::sampling_seed(rng_seed, 0, step, 0);
    return sampling::sample_khop(*g, batches[step], cfg, cache);
  };
  std::uint64_t seeds = 0;
  auto train_unit = [&](const sampling::SampleBatch& batch, const std::vector<float>& feats) {
    const auto fwd = train::forward(model, batch, feats.data());
    std::vector<std::uint32_t> labels(batch.num_seed_unique);
    for (std::size_t s = 0; s < batch.num_seed_unique; ++s) labels[s] = g->labels[batch.unique_nodes[s]];
    std::vector<train::Gradients> grads(1);
    train::backward(model, batch, feats.data(), fwd, labels, grads[0]);
    train::sgd_step(model, train::sync_gradients(grads), spec.learning_rate);
    seeds += batch.seeds.size();
  };
  auto run = [&](std::uint32_t first, std::uint32_t count) {
    if (mode == 0 || producers == 0) {
      for (std::uint32_t s = first; s < first + count; ++s) {
        const auto batch = sample_unit(s);
        auto [feats, stats] = cache::retrieve_features(batch, cache, *g, acc);
        train_unit(batch, feats);
      }
      return;
    }
    const bool producers_retrieve = mode == 1;
    struct Item {
      sampling::SampleBatch batch;
      std::vector<float> feats;
    };
    std::mutex mu;
    std::condition_variable cv_item, cv_space;
    std::map<std::uint32_t, Item> buf;
    std::uint32_t next = 0;
    std::atomic<std::uint32_t> next_unit{0};
    auto producer = [&] {
      for (;;) {
        const std::uint32_t seq = next_unit.fetch_add(1);
        if (seq >= count) return;
        Item it;
        it.batch = sample_unit(first + seq);
        if (producers_retrieve) it.feats = cache::retrieve_features(it.batch, cache, *g, acc).first;
        std::unique_lock lk(mu);
        cv_space.wait(lk, [&] { return seq < next + queue_capacity; });
        buf.emplace(seq, std::move(it));
        cv_item.notify_all();
      }
    };
    std::vector<std::thread> th;
    for (std::uint32_t i = 0; i < producers; ++i) th.emplace_back(producer);
    for (std::uint32_t seq = 0; seq < count; ++seq) {
      Item it;
      {
        std::unique_lock lk(mu);
        cv_item.wait(lk, [&] { return buf.count(seq) > 0; });
        auto node = buf.extract(seq);
        it = std::move(node.mapped());
        ++next;
        cv_space.notify_all();
      }
      if (!producers_retrieve) it.feats = cache::retrieve_features(it.batch, cache, *g, acc).first;
      train_unit(it.batch, it.feats);
    }
    for (auto& t : th) t.join();
  };
  run(0, warmup);
  seeds = 0;
  const auto t0 = std::chrono::steady_clock::now();
  run(warmup, units);
  *seeds_out = seeds;
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"
