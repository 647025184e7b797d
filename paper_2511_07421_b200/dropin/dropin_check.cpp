// dropin_check.cpp -- TEST DRIVER of the C++ drop-in. Written against the
// reference's public API only; run three ways (tests/test_dropin.py):
//   plain                          the reference alone (CPU)
//   LD_PRELOAD=liba3gnn_b200_sampling.so   sample_khop / retrieve_features /
//                                  build_static_cache interposed with the
//                                  device path inside the reference's own
//                                  train() and execute_pipeline()
//   LD_PRELOAD=liba3gnn_b200.so    additionally train() / evaluate_full_graph
// and prints one line per result so the runs can be compared.
#include <cstdio>
#include <cstring>
#include <string>

#include "a3gnn/cache.hpp"
#include "a3gnn/generators.hpp"
#include "a3gnn/pipeline.hpp"
#include "a3gnn/sampler.hpp"
#include "a3gnn/trainer.hpp"

using namespace a3gnn;

static std::uint64_t fnv(const void* p, std::size_t n, std::uint64_t h = 1469598103934665603ull) {
  const auto* b = static_cast<const unsigned char*>(p);
  for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

int main(int argc, char** argv) {
  const std::uint64_t n = argc > 1 ? std::stoull(argv[1]) : 20000;
  const graph::Graph g = graph::generate_power_law(n, 3, 2.5, 32, 1);
  cache::CacheConfig cc;
  cc.volume_bytes = (n / 5) * g.feat_dim * 4;
  const cache::CacheState cache = cache::build_static_cache(g, cc);
  std::printf("cache total=%llu hash=%016llx\n", (unsigned long long)cache.total_cached(),
              (unsigned long long)fnv(cache.device_map.data(), cache.device_map.size() * 4));
  // sampled batches + gathered rows
  cache::CacheAccounting acc(1);
  const auto batches = train::plan_epoch_batches(train::make_worker_contexts(g, nullptr, cache)[0].train_nodes, 0,
                                                 256, 7);
  for (int i = 0; i < 4; ++i) {
    sampling::SamplerConfig cfg;
    cfg.fanouts = {10, 5, 3};
    cfg.bias_rate = i % 2 ? 8.0 : 1.0;
    cfg.kind = i == 3 ? sampling::SamplerKind::uniform_baseline : sampling::SamplerKind::weighted_reservoir;
    cfg.rng_seed = train::sampling_seed(1, 0, i, 0);
    const auto b = sampling::sample_khop(g, batches[i], cfg, cache);
    std::uint64_t h = fnv(b.unique_nodes.data(), b.unique_nodes.size() * 4);
    for (const auto& l : b.layers) h = fnv(l.edges.data(), l.edges.size() * 8, h);
    const auto [feats, st] = cache::retrieve_features(b, cache, g, acc);
    std::printf("batch %d unique=%zu edges=%llu dups=%llu hash=%016llx feats=%016llx bytes=%llu\n", i,
                b.unique_nodes.size(), (unsigned long long)b.total_edges(),
                (unsigned long long)b.num_duplicates_removed, (unsigned long long)h,
                (unsigned long long)fnv(feats.data(), feats.size() * 4), (unsigned long long)st.batch_bytes);
  }
  std::printf("hit_rate %.17g\n", cache::hit_rate(acc));
  // lookup over a 2-device placement: per-id devices and per-device hits
  {
    cache::CacheConfig c2;
    c2.volume_bytes = (n / 10) * g.feat_dim * 4;
    c2.num_devices = 2;
    const cache::CacheState two = cache::build_static_cache(g, c2);
    cache::CacheAccounting acc2(2);
    std::vector<NodeId> ids;
    for (NodeId v = 0; v < n; v += 7) ids.push_back(v);
    const auto dev = cache::lookup(two, ids, acc2);
    std::printf("lookup2 %016llx hits=%llu misses=%llu d0=%llu d1=%llu lists=%zu,%zu bytes=%llu\n",
                (unsigned long long)fnv(dev.data(), dev.size() * 4), (unsigned long long)acc2.hits.load(),
                (unsigned long long)acc2.misses.load(), (unsigned long long)acc2.per_device_hits[0].load(),
                (unsigned long long)acc2.per_device_hits[1].load(), two.cached_per_device[0].size(),
                two.cached_per_device[1].size(), (unsigned long long)two.bytes_used[1]);
  }
  // a fresh CacheState per design point in the same stack slot (surrogate.cpp:272):
  // every sample must see its own cached set
  for (int k = 1; k <= 3; ++k) {
    cache::CacheConfig ck;
    ck.volume_bytes = (n * k / 8) * g.feat_dim * 4;
    const cache::CacheState cs = cache::build_static_cache(g, ck);
    sampling::SamplerConfig cfg;
    cfg.fanouts = {10, 5};
    cfg.bias_rate = 8.0;
    cfg.rng_seed = 11;
    const auto b = sampling::sample_khop(g, batches[0], cfg, cs);
    std::uint64_t h = fnv(b.unique_nodes.data(), b.unique_nodes.size() * 4);
    for (const auto& l : b.layers) h = fnv(l.edges.data(), l.edges.size() * 8, h);
    std::printf("design %d unique=%zu hash=%016llx\n", k, b.unique_nodes.size(), (unsigned long long)h);
  }
  // reservoir on one list, with the caller's stream advanced like the reference
  {
    std::vector<NodeId> nb(300);
    std::vector<double> w(300);
    for (int i = 0; i < 300; ++i) {
      nb[i] = i * 3;
      w[i] = i % 3 ? 1.0 : 4.0;
    }
    RngStream r(5, 9);
    const auto a = sampling::weighted_reservoir_sample(nb, w, 12, r);
    const auto b = sampling::uniform_reservoir_sample(nb, 12, r);
    std::printf("reservoirs %016llx %016llx draws=%llu next=%016llx\n",
                (unsigned long long)fnv(a.data(), a.size() * 4), (unsigned long long)fnv(b.data(), b.size() * 4),
                (unsigned long long)r.draws(), (unsigned long long)r.next_u64());
  }
  // error mapping (ParameterError, in the reference's order)
  try {
    sampling::SamplerConfig cfg;
    cfg.fanouts = {5};
    cfg.bias_rate = 0.5;
    sampling::sample_khop(g, {1, 2}, cfg, cache);
    std::printf("error none\n");
  } catch (const ParameterError& e) {
    std::printf("error ParameterError %s\n", e.what());
  }
  // train(): the reference's loop, or the device loop when interposed
  train::ModelSpec spec;
  spec.feat_dim = g.feat_dim;
  spec.hidden_dim = 16;
  spec.num_classes = 4;
  sampling::SamplerConfig scfg;
  scfg.fanouts = {10, 5};
  scfg.bias_rate = 8.0;
  scfg.rng_seed = 3;
  train::TrainOptions opts;
  opts.batch_size = 512;
  opts.epochs = 2;
  const auto rep = train::train(g, spec, scfg, cache, opts);
  for (std::size_t e = 0; e < rep.loss_curve.size(); ++e)
    std::printf("train epoch %zu loss %.17g hit %.17g\n", e, rep.loss_curve[e], rep.epoch_hit_rates[e]);
  std::printf("train accuracy %.17g batch_bytes %llu act_bytes %llu\n", rep.test_accuracy,
              (unsigned long long)rep.max_batch_bytes, (unsigned long long)rep.max_activation_bytes);
  // partitioned workers (u = 2, hash partitions with halos, localized caches)
  {
    train::TrainOptions o2 = opts;
    o2.u = 2;
    o2.epochs = 1;
    const auto r2 = train::train(g, spec, scfg, cache, o2);
    for (std::size_t e = 0; e < r2.loss_curve.size(); ++e)
      std::printf("train_u2 epoch %zu loss %.17g hit %.17g\n", e, r2.loss_curve[e], r2.epoch_hit_rates[e]);
    std::printf("train_u2 accuracy %.17g batch_bytes %llu act_bytes %llu\n", r2.test_accuracy,
                (unsigned long long)r2.max_batch_bytes, (unsigned long long)r2.max_activation_bytes);
    ResolvedDesign d;
    d.batch_size = 512;
    d.partitions = 2;
    d.bias_rate = 8.0;
    d.workers = 2;
    d.cache_volume = cc.volume_bytes;
    d.mode = Mode::pmode1;
    pipeline::PlatformSpec plat;
    pipeline::ExecOptions eo;
    eo.epochs = 1;
    sampling::SamplerConfig pcfg;
    pcfg.fanouts = {10, 5};
    pcfg.rng_seed = 3;
    const auto ex = pipeline::execute_pipeline(g, d, plat, spec, pcfg, eo);
    std::printf("pipeline_p2 accuracy %.17g hit %.17g batch_bytes %llu model_bytes %llu\n", ex.metrics.accuracy,
                ex.hit_rate, (unsigned long long)ex.batch_bytes_max, (unsigned long long)ex.model_bytes);
    const auto c = pipeline::profile_stage_costs(g, d, plat, spec, pcfg, 4);
    std::printf("profile_p2 iters %llu positive %d\n", (unsigned long long)c.iters_per_epoch,
                c.t_sample > 0 && c.t_batch > 0 && c.t_train > 0 ? 1 : 0);
  }
  // the per-batch model entry points on one explicit batch (trainer.cpp:59-239)
  {
    sampling::SamplerConfig cfg;
    cfg.fanouts = {10, 5};
    cfg.bias_rate = 8.0;
    cfg.rng_seed = train::sampling_seed(3, 0, 0, 0);
    const auto b = sampling::sample_khop(g, batches[1], cfg, cache);
    cache::CacheAccounting a1(1);
    const auto feats = cache::retrieve_features(b, cache, g, a1).first;
    const train::Model m = train::init_model(spec, 1);
    const auto fwd = train::forward(m, b, feats.data());
    double lsum = 0, asum = 0, hsum = 0;
    for (double x : fwd.logits) lsum += x * x;
    for (double x : fwd.agg_inner) asum += x * x;
    for (double x : fwd.h1) hsum += x * x;
    std::uint64_t ih = fnv(fwd.inner_nodes.data(), fwd.inner_nodes.size() * 4);
    ih = fnv(fwd.inner_pos.data(), fwd.inner_pos.size() * 4, ih);
    std::uint64_t dh = fnv(fwd.inner_deg.data(), fwd.inner_deg.size() * 4);
    dh = fnv(fwd.outer_deg.data(), fwd.outer_deg.size() * 4, dh);
    std::printf("model forward n_inner %zu inner %016llx deg %016llx act %llu logits2 %.17g agg2 %.17g h12 %.17g\n",
                fwd.inner_nodes.size(), (unsigned long long)ih, (unsigned long long)dh,
                (unsigned long long)fwd.activation_bytes, lsum, asum, hsum);
    std::vector<std::uint32_t> labels(b.num_seed_unique);
    for (std::size_t i = 0; i < labels.size(); ++i) labels[i] = g.labels[b.unique_nodes[i]];
    train::Gradients gb, gg;
    const double lb = train::backward(m, b, feats.data(), fwd, labels, gb);
    const double lg = train::grad_on_batch(m, g, b, feats.data(), gg);
    double n1 = 0, n2 = 0;
    for (double x : gg.w1) n1 += x * x;
    for (double x : gg.w2) n2 += x * x;
    std::printf("model grad loss %.17g backward_loss %.17g gw1 %.17g gw2 %.17g\n", lg, lb, n1, n2);
    // sync_gradients / sgd_step on fixed inputs (init_model draws): bit-identical
    // to the reference's active kernel table
    const train::Model ma = train::init_model(spec, 11), mb = train::init_model(spec, 12);
    train::Gradients x, y;
    x.w1 = ma.w1;
    x.w2 = ma.w2;
    y.w1 = mb.w1;
    y.w2 = mb.w2;
    const auto mean = train::sync_gradients({x, y, x});
    train::Model m2 = m;
    train::sgd_step(m2, mean, 0.2);
    std::printf("sync %016llx sgd %016llx %016llx\n", (unsigned long long)fnv(mean.w1.data(), mean.w1.size() * 8,
                                                                               fnv(mean.w2.data(), mean.w2.size() * 8)),
                (unsigned long long)fnv(m2.w1.data(), m2.w1.size() * 8),
                (unsigned long long)fnv(m2.w2.data(), m2.w2.size() * 8));
    try {
      train::sync_gradients({});
    } catch (const ParameterError& e) {
      std::printf("error ParameterError %s\n", e.what());
    }
  }
  // profile_stage_costs: the three stage medians the analytic model consumes
  {
    ResolvedDesign d;
    d.batch_size = 512;
    d.bias_rate = 8.0;
    d.cache_volume = cc.volume_bytes;
    pipeline::PlatformSpec plat;
    sampling::SamplerConfig pcfg;
    pcfg.fanouts = {10, 5};
    pcfg.rng_seed = 3;
    const auto c = pipeline::profile_stage_costs(g, d, plat, spec, pcfg, 3);
    std::printf("profile iters %llu positive %d\n", (unsigned long long)c.iters_per_epoch,
                c.t_sample > 0 && c.t_batch > 0 && c.t_train > 0 ? 1 : 0);
  }
  // execute_pipeline in the three modes (sequential; pmode1 / pmode2 with 4 workers)
  for (Mode mode : {Mode::sequential, Mode::pmode2}) {
    ResolvedDesign d;
    d.batch_size = 512;
    d.bias_rate = 8.0;
    d.workers = 4;
    d.cache_volume = cc.volume_bytes;
    d.mode = mode;
    pipeline::PlatformSpec plat;
    pipeline::ExecOptions eo;
    eo.epochs = 1;
    sampling::SamplerConfig pcfg;
    pcfg.fanouts = {10, 5};
    pcfg.rng_seed = 3;
    const auto ex = pipeline::execute_pipeline(g, d, plat, spec, pcfg, eo);
    std::printf("pipeline %s accuracy %.17g hit %.17g batch_bytes %llu model_bytes %llu\n", to_string(mode).c_str(),
                ex.metrics.accuracy, ex.hit_rate, (unsigned long long)ex.batch_bytes_max,
                (unsigned long long)ex.model_bytes);
  }
  // execute_pipeline pmode1 with 4 producer threads: concurrent sample_khop
  ResolvedDesign d;
  d.batch_size = 512;
  d.bias_rate = 8.0;
  d.workers = 4;
  d.cache_volume = cc.volume_bytes;
  d.mode = Mode::pmode1;
  pipeline::PlatformSpec plat;
  pipeline::ExecOptions eo;
  eo.epochs = 1;
  sampling::SamplerConfig pcfg;
  pcfg.fanouts = {10, 5};
  pcfg.rng_seed = 3;
  const auto ex = pipeline::execute_pipeline(g, d, plat, spec, pcfg, eo);
  std::printf("pipeline accuracy %.17g hit %.17g\n", ex.metrics.accuracy, ex.hit_rate);
  return 0;
}
