// registry.cpp -- device copies of reference objects for the C++ drop-in.
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <tuple>

#include "dropin.hpp"

namespace a3gnn::b200 {
namespace {

struct GraphKey {
  const void* obj;
  const void* col;
  const void* feat;
  std::uint64_t n, m;
  bool operator<(const GraphKey& o) const {
    return std::tie(obj, col, feat, n, m) < std::tie(o.obj, o.col, o.feat, o.n, o.m);
  }
};

struct Registry {
  std::mutex mu;
  std::map<GraphKey, a3g_graph*> graphs;
  std::map<std::tuple<a3g_graph*, const void*, const void*, std::size_t>, a3g_cache*> caches;
  std::uint64_t generation = 0;  // bumped by release(): invalidates thread arenas
  ~Registry() {
    for (auto& [k, c] : caches) a3g_cache_destroy(c);
    for (auto& [k, g] : graphs) a3g_graph_destroy(g);
  }
};
Registry& reg() {
  static Registry r;
  return r;
}

GraphKey key_of(const graph::Graph& g) {
  return GraphKey{&g, g.col_indices.data(), g.features.data(), g.num_nodes, g.num_edges};
}

struct Arena {
  a3g_sampler* s = nullptr;
  std::uint32_t cap = 0;
  std::vector<std::uint32_t> fanouts;
  std::uint64_t generation = 0;
};
struct ThreadArenas {
  std::map<std::pair<a3g_graph*, a3g_cache*>, Arena> m;
  ~ThreadArenas() {
    for (auto& [k, a] : m) a3g_sampler_destroy(a.s);
  }
};
thread_local ThreadArenas t_arenas;

}  // namespace

[[noreturn]] void raise_status(a3g_status st) {
  const std::string msg = a3g_last_error();
  switch (st) {
    case A3G_ERR_PARAMETER: throw ParameterError(msg);
    case A3G_ERR_LOOKUP: throw LookupError(msg);
    case A3G_ERR_CONFIG: throw ConfigError(msg);
    case A3G_ERR_IO: throw IoError(msg);
    case A3G_ERR_OOM: throw std::bad_alloc();
    default: throw std::runtime_error("a3gnn-b200 (CUDA/NCCL): " + msg);
  }
}

int device() {
  static const int d = [] {
    const char* e = std::getenv("A3GNN_B200_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return d;
}

a3g_graph* device_graph(const graph::Graph& g) {
  Registry& r = reg();
  std::lock_guard<std::mutex> lk(r.mu);
  const GraphKey k = key_of(g);
  auto it = r.graphs.find(k);
  if (it != r.graphs.end()) return it->second;
  a3g_graph* h = nullptr;
  check(a3g_graph_create(device(), g.num_nodes, g.num_edges, g.feat_dim, g.row_offsets.data(),
                         g.col_indices.data(), g.features.empty() ? nullptr : g.features.data(), A3G_FEAT_F32,
                         g.labels.size() == g.num_nodes ? g.labels.data() : nullptr, &h));
  r.graphs.emplace(k, h);
  return h;
}

a3g_cache* device_cache(const graph::Graph& g, const cache::CacheState& c) {
  a3g_graph* dg = device_graph(g);
  Registry& r = reg();
  std::lock_guard<std::mutex> lk(r.mu);
  const auto k = std::make_tuple(dg, static_cast<const void*>(&c), static_cast<const void*>(c.device_map.data()),
                                 c.device_map.size());
  auto it = r.caches.find(k);
  if (it != r.caches.end()) return it->second;
  if (c.device_map.size() != g.num_nodes && !c.device_map.empty())
    throw ParameterError("cache: device_map size does not match the graph");
  a3g_cache* h = nullptr;
  const std::uint32_t nd = static_cast<std::uint32_t>(std::max<std::size_t>(1, c.cached_per_device.size()));
  check(a3g_cache_from_map(dg, c.device_map.empty() ? nullptr : c.device_map.data(), nd, &h));
  r.caches.emplace(k, h);
  return h;
}

a3g_sampler* thread_sampler(a3g_graph* g, a3g_cache* c, std::uint32_t n_seeds,
                            const std::vector<std::uint32_t>& fanouts) {
  const std::uint64_t gen = [] {
    std::lock_guard<std::mutex> lk(reg().mu);
    return reg().generation;
  }();
  Arena& a = t_arenas.m[{g, c}];
  if (a.s && (a.cap < n_seeds || a.fanouts != fanouts || a.generation != gen)) {
    a3g_sampler_destroy(a.s);
    a.s = nullptr;
  }
  if (!a.s) {
    const std::uint32_t cap = std::max<std::uint32_t>(n_seeds, std::max<std::uint32_t>(a.cap, 1));
    check(a3g_sampler_create(g, c, cap, fanouts.data(), static_cast<std::uint32_t>(fanouts.size()), &a.s));
    a.cap = cap;
    a.fanouts = fanouts;
    a.generation = gen;
  }
  return a.s;
}

void release(const graph::Graph& g) {
  Registry& r = reg();
  std::lock_guard<std::mutex> lk(r.mu);
  auto it = r.graphs.find(key_of(g));
  if (it == r.graphs.end()) return;
  for (auto c = r.caches.begin(); c != r.caches.end();) {
    if (std::get<0>(c->first) == it->second) {
      a3g_cache_destroy(c->second);
      c = r.caches.erase(c);
    } else {
      ++c;
    }
  }
  ++r.generation;
  // arenas of other threads still reference the graph until their next call
  // notices the generation; the reference never releases a graph mid-run
  a3g_graph_destroy(it->second);
  r.graphs.erase(it);
}

}  // namespace a3gnn::b200
