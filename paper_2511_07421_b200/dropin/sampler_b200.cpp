// sampler_b200.cpp -- drop-in for proj/src/sampler.cpp (sampler.hpp:48-69):
// the same declarations, executed by the sm_100a sampler through the C-ABI.
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "a3gnn/sampler.hpp"
#include "dropin.hpp"

namespace a3gnn::sampling {
namespace {

// RngStream keeps (key, counter, draws) private (rng.hpp:79-82); the device
// reservoirs need the key and counter and must advance the caller's stream
// exactly as the reference does (one draw per neighbour for the weighted
// reservoir, one per position >= m for Algorithm R).
static_assert(std::is_standard_layout_v<RngStream> && sizeof(RngStream) == 3 * sizeof(std::uint64_t),
              "RngStream layout (rng.hpp:79-82) changed");
struct RngState {
  std::uint64_t key, counter, draws;
};
RngState state_of(const RngStream& r) {
  RngState s;
  std::memcpy(&s, &r, sizeof s);
  return s;
}
void advance(RngStream& r, std::uint64_t n) {
  RngState s = state_of(r);
  s.counter += n;
  s.draws += n;
  std::memcpy(static_cast<void*>(&r), &s, sizeof s);
}

}  // namespace

std::vector<NodeId> weighted_reservoir_sample(std::span<const NodeId> neighbors, std::span<const double> weights,
                                              std::uint32_t m, RngStream& rng) {
  if (neighbors.size() != weights.size())
    throw ParameterError("weighted_reservoir_sample: |neighbors| != |weights|");
  if (m < 1) throw ParameterError("weighted_reservoir_sample: m must be >= 1");
  if (neighbors.empty()) return {};
  const RngState s = state_of(rng);
  std::vector<NodeId> out(std::min<std::size_t>(m, neighbors.size()));
  std::uint64_t cnt = 0;
  b200::check(a3g_weighted_reservoir(neighbors.data(), weights.data(), neighbors.size(), m, s.key, s.counter,
                                     out.data(), &cnt));
  out.resize(cnt);
  advance(rng, neighbors.size());
  return out;
}

std::vector<NodeId> uniform_reservoir_sample(std::span<const NodeId> neighbors, std::uint32_t m, RngStream& rng) {
  if (m < 1) throw ParameterError("uniform_reservoir_sample: m must be >= 1");
  if (neighbors.empty()) return {};
  const RngState s = state_of(rng);
  std::vector<NodeId> out(std::min<std::size_t>(m, neighbors.size()));
  std::uint64_t cnt = 0;
  b200::check(a3g_uniform_reservoir(neighbors.data(), neighbors.size(), m, s.key, s.counter, out.data(), &cnt));
  out.resize(cnt);
  if (neighbors.size() > m) advance(rng, neighbors.size() - m);
  return out;
}

// Host utility (the device sampler reads the cached bitmap directly).
std::vector<double> assign_weights(std::span<const NodeId> neighbors, const CacheState& cache, double gamma) {
  if (gamma < 1.0) throw ParameterError("assign_weights: gamma must be >= 1");
  std::vector<double> w(neighbors.size(), 1.0);
  for (std::size_t i = 0; i < neighbors.size(); ++i)
    if (cache.is_cached(neighbors[i])) w[i] = gamma;
  return w;
}

SampleBatch sample_khop(const Graph& g, const std::vector<NodeId>& seeds, const SamplerConfig& cfg,
                        const CacheState& cache) {
  // validation in the reference's order (sampler.cpp:91-94, 110, assign_weights :62)
  if (seeds.empty()) throw ParameterError("sample_khop: seeds must be non-empty");
  bool any_deg = false;
  for (NodeId s : seeds) {
    if (s >= g.num_nodes) throw ParameterError("sample_khop: seed out of range");
    any_deg |= g.out_degree(s) > 0;
  }
  const bool weighted = cfg.kind == SamplerKind::weighted_reservoir;
  for (std::size_t l = 0; l < cfg.fanouts.size(); ++l) {
    if (cfg.fanouts[l] < 1) throw ParameterError("sample_khop: fanout must be >= 1");
    if (l == 0 && weighted && any_deg && cfg.bias_rate < 1.0)
      throw ParameterError("assign_weights: gamma must be >= 1");
  }
  a3g_graph* dg = b200::device_graph(g);
  a3g_cache* dc = b200::device_cache(g, cache);
  a3g_sampler* sm = b200::thread_sampler(dg, dc, static_cast<std::uint32_t>(seeds.size()), cfg.fanouts);
  b200::check(a3g_sample_khop(sm, seeds.data(), static_cast<std::uint32_t>(seeds.size()), 0, cfg.bias_rate,
                              weighted ? A3G_SAMPLER_WEIGHTED : A3G_SAMPLER_UNIFORM, cfg.rng_seed, nullptr));
  const std::size_t L = cfg.fanouts.size();
  std::uint64_t nu = 0, nsu = 0, dups = 0;
  std::vector<std::uint64_t> le(std::max<std::size_t>(L, 1));
  b200::check(a3g_batch_sizes(sm, &nu, &nsu, &dups, le.data()));
  SampleBatch b;
  b.seeds = seeds;
  b.unique_nodes.resize(nu);
  b.num_seed_unique = nsu;
  b.num_duplicates_removed = dups;
  b.layers.resize(L);
  std::vector<std::vector<std::uint32_t>> dst(L), src(L);
  std::vector<std::uint32_t*> pd(L), ps(L);
  for (std::size_t l = 0; l < L; ++l) {
    dst[l].resize(le[l]);
    src[l].resize(le[l]);
    pd[l] = dst[l].data();
    ps[l] = src[l].data();
  }
  b200::check(a3g_batch_copy(sm, b.unique_nodes.data(), pd.data(), ps.data()));
  for (std::size_t l = 0; l < L; ++l) {
    auto& e = b.layers[l].edges;
    e.resize(le[l]);
    for (std::size_t i = 0; i < le[l]; ++i) e[i] = {dst[l][i], src[l][i]};
  }
  return b;
}

double dedup_ratio(const SampleBatch& b) {
  const double d = static_cast<double>(b.num_duplicates_removed);
  return d / (d + static_cast<double>(b.unique_nodes.size()));
}

// Test utility (sampler.cpp:144-165 semantics; sorted-copy uniqueness check).
void validate_batch(const Graph& g, const SampleBatch& b) {
  for (const auto& layer : b.layers) {
    for (const auto& [d, s] : layer.edges) {
      if (d >= b.unique_nodes.size() || s >= b.unique_nodes.size())
        throw ParameterError("validate_batch: edge index out of range");
      const auto nbrs = g.out_neighbors(b.unique_nodes[d]);
      if (!std::binary_search(nbrs.begin(), nbrs.end(), b.unique_nodes[s]))
        throw ParameterError("validate_batch: sampled edge not in CSR");
    }
  }
  std::vector<NodeId> u(b.unique_nodes);
  std::sort(u.begin(), u.end());
  if (std::adjacent_find(u.begin(), u.end()) != u.end())
    throw ParameterError("validate_batch: unique_nodes has repeats");
}

}  // namespace a3gnn::sampling
