// host_graph.cpp -- host-side graph synthesis and A3G1 I/O.
//
// generate_power_law (proj/src/generators.cpp:79-149, + fill_features_and_masks
// :12-40) restated so that the output is bit-identical to the reference's
// sequential generator, but multithreaded: every draw is counter-indexed
// (rng.hpp:43-46), so degrees, Gaussian feature noise and target draws are
// computed in parallel; only the rejection walk over target draws
// (generators.cpp:113-139) and the Fisher-Yates split (:28-29) stay
// sequential. Uses the same libm calls (pow/log/cos/sqrt) as the reference.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "a3g_internal.cuh"

namespace a3g {
namespace {

struct Stream {
  uint64_t key;
  explicit Stream(uint64_t seed, uint64_t stream) : key(hash2(seed, stream)) {}
  Stream sub(uint64_t id) const {  // rng.hpp:37-41
    Stream s(0, 0);
    s.key = hash2(key, id ^ 0xd6e8feb86659fd93ull);
    return s;
  }
  double unit(uint64_t i) const { return unit_of(draw(key, i)); }
};

template <typename F>
void parallel_for(uint64_t n, int threads, F&& fn) {
  if (threads <= 1 || n < 4096) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> th;
  const uint64_t per = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const uint64_t b = t * per, e = std::min<uint64_t>(n, b + per);
    if (b >= e) break;
    th.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& x : th) x.join();
}

a3g_host_graph* alloc_host(uint64_t n, uint64_t m, uint32_t f) {
  auto* g = new a3g_host_graph{};
  g->num_nodes = n;
  g->num_edges = m;
  g->feat_dim = f;
  g->row_offsets = new uint64_t[n + 1]();
  g->col_indices = new uint32_t[m > 0 ? m : 1]();
  g->features = new float[n * f > 0 ? n * f : 1]();
  g->labels = new uint32_t[n > 0 ? n : 1]();
  g->train_mask = new uint8_t[n > 0 ? n : 1]();
  g->test_mask = new uint8_t[n > 0 ? n : 1]();
  return g;
}

// generators.cpp:12-40
void fill_features_and_masks(a3g_host_graph* g, const Stream& rng, int threads) {
  const uint32_t f = g->feat_dim;
  const uint64_t n = g->num_nodes;
  const Stream noise = rng.sub(0xfea7);
  parallel_for(n, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v) {
      float* row = g->features + v * f;
      uint64_t ctr = 2 * v * f;  // each Gaussian uses two draws (rng.hpp:60-65)
      for (uint32_t d = 0; d < f; ++d) {
        double u1 = noise.unit(++ctr);
        const double u2 = noise.unit(++ctr);
        if (u1 <= 0.0) u1 = 0x1.0p-53;
        row[d] = static_cast<float>(std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925 * u2));
      }
      row[g->labels[v] % f] += 1.0f;
    }
  });
  std::vector<uint32_t> order(n);
  std::iota(order.begin(), order.end(), 0u);
  const Stream split = rng.sub(0x5411);
  uint64_t ctr = 0;
  for (uint64_t i = n; i > 1; --i) {  // rng.hpp:69-74
    const uint64_t j = static_cast<uint64_t>(
        (static_cast<unsigned __int128>(draw(split.key, ++ctr)) * static_cast<uint32_t>(i)) >> 64);
    std::swap(order[i - 1], order[j]);
  }
  const uint64_t n_train = (n * 6) / 10;
  for (uint64_t i = 0; i < n; ++i) {
    if (i < n_train)
      g->train_mask[order[i]] = 1;
    else
      g->test_mask[order[i]] = 1;
  }
}

}  // namespace

a3g_host_graph* power_law(uint64_t n, uint32_t min_degree, double exponent, uint32_t f, uint64_t seed,
                          int threads) {
  if (exponent <= 1.0) raise(A3G_ERR_PARAMETER, "generate_power_law: exponent must be > 1");
  if (min_degree < 1) raise(A3G_ERR_PARAMETER, "generate_power_law: min_degree must be >= 1");
  if (f < 1) raise(A3G_ERR_PARAMETER, "generate_power_law: feat_dim must be >= 1");
  if (n < 2) raise(A3G_ERR_PARAMETER, "generate_power_law: need at least 2 nodes");
  if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const Stream rng(seed, 0x97a3);
  const Stream deg_rng = rng.sub(0xde6);
  const uint64_t cap = n - 1;
  std::vector<uint64_t> degree(n);
  parallel_for(n, threads, [&](uint64_t b, uint64_t e) {  // generators.cpp:90-98
    for (uint64_t v = b; v < e; ++v) {
      double u = deg_rng.unit(v + 1);
      if (u <= 0.0) u = 0x1.0p-53;
      const double d = std::floor(min_degree * std::pow(u, -1.0 / (exponent - 1.0)));
      degree[v] = std::min<uint64_t>(cap, std::max<uint64_t>(min_degree, static_cast<uint64_t>(d)));
    }
  });
  // cumulative of (deg+1): sums of integers < 2^53 are exact in fp64, so the
  // integer prefix sum equals the reference's sequential fp64 accumulation.
  std::vector<double> cumulative(n);
  uint64_t acc = 0;
  for (uint64_t v = 0; v < n; ++v) {
    acc += degree[v] + 1;
    cumulative[v] = static_cast<double>(acc);
  }
  if (acc >= (1ull << 53)) raise(A3G_ERR_PARAMETER, "generate_power_law: graph too large for exact cumulative");
  const double total = static_cast<double>(acc);
  uint64_t m = 0;
  for (uint64_t v = 0; v < n; ++v) m += degree[v];
  a3g_host_graph* g = alloc_host(n, m, f);
  for (uint64_t v = 0; v < n; ++v) g->row_offsets[v + 1] = g->row_offsets[v] + degree[v];

  // Target draws of pick_rng (generators.cpp:113-139), computed ahead in
  // parallel blocks; the rejection walk consumes them in draw order.
  const Stream pick = rng.sub(0x91c4);
  const uint64_t kBlock = 1ull << 22;
  std::vector<uint32_t> targets(kBlock);
  uint64_t block_first = 1, block_end = 1;  // draw numbers [first, end) held in targets
  auto refill = [&](uint64_t first) {
    parallel_for(kBlock, threads, [&](uint64_t b, uint64_t e) {
      for (uint64_t i = b; i < e; ++i) {
        const double r = pick.unit(first + i) * total;
        targets[i] = static_cast<uint32_t>(std::lower_bound(cumulative.begin(), cumulative.end(), r) -
                                           cumulative.begin());
      }
    });
    block_first = first;
    block_end = first + kBlock;
  };
  uint64_t next_draw = 1;
  std::vector<uint8_t> used(n, 0);
  for (uint64_t src = 0; src < n; ++src) {
    const uint64_t want = degree[src];
    uint32_t* chosen = g->col_indices + g->row_offsets[src];
    uint64_t nch = 0, attempts = 0;
    const uint64_t max_attempts = 30 * want + 64;
    while (nch < want && attempts < max_attempts) {
      ++attempts;
      if (next_draw >= block_end) refill(next_draw);
      const uint32_t t = targets[next_draw - block_first];
      ++next_draw;
      if (t == src || used[t]) continue;
      used[t] = 1;
      chosen[nch++] = t;
    }
    if (nch < want) {  // dense saturation: scan in order (generators.cpp:127-133)
      for (uint64_t t = 0; t < n && nch < want; ++t) {
        if (t == src || used[t]) continue;
        used[t] = 1;
        chosen[nch++] = static_cast<uint32_t>(t);
      }
    }
    for (uint64_t i = 0; i < nch; ++i) used[chosen[i]] = 0;
  }
  // from_edges sorts (src,dst): rows ascending (graph.cpp:66)
  parallel_for(n, threads, [&](uint64_t b, uint64_t e) {
    for (uint64_t v = b; v < e; ++v)
      std::sort(g->col_indices + g->row_offsets[v], g->col_indices + g->row_offsets[v + 1]);
  });
  for (uint64_t v = 0; v < n; ++v) g->labels[v] = static_cast<uint32_t>(mix64(v ^ 0xabcd) % 4);
  fill_features_and_masks(g, rng, threads);
  return g;
}

a3g_host_graph* from_edges(uint64_t n, const uint32_t* src, const uint32_t* dst, uint64_t m, uint32_t f) {
  std::vector<std::pair<uint32_t, uint32_t>> e(m);
  for (uint64_t i = 0; i < m; ++i) {
    if (src[i] >= n || dst[i] >= n) raise(A3G_ERR_PARAMETER, "from_edges: endpoint out of range");
    e[i] = {src[i], dst[i]};
  }
  std::sort(e.begin(), e.end());
  a3g_host_graph* g = alloc_host(n, m, f);
  for (const auto& p : e) ++g->row_offsets[p.first + 1];
  for (uint64_t i = 1; i <= n; ++i) g->row_offsets[i] += g->row_offsets[i - 1];
  for (uint64_t i = 0; i < m; ++i) g->col_indices[i] = e[i].second;
  return g;
}

void free_host(a3g_host_graph* g) {
  if (!g) return;
  delete[] g->row_offsets;
  delete[] g->col_indices;
  delete[] g->features;
  delete[] g->labels;
  delete[] g->train_mask;
  delete[] g->test_mask;
  delete g;
}

// graph_io.cpp:40-58 (format graph_io.hpp:3-7)
void save_host(const a3g_host_graph* g, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) raise(A3G_ERR_IO, "save_graph: cannot open " + path);
  out.write("A3G1", 4);
  out.write(reinterpret_cast<const char*>(&g->num_nodes), 8);
  out.write(reinterpret_cast<const char*>(&g->num_edges), 8);
  out.write(reinterpret_cast<const char*>(&g->feat_dim), 4);
  const uint64_t n = g->num_nodes;
  out.write(reinterpret_cast<const char*>(g->row_offsets), (n + 1) * 8);
  out.write(reinterpret_cast<const char*>(g->col_indices), g->num_edges * 4);
  out.write(reinterpret_cast<const char*>(g->features), n * g->feat_dim * 4);
  out.write(reinterpret_cast<const char*>(g->labels), n * 4);
  std::vector<uint8_t> masks(n);
  for (uint64_t v = 0; v < n; ++v)
    masks[v] = static_cast<uint8_t>((g->train_mask[v] ? 1 : 0) | (g->test_mask[v] ? 2 : 0));
  out.write(reinterpret_cast<const char*>(masks.data()), n);
  if (!out) raise(A3G_ERR_IO, "save_graph: write failed for " + path);
}

// graph_io.cpp:60-87 (+ validate, graph.cpp:13-40)
a3g_host_graph* load_host(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) raise(A3G_ERR_IO, "load_graph: cannot open " + path);
  char magic[4];
  in.read(magic, 4);
  if (!in || std::memcmp(magic, "A3G1", 4) != 0) raise(A3G_ERR_IO, "load_graph: bad magic in " + path);
  uint64_t n = 0, m = 0;
  uint32_t f = 0;
  in.read(reinterpret_cast<char*>(&n), 8);
  in.read(reinterpret_cast<char*>(&m), 8);
  in.read(reinterpret_cast<char*>(&f), 4);
  if (!in) raise(A3G_ERR_IO, "load_graph: truncated file " + path);
  a3g_host_graph* g = alloc_host(n, m, f);
  in.read(reinterpret_cast<char*>(g->row_offsets), (n + 1) * 8);
  in.read(reinterpret_cast<char*>(g->col_indices), m * 4);
  in.read(reinterpret_cast<char*>(g->features), n * f * 4);
  in.read(reinterpret_cast<char*>(g->labels), n * 4);
  std::vector<uint8_t> masks(n);
  in.read(reinterpret_cast<char*>(masks.data()), n);
  if (!in) {
    free_host(g);
    raise(A3G_ERR_IO, "load_graph: truncated file " + path);
  }
  for (uint64_t v = 0; v < n; ++v) {
    g->train_mask[v] = masks[v] & 1;
    g->test_mask[v] = (masks[v] >> 1) & 1;
  }
  // validate (graph.cpp:13-40)
  if (f < 1 || g->row_offsets[0] != 0 || g->row_offsets[n] != m) {
    free_host(g);
    raise(A3G_ERR_PARAMETER, "graph: CSR invariant violated");
  }
  for (uint64_t i = 0; i < n; ++i)
    if (g->row_offsets[i] > g->row_offsets[i + 1]) {
      free_host(g);
      raise(A3G_ERR_PARAMETER, "graph: row_offsets not non-decreasing");
    }
  for (uint64_t i = 0; i < m; ++i)
    if (g->col_indices[i] >= n) {
      free_host(g);
      raise(A3G_ERR_PARAMETER, "graph: col_index out of range");
    }
  return g;
}

}  // namespace a3g
