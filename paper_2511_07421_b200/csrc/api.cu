// api.cu -- the extern "C" boundary (include/a3g.h): handle lifetimes,
// reference-order validation, status <-> exception mapping, host<->device
// staging. Kernels live in sampler.cu / train.cu.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "trainer.cuh"

namespace a3g {
a3g_host_graph* power_law(uint64_t n, uint32_t min_degree, double exponent, uint32_t f, uint64_t seed,
                          int threads);
a3g_host_graph* from_edges(uint64_t n, const uint32_t* src, const uint32_t* dst, uint64_t m, uint32_t f);
void free_host(a3g_host_graph* g);
void save_host(const a3g_host_graph* g, const std::string& path);
a3g_host_graph* load_host(const std::string& path);
void comm_unique_id(uint8_t out[128]);
a3g_comm* comm_create(const uint8_t id[128], int nranks, int rank, int device);
a3g_comm* comm_create_host(int nranks, int rank, a3g_allreduce_fn fn, void* user);
void comm_destroy(a3g_comm* c);
}  // namespace a3g

using namespace a3g;

namespace a3g {
void set_error(const std::string& msg);
}

namespace {
// The pipeline drives nine streams (eight sampling streams and the compute
// stream); with the default 8 hardware work queues two of them share a queue and serialise behind each other's kernels. Ask for 32
// when the library loads before the process creates its CUDA context (a
// preset value wins; a context that already exists keeps its own). C2 step
// 0.288 -> 0.277 ms at 100 steps (profiles/r02_sampler_experiments.md).
struct HwQueues {
  HwQueues() { setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0); }
} g_hw_queues;
}  // namespace

namespace {
thread_local std::string g_err;
template <typename T>
T* dalloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  A3G_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return static_cast<T*>(p);
}
template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

int sm_count_of(int dev) {
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

void sampler_alloc(SamplerState& s, a3g_graph* g, a3g_cache* c, uint32_t max_seeds, const uint32_t* fanouts,
                   uint32_t L) {
  if (L > static_cast<uint32_t>(kMaxLayers)) raise(A3G_ERR_PARAMETER, "sample_khop: too many layers");
  if (max_seeds < 1) raise(A3G_ERR_PARAMETER, "sample_khop: max_seeds must be >= 1");
  for (uint32_t l = 0; l < L; ++l)
    if (fanouts[l] < 1) raise(A3G_ERR_PARAMETER, "sample_khop: fanout must be >= 1");
  A3G_CUDA(cudaSetDevice(g->device));
  s.g = g;
  s.c = c;
  s.max_seeds = max_seeds;
  s.L = L;
  s.fanouts.assign(fanouts, fanouts + L);
  s.sm_count = sm_count_of(g->device);
  s.device = g->device;
  const uint64_t n = g->n;
  uint64_t rows = std::min<uint64_t>(max_seeds, n);
  uint64_t ucap = rows;
  uint64_t max_pos = 0;
  for (uint32_t l = 0; l < L; ++l) {
    LayerArena& la = s.layer[l];
    la.f = fanouts[l];
    la.cap_rows = rows;
    la.front = dalloc<uint32_t>(rows);
    la.front_idx = dalloc<uint32_t>(rows);
    la.cnt = dalloc<uint32_t>(rows);
    const uint64_t pos = rows * la.f;
    if (pos >= (1ull << 32)) raise(A3G_ERR_PARAMETER, "sample_khop: batch too large for 32-bit positions");
    la.S = dalloc<uint32_t>(pos);
    la.sidx = dalloc<uint32_t>(pos);
    if (la.f > 32) la.scratch = dalloc<double>(pos);
    max_pos = std::max(max_pos, pos);
    ucap += pos;
    if (l == 0) s.cap_inner = std::min<uint64_t>(n, rows + pos);
    rows = std::min<uint64_t>(pos, n);  // next frontier <= edges, <= n
  }
  if (L == 0) s.cap_inner = std::min<uint64_t>(n, max_seeds);
  s.cap_unique = std::min<uint64_t>(ucap, n);
  max_pos = std::max<uint64_t>(max_pos, max_seeds);
  s.blk_cap = (max_pos + 2047) / 2048 + 1;
  s.d_seeds = dalloc<uint32_t>(max_seeds);
  s.d_unique = dalloc<uint32_t>(s.cap_unique);
  s.d_inv1 = dalloc<int32_t>(std::max<uint64_t>(s.cap_inner, 1));
  s.d_first = dalloc<uint64_t>(n);
  s.d_gidx = dalloc<uint64_t>(n);
  A3G_CUDA(cudaMemset(s.d_first, 0, n * sizeof(uint64_t)));
  A3G_CUDA(cudaMemset(s.d_gidx, 0, n * sizeof(uint64_t)));
  s.d_blk = dalloc<uint4>(s.blk_cap);
  // hub-splitting arena: every frontier row could be a hub; the segment pool
  // covers sum(deg)/seg of a layer's hubs up to 64K segments (rows beyond
  // capacity fall back to the in-row warp replay, still exact).
  uint64_t max_rows = 0;
  for (uint32_t l = 0; l < L; ++l) max_rows = std::max<uint64_t>(max_rows, s.layer[l].cap_rows);
  HubArena& hb = s.hub;
  hb.hub_cap = static_cast<uint32_t>(std::max<uint64_t>(1, max_rows));
  // r01 sweeps (pipelined step time): C2 4096 -> 8192 0.443 -> 0.420 ms,
  // C5 2048 -> 4096 1.85 -> 1.71 ms, C3 2048 = 4096
  s.seg = g->n && g->m / g->n >= 128 ? 4 * kSegMin : 2 * kSegMin;
  if (const char* e = std::getenv("A3G_SEG")) {  // tuning sweeps: hub segment length (power of two >= 256)
    const uint32_t v = static_cast<uint32_t>(std::strtoul(e, nullptr, 10));
    if (v >= 256 && (v & (v - 1)) == 0) s.seg = v;
  }
  hb.seg_cap = static_cast<uint32_t>(std::min<uint64_t>(65536, std::max<uint64_t>(1, g->m / s.seg + max_rows)));
  hb.row = dalloc<uint32_t>(hb.hub_cap);
  hb.seg0 = dalloc<uint32_t>(hb.hub_cap);
  hb.nseg = dalloc<uint32_t>(hb.hub_cap);
  hb.big = dalloc<uint32_t>(hb.hub_cap);
  hb.small = dalloc<uint32_t>(hb.hub_cap);
  hb.seg_hub = dalloc<uint32_t>(hb.seg_cap);
  hb.rec_cnt = dalloc<uint32_t>(hb.seg_cap);
  hb.tau = dalloc<uint64_t>(hb.seg_cap);
  hb.tau_ok = dalloc<uint32_t>(hb.seg_cap);
  hb.rec_id = dalloc<uint32_t>(static_cast<size_t>(hb.seg_cap) * kRecCap);
  hb.rec_key = dalloc<uint64_t>(static_cast<size_t>(hb.seg_cap) * kRecCap);
  hb.slot_last = dalloc<uint32_t>(static_cast<size_t>(hb.seg_cap) * 32);
  hb.item_cap = hb.hub_cap + hb.seg_cap;
  hb.items = dalloc<uint4>(hb.item_cap);
  hb.sort_keys[0] = dalloc<uint32_t>(static_cast<uint64_t>(kLenClasses) * hb.item_cap);
  s.d_ctr = dalloc<BatchCounters>(1);
  A3G_CUDA(cudaMallocHost(&s.h_ctr, sizeof(BatchCounters)));
  A3G_CUDA(cudaMallocHost(&s.h_seeds, max_seeds * sizeof(uint32_t)));
  A3G_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  s.own_stream = true;
  A3G_CUDA(cudaEventCreateWithFlags(&s.ev_fork, cudaEventDisableTiming));
  A3G_CUDA(cudaEventCreateWithFlags(&s.ev_join, cudaEventDisableTiming));
}

void sampler_free(SamplerState& s) {
  for (uint32_t l = 0; l < s.L; ++l) {
    LayerArena& la = s.layer[l];
    dfree(la.front);
    dfree(la.front_idx);
    dfree(la.cnt);
    dfree(la.S);
    dfree(la.sidx);
    dfree(la.scratch);
  }
  dfree(s.d_seeds);
  dfree(s.d_unique);
  dfree(s.d_inv1);
  dfree(s.d_first);
  dfree(s.d_gidx);
  dfree(s.d_blk);
  dfree(s.hub.row);
  dfree(s.hub.seg0);
  dfree(s.hub.nseg);
  dfree(s.hub.big);
  dfree(s.hub.small);
  dfree(s.hub.seg_hub);
  dfree(s.hub.rec_cnt);
  dfree(s.hub.tau);
  dfree(s.hub.tau_ok);
  dfree(s.hub.rec_id);
  dfree(s.hub.rec_key);
  dfree(s.hub.slot_last);
  dfree(s.hub.items);
  dfree(s.hub.sort_keys[0]);
  dfree(s.d_ctr);
  if (s.h_ctr) cudaFreeHost(s.h_ctr);
  if (s.h_seeds) cudaFreeHost(s.h_seeds);
  if (s.own_stream && s.stream) cudaStreamDestroy(s.stream);
  if (s.ev_fork) cudaEventDestroy(s.ev_fork);
  if (s.ev_join) cudaEventDestroy(s.ev_join);
}

// sample_khop validation in the reference's order (sampler.cpp:91-94, :110,
// assign_weights :62 reached in layer 0 iff some unique seed has deg > 0).
void validate_sample(const SamplerState& s, const uint32_t* seeds, uint32_t n_seeds, bool host_seeds,
                     double gamma, int kind) {
  if (n_seeds == 0) raise(A3G_ERR_PARAMETER, "sample_khop: seeds must be non-empty");
  if (n_seeds > s.max_seeds) raise(A3G_ERR_PARAMETER, "sample_khop: more seeds than the arena holds");
  if (kind != A3G_SAMPLER_WEIGHTED && kind != A3G_SAMPLER_UNIFORM)
    raise(A3G_ERR_PARAMETER, "sample_khop: unknown sampler kind");
  if (!host_seeds) {
    // device-resident seeds: the range check runs on the device (k_check_seeds,
    // raised at the next sync); gamma is checked here without the degree
    // condition, which needs the seeds on the host
    if (kind == A3G_SAMPLER_WEIGHTED && s.L > 0 && gamma < 1.0)
      raise(A3G_ERR_PARAMETER, "assign_weights: gamma must be >= 1");
    return;
  }
  const a3g_graph* g = s.g;
  for (uint32_t i = 0; i < n_seeds; ++i)
    if (seeds[i] >= g->n) raise(A3G_ERR_PARAMETER, "sample_khop: seed out of range");
  // assign_weights is reached (and throws on gamma < 1) only if some unique
  // seed has neighbours; the degree lookups (random reads of the host CSR
  // offsets, ~16 ms per 164K seeds at papers scale) only when gamma < 1
  if (kind == A3G_SAMPLER_WEIGHTED && s.L > 0 && gamma < 1.0) {
    bool any_deg = false;
    for (uint32_t i = 0; i < n_seeds && !any_deg; ++i) any_deg = g->h_ro[seeds[i] + 1] > g->h_ro[seeds[i]];
    if (any_deg) raise(A3G_ERR_PARAMETER, "assign_weights: gamma must be >= 1");
  }
}

// prevalidated: device seeds that the host already checked (a3g_train_steps_v
// copies validated host seeds to the device first)
void sample_impl(SamplerState& s, const uint32_t* seeds, uint32_t n_seeds, bool on_device, double gamma,
                 int kind, uint64_t rng_seed, cudaStream_t st, bool prevalidated = false) {
  if (!prevalidated) validate_sample(s, seeds, n_seeds, !on_device, gamma, kind);
  s.check_seeds = on_device && !prevalidated;
  A3G_CUDA(cudaSetDevice(s.g->device));
  if (on_device) {
    if (seeds != s.d_seeds)
      A3G_CUDA(cudaMemcpyAsync(s.d_seeds, seeds, n_seeds * 4ull, cudaMemcpyDeviceToDevice, st));
  } else {
    // stage through pinned memory (the previous copy from it has completed
    // once the stream passed it: sync on reuse)
    A3G_CUDA(cudaStreamSynchronize(st));
    std::memcpy(s.h_seeds, seeds, n_seeds * 4ull);
    A3G_CUDA(cudaMemcpyAsync(s.d_seeds, s.h_seeds, n_seeds * 4ull, cudaMemcpyHostToDevice, st));
  }
  launch_sample(s, n_seeds, gamma, kind, rng_seed, st);
  s.last_n_seeds = n_seeds;
  s.has_batch = true;
}

void read_counters(SamplerState& s, cudaStream_t st) {
  A3G_CUDA(cudaMemcpyAsync(s.h_ctr, s.d_ctr, sizeof(BatchCounters), cudaMemcpyDeviceToHost, st));
  A3G_CUDA(cudaStreamSynchronize(st));
  if (s.h_ctr->bad_seeds) raise(A3G_ERR_PARAMETER, "sample_khop: seed out of range");
}

// init_model (trainer.cpp:12-28)
void init_weights(uint32_t F, uint32_t H, uint32_t C, uint64_t seed, std::vector<double>& w1,
                  std::vector<double>& w2) {
  const uint64_t key = hash2(seed, 0x6a10);
  uint64_t ctr = 0;
  w1.resize(static_cast<size_t>(F) * H);
  w2.resize(static_cast<size_t>(H) * C);
  double a = std::sqrt(6.0 / (static_cast<double>(F) + H));
  for (double& x : w1) x = (2.0 * unit_of(draw(key, ++ctr)) - 1.0) * a;
  a = std::sqrt(6.0 / (static_cast<double>(H) + C));
  for (double& x : w2) x = (2.0 * unit_of(draw(key, ++ctr)) - 1.0) * a;
}

}  // namespace

void a3g::set_error(const std::string& msg) { g_err = msg; }

namespace {
struct TlEvent {
  const char* name;
  cudaStream_t st;
  cudaEvent_t ev;
};
thread_local bool g_tl_on = false;
thread_local std::vector<TlEvent> g_tl;
}  // namespace

void a3g::tl_mark(const char* name, cudaStream_t st) {
  if (!g_tl_on) return;
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, st);
  g_tl.push_back(TlEvent{name, st, e});
}

// ====================================================================== ABI
extern "C" {

const char* a3g_last_error(void) { return g_err.c_str(); }
const char* a3g_version(void) { return "a3gnn-b200 0.1 (sm_100a)"; }

a3g_status a3g_host_graph_power_law(uint64_t n, uint32_t min_degree, double exponent, uint32_t feat_dim,
                                    uint64_t seed, int threads, a3g_host_graph** out) {
  return guard([&] { *out = power_law(n, min_degree, exponent, feat_dim, seed, threads); });
}
a3g_status a3g_host_graph_load(const char* path, a3g_host_graph** out) {
  return guard([&] { *out = load_host(path); });
}
a3g_status a3g_host_graph_save(const a3g_host_graph* g, const char* path) {
  return guard([&] { save_host(g, path); });
}
a3g_status a3g_host_graph_from_edges(uint64_t n, const uint32_t* src, const uint32_t* dst, uint64_t m,
                                     uint32_t f, a3g_host_graph** out) {
  return guard([&] { *out = from_edges(n, src, dst, m, f); });
}
void a3g_host_graph_free(a3g_host_graph* g) { free_host(g); }

uint64_t a3g_sampling_seed(uint64_t base, uint32_t epoch, uint32_t step, uint32_t worker) {
  return hash3(base, hash2(epoch, step), worker);  // trainer.cpp:345-348
}

void a3g_plan_epoch_order(const uint32_t* train_nodes, uint64_t n, uint32_t epoch, uint64_t seed,
                          uint32_t* order) {
  std::memcpy(order, train_nodes, n * 4);
  const uint64_t key = hash2(seed, hash2(0x5f1e, epoch));  // trainer.cpp:335
  uint64_t ctr = 0;
  for (uint64_t i = n; i > 1; --i) {  // rng.hpp:69-74
    const uint64_t j = static_cast<uint64_t>(
        (static_cast<unsigned __int128>(draw(key, ++ctr)) * static_cast<uint32_t>(i)) >> 64);
    std::swap(order[i - 1], order[j]);
  }
}

// ------------------------------------------------------------------ graph
a3g_status a3g_graph_create(int device, uint64_t n, uint64_t m, uint32_t F, const uint64_t* ro,
                            const uint32_t* col, const float* features, int feat_dtype,
                            const uint32_t* labels, a3g_graph** out) {
  return guard([&] {
    if (F < 1) raise(A3G_ERR_PARAMETER, "graph: feat_dim must be >= 1");
    if (n >= (1ull << 32) - 1) raise(A3G_ERR_PARAMETER, "graph: num_nodes exceeds NodeId range");
    if (ro[0] != 0 || ro[n] != m) raise(A3G_ERR_PARAMETER, "graph: row_offsets invariant violated");
    A3G_CUDA(cudaSetDevice(device));
    auto* g = new a3g_graph;
    g->device = device;
    g->n = n;
    g->m = m;
    g->F = F;
    g->pitch = (F + 7) / 8 * 8;
    g->feat_dtype = feat_dtype;
    g->h_ro.assign(ro, ro + n + 1);
    g->d_ro = dalloc<uint64_t>(n + 1);
    g->d_col = dalloc<uint32_t>(m + 8);  // +8: 16-byte rounded TMA pieces may read past the end
    A3G_CUDA(cudaMemset(g->d_col + m, 0, 8 * 4));
    A3G_CUDA(cudaMemcpy(g->d_ro, ro, (n + 1) * 8, cudaMemcpyHostToDevice));
    if (m) A3G_CUDA(cudaMemcpy(g->d_col, col, m * 4, cudaMemcpyHostToDevice));
    g->d_labels = dalloc<uint32_t>(n);
    if (labels) {
      g->h_labels.assign(labels, labels + n);
      A3G_CUDA(cudaMemcpy(g->d_labels, labels, n * 4, cudaMemcpyHostToDevice));
    } else {
      A3G_CUDA(cudaMemset(g->d_labels, 0, n * 4));
    }
    const size_t esz = feat_dtype == A3G_FEAT_BF16 ? 2 : 4;
    const size_t row_bytes = static_cast<size_t>(g->pitch) * esz;
    g->view.loc = nullptr;
    g->view.row_bytes = static_cast<uint32_t>(row_bytes);
    if (features) {
      void* d = nullptr;
      A3G_CUDA(cudaMalloc(&d, std::max<size_t>(1, n * row_bytes)));
      g->d_feat = d;
      g->view.base[0] = static_cast<const uint8_t*>(d);
      g->has_features = true;
      // pitched upload in slabs through a host staging buffer
      const uint64_t slab = std::max<uint64_t>(1, (64ull << 20) / row_bytes);
      std::vector<uint8_t> stage(slab * row_bytes);
      for (uint64_t v0 = 0; v0 < n; v0 += slab) {
        const uint64_t cnt = std::min<uint64_t>(slab, n - v0);
        std::memset(stage.data(), 0, cnt * row_bytes);
        for (uint64_t i = 0; i < cnt; ++i) {
          const float* src = features + (v0 + i) * F;
          if (esz == 4) {
            std::memcpy(stage.data() + i * row_bytes, src, F * 4ull);
          } else {  // round-to-nearest-even bf16
            uint16_t* dst = reinterpret_cast<uint16_t*>(stage.data() + i * row_bytes);
            for (uint32_t c = 0; c < F; ++c) {
              uint32_t x;
              std::memcpy(&x, src + c, 4);
              const uint32_t lsb = (x >> 16) & 1u;
              dst[c] = static_cast<uint16_t>((x + 0x7fffu + lsb) >> 16);
            }
          }
        }
        A3G_CUDA(cudaMemcpy(static_cast<uint8_t*>(d) + v0 * row_bytes, stage.data(), cnt * row_bytes,
                            cudaMemcpyHostToDevice));
      }
    }
    *out = g;
  });
}

void a3g_graph_destroy(a3g_graph* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  if (g->store) a3g_store_destroy(g->store);
  dfree(g->d_ro);
  dfree(g->d_col);
  dfree(g->d_labels);
  if (g->d_feat) cudaFree(g->d_feat);
  delete g;
}

// ------------------------------------------------------------------ cache
static a3g_cache* cache_from(a3g_graph* g, std::vector<int32_t>&& dm, uint32_t num_devices) {
  auto* c = new a3g_cache;
  c->g = g;
  c->num_devices = num_devices;
  c->device_map = std::move(dm);
  uint64_t cached = 0;
  std::vector<uint32_t> bits((g->n + 31) / 32 + 1, 0);
  for (uint64_t v = 0; v < g->n; ++v)
    if (c->device_map[v] != -1) {
      ++cached;
      bits[v >> 5] |= 1u << (v & 31);
    }
  c->total_cached = cached;
  c->all_cached = cached == g->n;
  c->none_cached = cached == 0;
  A3G_CUDA(cudaSetDevice(g->device));
  c->d_bits = dalloc<uint32_t>(bits.size());
  A3G_CUDA(cudaMemcpy(c->d_bits, bits.data(), bits.size() * 4, cudaMemcpyHostToDevice));
  if (num_devices > 1) {
    c->d_map = dalloc<int32_t>(std::max<uint64_t>(g->n, 1));
    A3G_CUDA(cudaMemcpy(c->d_map, c->device_map.data(), g->n * 4, cudaMemcpyHostToDevice));
  }
  if (!c->all_cached && !c->none_cached && g->m) {
    const uint64_t words = (g->m + 31) / 32 + 1;
    c->d_ebits = dalloc<uint32_t>(words);
    A3G_CUDA(cudaMemset(c->d_ebits, 0, words * 4));
    int sms = 0;
    A3G_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
    build_edge_bits(g->d_col, g->m, c->d_bits, c->d_ebits, sms, 0);
    A3G_CUDA(cudaDeviceSynchronize());
  }
  return c;
}

a3g_status a3g_cache_build(a3g_graph* g, uint64_t volume, uint32_t num_devices, int32_t* dm_out,
                           a3g_cache** out) {
  return guard([&] {
    if (num_devices < 1) raise(A3G_ERR_PARAMETER, "build_static_cache: num_devices >= 1");
    const uint64_t n = g->n;
    std::vector<int32_t> dm(n, -1);
    std::vector<uint32_t> order;
    const uint64_t cost = static_cast<uint64_t>(g->F) * 4;  // cache.cpp:20
    if (volume >= cost) {
      // hotness order (cache.cpp:24-29): degree desc, id asc
      order.resize(n);
      std::iota(order.begin(), order.end(), 0u);
      const uint64_t per_dev = volume / cost;
      const uint64_t want = std::min<uint64_t>(n, per_dev * num_devices);
      auto cmp = [&](uint32_t a, uint32_t b) {
        const uint64_t da = g->h_ro[a + 1] - g->h_ro[a], db = g->h_ro[b + 1] - g->h_ro[b];
        return da != db ? da > db : a < b;
      };
      if (want < n)
        std::partial_sort(order.begin(), order.begin() + want, order.end(), cmp);
      else
        std::sort(order.begin(), order.end(), cmp);
      // round-robin with full-device skipping (cache.cpp:31-44); every device
      // holds per_dev nodes, so plain round-robin over the first `want`.
      for (uint64_t i = 0; i < want; ++i) dm[order[i]] = static_cast<int32_t>(i % num_devices);
      order.resize(want);
    } else {
      order.clear();
    }
    if (dm_out) std::memcpy(dm_out, dm.data(), n * 4);
    *out = cache_from(g, std::move(dm), num_devices);
    (*out)->hot_order = std::move(order);
  });
}

a3g_status a3g_cache_from_map(a3g_graph* g, const int32_t* dm, uint32_t num_devices, a3g_cache** out) {
  return guard([&] {
    std::vector<int32_t> v(dm ? dm : nullptr, dm ? dm + g->n : nullptr);
    if (!dm) v.assign(g->n, -1);
    *out = cache_from(g, std::move(v), std::max<uint32_t>(1, num_devices));
  });
}

uint64_t a3g_cache_total_cached(const a3g_cache* c) { return c->total_cached; }

a3g_status a3g_cache_hot_order(const a3g_cache* c, uint32_t* out) {
  return guard([&] {
    if (c->hot_order.size() != c->total_cached)
      raise(A3G_ERR_PARAMETER, "cache_hot_order: cache was not built by a3g_cache_build");
    std::memcpy(out, c->hot_order.data(), c->hot_order.size() * 4);
  });
}

a3g_status a3g_cache_lookup(a3g_cache* c, const uint32_t* ids, uint64_t n, int32_t* device_out, uint64_t* hits,
                            uint64_t* misses, uint64_t* per_device_hits) {
  return guard([&] {
    a3g_graph* g = c->g;
    for (uint64_t i = 0; i < n; ++i)
      if (ids[i] >= g->n) raise(A3G_ERR_PARAMETER, "lookup: node out of range");
    if (c->num_devices > kMaxCacheDevices) raise(A3G_ERR_PARAMETER, "lookup: more than 64 cache devices");
    A3G_CUDA(cudaSetDevice(g->device));
    const uint32_t nd = c->num_devices;
    std::vector<unsigned long long> cnt(2 + nd, 0);
    if (n) {
      uint32_t* d_ids = dalloc<uint32_t>(n);
      int32_t* d_dev = device_out ? dalloc<int32_t>(n) : nullptr;
      unsigned long long* d_cnt = dalloc<unsigned long long>(2 + nd);
      A3G_CUDA(cudaMemcpy(d_ids, ids, n * 4, cudaMemcpyHostToDevice));
      A3G_CUDA(cudaMemset(d_cnt, 0, (2 + nd) * 8));
      launch_cache_lookup(c, d_ids, n, d_dev, d_cnt, sm_count_of(g->device), nullptr);
      A3G_CUDA(cudaMemcpy(cnt.data(), d_cnt, (2 + nd) * 8, cudaMemcpyDeviceToHost));
      if (device_out) A3G_CUDA(cudaMemcpy(device_out, d_dev, n * 4, cudaMemcpyDeviceToHost));
      dfree(d_ids);
      dfree(d_dev);
      dfree(d_cnt);
    }
    if (hits) *hits = cnt[0];
    if (misses) *misses = cnt[1];
    if (per_device_hits)
      for (uint32_t d = 0; d < nd; ++d) per_device_hits[d] = cnt[2 + d];
  });
}

void a3g_cache_destroy(a3g_cache* c) {
  if (!c) return;
  dfree(c->d_map);
  dfree(c->d_bits);
  dfree(c->d_ebits);
  delete c;
}

// ---------------------------------------------------------------- sampler
a3g_status a3g_sampler_create(a3g_graph* g, a3g_cache* c, uint32_t max_seeds, const uint32_t* fanouts,
                              uint32_t L, a3g_sampler** out) {
  return guard([&] {
    auto* s = new a3g_sampler;
    try {
      sampler_alloc(s->st, g, c, max_seeds, fanouts, L);
    } catch (...) {
      sampler_free(s->st);
      delete s;
      throw;
    }
    *out = s;
  });
}

void a3g_sampler_destroy(a3g_sampler* s) {
  if (!s) return;
  cudaSetDevice(s->st.device);
  sampler_free(s->st);
  delete s;
}

a3g_status a3g_sample_khop(a3g_sampler* s, const uint32_t* seeds, uint32_t n_seeds, int on_device,
                           double gamma, int kind, uint64_t rng_seed, void* stream) {
  return guard([&] {
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : s->st.stream;
    sample_impl(s->st, seeds, n_seeds, on_device != 0, gamma, kind, rng_seed, st);
  });
}

a3g_status a3g_batch_sizes(a3g_sampler* s, uint64_t* nu, uint64_t* nsu, uint64_t* dups, uint64_t* le) {
  return guard([&] {
    SamplerState& st = s->st;
    if (!st.has_batch) raise(A3G_ERR_PARAMETER, "batch_sizes: no batch sampled");
    read_counters(st, st.stream);
    const BatchCounters& c = *st.h_ctr;
    const uint64_t U = c.ucount[st.L];
    uint64_t E = 0;
    for (uint32_t l = 0; l < st.L; ++l) {
      E += c.edges[l];
      if (le) le[l] = c.edges[l];
    }
    if (nu) *nu = U;
    if (nsu) *nsu = c.ucount[0];
    if (dups) *dups = c.n_seeds + E - U;  // #intern calls - |unique| (sampler.cpp:76-84)
  });
}

a3g_status a3g_batch_copy(a3g_sampler* s, uint32_t* unique, uint32_t* const* ldst, uint32_t* const* lsrc) {
  return guard([&] {
    SamplerState& st = s->st;
    if (!st.has_batch) raise(A3G_ERR_PARAMETER, "batch_copy: no batch sampled");
    read_counters(st, st.stream);
    const BatchCounters c = *st.h_ctr;
    const uint64_t U = c.ucount[st.L];
    if (unique && U) A3G_CUDA(cudaMemcpy(unique, st.d_unique, U * 4, cudaMemcpyDeviceToHost));
    for (uint32_t l = 0; l < st.L; ++l) {
      if (!(ldst && ldst[l]) && !(lsrc && lsrc[l])) continue;
      const LayerArena& la = st.layer[l];
      const uint64_t rows = c.nfront[l];
      std::vector<uint32_t> cnt(rows), fidx(rows), sidx(rows * la.f);
      if (rows) {
        A3G_CUDA(cudaMemcpy(cnt.data(), la.cnt, rows * 4, cudaMemcpyDeviceToHost));
        A3G_CUDA(cudaMemcpy(fidx.data(), la.front_idx, rows * 4, cudaMemcpyDeviceToHost));
        A3G_CUDA(cudaMemcpy(sidx.data(), la.sidx, rows * la.f * 4, cudaMemcpyDeviceToHost));
      }
      uint64_t e = 0;
      for (uint64_t k = 0; k < rows; ++k)
        for (uint32_t t = 0; t < cnt[k]; ++t, ++e) {
          if (ldst && ldst[l]) ldst[l][e] = fidx[k];
          if (lsrc && lsrc[l]) lsrc[l][e] = sidx[k * la.f + t];
        }
    }
  });
}

a3g_status a3g_retrieve_features(a3g_sampler* s, float* out, int out_on_device, uint64_t* hits,
                                 uint64_t* misses, uint64_t* batch_bytes, void* stream) {
  return guard([&] {
    SamplerState& st = s->st;
    if (!st.has_batch) raise(A3G_ERR_PARAMETER, "retrieve_features: no batch sampled");
    if (!st.g->has_features) raise(A3G_ERR_PARAMETER, "retrieve_features: graph has no features");
    cudaStream_t cs = stream ? static_cast<cudaStream_t>(stream) : st.stream;
    read_counters(st, cs);
    const uint64_t U = st.h_ctr->ucount[st.L];
    uint64_t E = 0;
    for (uint32_t l = 0; l < st.L; ++l) E += st.h_ctr->edges[l];
    const uint64_t F = st.g->F;
    float* dout = out;
    if (!out_on_device) dout = dalloc<float>(U * F);
    launch_gather_unique(st, dout, cs);
    read_counters(st, cs);
    if (!out_on_device) {
      if (U) A3G_CUDA(cudaMemcpy(out, dout, U * F * 4, cudaMemcpyDeviceToHost));
      cudaFree(dout);
    }
    if (hits) *hits = st.h_ctr->hits;
    if (misses) *misses = st.h_ctr->misses;
    if (batch_bytes) *batch_bytes = U * F * 4 + E * 2 * 4;  // cache.cpp:84
    // accounting counters are per call (CacheAccounting is the caller's)
    A3G_CUDA(cudaMemsetAsync(&st.d_ctr->hits, 0, 8, cs));
  });
}

a3g_status a3g_gather_rows(a3g_graph* g, a3g_cache* c, const uint32_t* ids, uint64_t n, float* out,
                           uint64_t* hits, uint64_t* misses) {
  return guard([&] {
    if (!g->has_features) raise(A3G_ERR_PARAMETER, "retrieve_features: graph has no features");
    for (uint64_t i = 0; i < n; ++i)
      if (ids[i] >= g->n) raise(A3G_ERR_PARAMETER, "retrieve_features: node out of range");
    if (n >= (1ull << 32)) raise(A3G_ERR_PARAMETER, "retrieve_features: too many ids");
    A3G_CUDA(cudaSetDevice(g->device));
    uint64_t h = 0, m = 0;
    if (n) {
      SamplerState tmp{};
      tmp.g = g;
      tmp.c = c;
      tmp.L = 0;
      tmp.sm_count = sm_count_of(g->device);
      tmp.d_unique = dalloc<uint32_t>(n);
      tmp.d_ctr = dalloc<BatchCounters>(1);
      float* dout = dalloc<float>(n * g->F);
      A3G_CUDA(cudaMemcpy(tmp.d_unique, ids, n * 4, cudaMemcpyHostToDevice));
      BatchCounters hc{};
      hc.ucount[0] = static_cast<uint32_t>(n);
      A3G_CUDA(cudaMemcpy(tmp.d_ctr, &hc, sizeof hc, cudaMemcpyHostToDevice));
      launch_gather_unique(tmp, dout, nullptr);
      A3G_CUDA(cudaMemcpy(out, dout, n * g->F * 4, cudaMemcpyDeviceToHost));
      A3G_CUDA(cudaMemcpy(&hc, tmp.d_ctr, sizeof hc, cudaMemcpyDeviceToHost));
      h = hc.hits;
      m = hc.misses;
      cudaFree(dout);
      dfree(tmp.d_unique);
      dfree(tmp.d_ctr);
    }
    if (hits) *hits = h;
    if (misses) *misses = m;
  });
}

a3g_status a3g_weighted_reservoir(const uint32_t* nbrs, const double* weights, uint64_t n, uint32_t m,
                                  uint64_t key, uint64_t ctr0, uint32_t* out, uint64_t* count) {
  return guard([&] {
    if (m < 1) raise(A3G_ERR_PARAMETER, "weighted_reservoir_sample: m must be >= 1");
    *count = 0;
    if (n == 0) return;
    for (uint64_t j = 0; j < n; ++j)
      if (!(weights[j] > 0.0)) raise(A3G_ERR_PARAMETER, "weighted_reservoir_sample: weights must be positive");
    uint32_t* d_nb = dalloc<uint32_t>(n);
    double* d_w = dalloc<double>(n);
    uint32_t* d_out = dalloc<uint32_t>(std::max<uint64_t>(m, 1));
    double* d_keys = dalloc<double>(std::max<uint64_t>(m, 1));
    A3G_CUDA(cudaMemcpy(d_nb, nbrs, n * 4, cudaMemcpyHostToDevice));
    A3G_CUDA(cudaMemcpy(d_w, weights, n * 8, cudaMemcpyHostToDevice));
    launch_reservoir_list(d_nb, d_w, n, m, key, ctr0, A3G_SAMPLER_WEIGHTED, d_out, d_keys, nullptr);
    const uint64_t cnt = std::min<uint64_t>(n, m);
    A3G_CUDA(cudaMemcpy(out, d_out, cnt * 4, cudaMemcpyDeviceToHost));
    cudaFree(d_nb);
    cudaFree(d_w);
    cudaFree(d_out);
    cudaFree(d_keys);
    *count = cnt;
  });
}

a3g_status a3g_uniform_reservoir(const uint32_t* nbrs, uint64_t n, uint32_t m, uint64_t key, uint64_t ctr0,
                                 uint32_t* out, uint64_t* count) {
  return guard([&] {
    if (m < 1) raise(A3G_ERR_PARAMETER, "uniform_reservoir_sample: m must be >= 1");
    *count = 0;
    if (n == 0) return;
    uint32_t* d_nb = dalloc<uint32_t>(n);
    uint32_t* d_out = dalloc<uint32_t>(std::max<uint64_t>(m, 1));
    A3G_CUDA(cudaMemcpy(d_nb, nbrs, n * 4, cudaMemcpyHostToDevice));
    launch_reservoir_list(d_nb, nullptr, n, m, key, ctr0, A3G_SAMPLER_UNIFORM, d_out, nullptr, nullptr);
    const uint64_t cnt = std::min<uint64_t>(n, m);
    A3G_CUDA(cudaMemcpy(out, d_out, cnt * 4, cudaMemcpyDeviceToHost));
    cudaFree(d_nb);
    cudaFree(d_out);
    *count = cnt;
  });
}

// ---------------------------------------------------------------- trainer
a3g_status a3g_init_model(uint32_t F, uint32_t H, uint32_t C, uint64_t seed, double* w1, double* w2) {
  return guard([&] {
    if (F < 1 || H < 1 || C < 1) raise(A3G_ERR_PARAMETER, "init_model: dims must be >= 1");
    std::vector<double> a, b;
    init_weights(F, H, C, seed, a, b);
    std::copy(a.begin(), a.end(), w1);
    std::copy(b.begin(), b.end(), w2);
  });
}

a3g_status a3g_trainer_create(a3g_graph* g, a3g_cache* c, uint32_t max_seeds, const uint32_t* fanouts,
                              uint32_t L, uint32_t H, uint32_t C, double lr, uint64_t model_seed,
                              a3g_trainer** out) {
  return guard([&] {
    if (g->F < 1 || H < 1 || C < 1) raise(A3G_ERR_PARAMETER, "init_model: dims must be >= 1");
    // H <= 16: h1 fused into the gather; 16 < H <= 32: dW1 on the CUDA cores;
    // up to 256: both products on tcgen05 (N = H, TMEM accumulators)
    if (H > 256 || C > 32) raise(A3G_ERR_PARAMETER, "trainer: hidden_dim must be <= 256 and num_classes <= 32");
    if (!g->has_features) raise(A3G_ERR_PARAMETER, "trainer: graph has no features");
    auto* tr = new a3g_trainer;
    TrainerState& t = tr->st;
    try {
      A3G_CUDA(cudaSetDevice(g->device));
      t.g = g;
      t.c = c;
      t.F = g->F;
      t.H = H;
      t.C = C;
      t.pitch = g->pitch;
      t.L = L;
      t.lr = lr;
      t.max_seeds = max_seeds;
      t.pipe_streams = max_seeds <= TrainerState::kSmallBatch ? TrainerState::kDefaultStreamsSmall
                                                               : TrainerState::kDefaultStreams;
      t.sm_count = sm_count_of(g->device);
      t.fanouts.assign(fanouts, fanouts + L);
      t.tc_gemms = std::getenv("A3G_TC_GEMMS") != nullptr;
      t.smp[0] = new a3g_sampler;
      sampler_alloc(t.smp[0]->st, g, c, max_seeds, fanouts, L);
      t.cap_inner = std::max<uint64_t>(1, t.smp[0]->st.cap_inner);
      if (tc_h1_smem(t.F, H) > 227 * 1024)
        raise(A3G_ERR_PARAMETER, "trainer: feat_dim too large for the tcgen05 dense update (F <= 1280)");
      t.d_w1 = dalloc<float>(static_cast<size_t>(t.F) * H);
      t.d_w2 = dalloc<float>(static_cast<size_t>(H) * C);
      t.d_gw = dalloc<float>(static_cast<size_t>(t.F) * H + H * C + 2);
      t.d_agg_inner = dalloc<float>(t.cap_inner * g->pitch);
      t.d_dh1_fx = dalloc<unsigned long long>(t.cap_inner * H);
      A3G_CUDA(cudaMemset(t.d_dh1_fx, 0, t.cap_inner * H * 8));
      t.d_h1 = dalloc<float>(t.cap_inner * H);
      t.d_dh1 = dalloc<float>(t.cap_inner * H);
      t.d_agg_outer = dalloc<float>(static_cast<size_t>(max_seeds) * H);
      t.d_logits = dalloc<float>(static_cast<size_t>(max_seeds) * C);
      t.d_dlogits = dalloc<float>(static_cast<size_t>(max_seeds) * C);
      t.d_loss_s = dalloc<float>(max_seeds);
      t.d_dagg = dalloc<float>(static_cast<size_t>(max_seeds) * H);
      t.d_amax = dalloc<uint32_t>(1);
      t.nparts = static_cast<uint32_t>(t.sm_count);
      t.tc_splits = std::max<uint32_t>(1, static_cast<uint32_t>(t.sm_count) / ((t.F + 127) / 128));
      t.h1_split_cap = std::min<uint32_t>(8, (t.F + 63) / 64);
      t.d_hpart = dalloc<float>(static_cast<size_t>(t.h1_split_cap) * t.cap_inner * H);
      t.dw1_splits = static_cast<uint32_t>((t.cap_inner + 127) / 128);  // kDw1Rows
      t.d_part = dalloc<float>(static_cast<size_t>(std::max({t.nparts, t.tc_splits, t.dw1_splits})) * t.F * H);
      t.d_agg_bytes = dalloc<unsigned long long>(2);  // [k_agg1 bytes | sticky bad-seed flag]
      A3G_CUDA(cudaMemset(t.d_agg_bytes, 0, 16));
      t.losses_cap = 1;
      t.d_losses = dalloc<double>(1);
      A3G_CUDA(cudaMallocHost(&t.h_losses, 8));
      // the compute stream runs at the highest priority: it is the pipeline's
      // serial chain; the sampling streams fill the SMs it leaves idle
      int prio_lo = 0, prio_hi = 0;
      A3G_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
      static const bool no_prio = std::getenv("A3G_NO_PRIORITY") != nullptr;
      A3G_CUDA(cudaStreamCreateWithPriority(&t.s_comp, cudaStreamNonBlocking, no_prio ? prio_lo : prio_hi));
      A3G_CUDA(cudaStreamCreateWithFlags(&t.s_samp, cudaStreamNonBlocking));
      t.s_sx[0] = t.s_samp;
      for (int i = 1; i < TrainerState::kSampStreams; ++i)
        A3G_CUDA(cudaStreamCreateWithFlags(&t.s_sx[i], cudaStreamNonBlocking));
      A3G_CUDA(cudaEventCreateWithFlags(&t.ev_seeds, cudaEventDisableTiming));
      for (int i = 0; i < TrainerState::kArenas; ++i) {
        A3G_CUDA(cudaEventCreateWithFlags(&t.ev_sampled[i], cudaEventDisableTiming));
        A3G_CUDA(cudaEventCreateWithFlags(&t.ev_consumed[i], cudaEventDisableTiming));
      }
      A3G_CUDA(cudaEventCreate(&t.ev_t0));
      A3G_CUDA(cudaEventCreate(&t.ev_t1));
      std::vector<double> w1, w2;
      init_weights(t.F, H, C, model_seed, w1, w2);
      std::vector<float> f1(w1.begin(), w1.end()), f2(w2.begin(), w2.end());
      A3G_CUDA(cudaMemcpy(t.d_w1, f1.data(), f1.size() * 4, cudaMemcpyHostToDevice));
      A3G_CUDA(cudaMemcpy(t.d_w2, f2.data(), f2.size() * 4, cudaMemcpyHostToDevice));
    } catch (...) {
      a3g_trainer_destroy(tr);
      throw;
    }
    *out = tr;
  });
}

void a3g_trainer_destroy(a3g_trainer* tr) {
  if (!tr) return;
  TrainerState& t = tr->st;
  if (t.g) cudaSetDevice(t.g->device);
  if (t.s_comp) cudaStreamSynchronize(t.s_comp);
  if (t.s_samp) cudaStreamSynchronize(t.s_samp);
  for (int i = 1; i < TrainerState::kSampStreams; ++i)
    if (t.s_sx[i]) cudaStreamSynchronize(t.s_sx[i]);
  for (int i = 0; i < TrainerState::kArenas; ++i)
    if (t.smp[i]) {
      sampler_free(t.smp[i]->st);
      delete t.smp[i];
    }
  dfree(t.d_w1);
  dfree(t.d_w2);
  dfree(t.d_gw);
  dfree(t.d_agg_inner);
  dfree(t.d_h1);
  dfree(t.d_dh1);
  dfree(t.d_agg_outer);
  dfree(t.d_logits);
  dfree(t.d_dlogits);
  dfree(t.d_loss_s);
  dfree(t.d_dagg);
  dfree(t.d_dh1_fx);
  dfree(t.d_amax);
  dfree(t.d_part);
  dfree(t.d_hpart);
  dfree(t.d_gather);
  dfree(t.d_tier_seen);
  dfree(t.d_tier_rows);
  dfree(t.d_agg_bytes);
  dfree(t.d_losses);
  dfree(t.d_stats);
  dfree(t.d_seed_buf);
  if (t.h_seed_stage) cudaFreeHost(t.h_seed_stage);
  if (t.h_losses) cudaFreeHost(t.h_losses);
  for (cudaEvent_t e : t.ev_pool) cudaEventDestroy(e);
  for (int i = 0; i < TrainerState::kArenas; ++i) {
    if (t.ev_sampled[i]) cudaEventDestroy(t.ev_sampled[i]);
    if (t.ev_consumed[i]) cudaEventDestroy(t.ev_consumed[i]);
  }
  if (t.ev_seeds) cudaEventDestroy(t.ev_seeds);
  for (int i = 1; i < TrainerState::kSampStreams; ++i)
    if (t.s_sx[i]) cudaStreamDestroy(t.s_sx[i]);
  if (t.ev_t0) cudaEventDestroy(t.ev_t0);
  if (t.ev_t1) cudaEventDestroy(t.ev_t1);
  if (t.s_comp) cudaStreamDestroy(t.s_comp);
  if (t.s_samp) cudaStreamDestroy(t.s_samp);
  delete tr;
}

a3g_status a3g_trainer_set_weights(a3g_trainer* tr, const double* w1, const double* w2) {
  return guard([&] {
    TrainerState& t = tr->st;
    A3G_CUDA(cudaSetDevice(t.g->device));
    std::vector<float> f1(w1, w1 + static_cast<size_t>(t.F) * t.H), f2(w2, w2 + static_cast<size_t>(t.H) * t.C);
    A3G_CUDA(cudaStreamSynchronize(t.s_comp));
    A3G_CUDA(cudaMemcpy(t.d_w1, f1.data(), f1.size() * 4, cudaMemcpyHostToDevice));
    A3G_CUDA(cudaMemcpy(t.d_w2, f2.data(), f2.size() * 4, cudaMemcpyHostToDevice));
  });
}

a3g_status a3g_trainer_get_weights(a3g_trainer* tr, double* w1, double* w2) {
  return guard([&] {
    TrainerState& t = tr->st;
    A3G_CUDA(cudaSetDevice(t.g->device));
    A3G_CUDA(cudaStreamSynchronize(t.s_comp));
    std::vector<float> f1(static_cast<size_t>(t.F) * t.H), f2(static_cast<size_t>(t.H) * t.C);
    A3G_CUDA(cudaMemcpy(f1.data(), t.d_w1, f1.size() * 4, cudaMemcpyDeviceToHost));
    A3G_CUDA(cudaMemcpy(f2.data(), t.d_w2, f2.size() * 4, cudaMemcpyDeviceToHost));
    if (w1) std::copy(f1.begin(), f1.end(), w1);
    if (w2) std::copy(f2.begin(), f2.end(), w2);
  });
}

a3g_status a3g_trainer_set_pipeline(a3g_trainer* tr, int sampling_streams) {
  return guard([&] {
    if (sampling_streams < 0 || sampling_streams > TrainerState::kSampStreams)
      raise(A3G_ERR_PARAMETER, "set_pipeline: sampling streams must be in [0, 8]");
    tr->st.pipe_streams = sampling_streams;
  });
}

a3g_status a3g_trainer_set_comm(a3g_trainer* tr, a3g_comm* comm) {
  return guard([&] { tr->st.comm = comm; });
}

a3g_status a3g_train_step(a3g_trainer* tr, const uint32_t* seeds, uint32_t n_seeds, int on_device,
                          double gamma, int kind, uint64_t rng_seed, double lr, double* loss_out) {
  return guard([&] {
    TrainerState& t = tr->st;
    A3G_CUDA(cudaSetDevice(t.g->device));
    a3g_sampler* smp = t.smp[0];
    sample_impl(smp->st, seeds, n_seeds, on_device != 0, gamma, kind, rng_seed, t.s_comp);
    launch_train_compute(t, smp, lr < 0 ? t.lr : lr, t.d_losses, nullptr, t.s_comp, false);
    if (on_device) read_counters(smp->st, t.s_comp);  // raises on out-of-range device seeds
    if (loss_out) {
      A3G_CUDA(cudaMemcpyAsync(t.h_losses, t.d_losses, 8, cudaMemcpyDeviceToHost, t.s_comp));
      A3G_CUDA(cudaStreamSynchronize(t.s_comp));
      *loss_out = t.h_losses[0];
    }
  });
}

a3g_status a3g_train_steps(a3g_trainer* tr, const uint32_t* seeds, uint32_t B, uint32_t K,
                           const uint64_t* rng_seeds, double gamma, int kind, int on_device, double* losses_out) {
  std::vector<uint64_t> off(static_cast<size_t>(K) + 1);
  for (uint32_t i = 0; i <= K; ++i) off[i] = static_cast<uint64_t>(i) * B;
  return a3g_train_steps_v(tr, seeds, off.data(), K, rng_seeds, gamma, kind, on_device, losses_out);
}

a3g_status a3g_train_steps_v(a3g_trainer* tr, const uint32_t* seeds, const uint64_t* off, uint32_t K,
                             const uint64_t* rng_seeds, double gamma, int kind, int on_device, double* losses_out) {
  return guard([&] {
    TrainerState& t = tr->st;
    A3G_CUDA(cudaSetDevice(t.g->device));
    t.last_steps = 0;
    t.last_seeds_on_device = on_device != 0;
    if (K == 0) return;
    if (off[0] != 0) raise(A3G_ERR_PARAMETER, "train_steps: offsets[0] must be 0");
    for (uint32_t i = 0; i < K; ++i) {
      if (off[i + 1] < off[i]) raise(A3G_ERR_PARAMETER, "train_steps: offsets must be non-decreasing");
      const uint64_t b = off[i + 1] - off[i];
      if (b > t.max_seeds) raise(A3G_ERR_PARAMETER, "train_steps: batch larger than the arena");
      validate_sample(t.smp[0]->st, on_device ? nullptr : seeds + off[i], static_cast<uint32_t>(b), !on_device,
                      gamma, kind);
    }
    const uint64_t total = off[K];
    if (K > t.losses_cap) {
      dfree(t.d_losses);
      cudaFreeHost(t.h_losses);
      t.d_losses = dalloc<double>(K);
      A3G_CUDA(cudaMallocHost(&t.h_losses, K * 8ull));
      t.losses_cap = K;
    }
    if (K > t.stats_cap) {
      dfree(t.d_stats);
      t.d_stats = dalloc<unsigned long long>(static_cast<size_t>(K) * A3G_STEP_STATS);
      t.stats_cap = K;
    }
    t.ev_agg.clear();  // the events return to the pool
    t.ev_h1.clear();
    t.ev_dw1.clear();
    t.ev_used = 0;
    A3G_CUDA(cudaMemsetAsync(t.d_agg_bytes, 0, 16, t.s_comp));
    if (t.d_tier_rows) A3G_CUDA(cudaMemsetAsync(t.d_tier_rows, 0, kMaxTiers * 8, t.s_comp));
    A3G_CUDA(cudaMemsetAsync(t.d_stats, 0, static_cast<size_t>(K) * A3G_STEP_STATS * 8, t.s_comp));
    A3G_CUDA(cudaEventRecord(t.ev_t0, t.s_comp));
    A3G_CUDA(cudaStreamWaitEvent(t.s_samp, t.ev_t0, 0));
    const uint32_t* dseeds = seeds;
    if (!on_device) {  // H2D of every step's seeds (inside the timed region)
      if (total > t.seed_buf_cap) {  // grow geometrically: reallocation (a device sync) stays rare;
        // the first allocation covers 256 batches (a short warm-up call sizes it for long ones)
        const uint64_t cap = std::max<uint64_t>(total, std::max<uint64_t>(2 * t.seed_buf_cap,
                                                                          256ull * t.max_seeds));
        dfree(t.d_seed_buf);
        if (t.h_seed_stage) cudaFreeHost(t.h_seed_stage);
        t.h_seed_stage = nullptr;
        t.d_seed_buf = dalloc<uint32_t>(cap);
        A3G_CUDA(cudaMallocHost(&t.h_seed_stage, cap * 4));
        t.seed_buf_cap = cap;
      }
      std::memcpy(t.h_seed_stage, seeds, total * 4);
      A3G_CUDA(cudaMemcpyAsync(t.d_seed_buf, t.h_seed_stage, total * 4, cudaMemcpyHostToDevice, t.s_samp));
      dseeds = t.d_seed_buf;
    }
    // stream pipeline: step i samples into arena i % kArenas on sampling
    // stream i % 2 (two batches in sampling at once), compute consumes the
    // arenas in order on s_comp; arena reuse waits for its previous compute.
    A3G_CUDA(cudaEventRecord(t.ev_seeds, t.s_samp));
    for (int j = 1; j < TrainerState::kSampStreams; ++j) A3G_CUDA(cudaStreamWaitEvent(t.s_sx[j], t.ev_seeds, 0));
    static const bool tl_env = std::getenv("A3G_TIMELINE") != nullptr;
    // A3G_STEP_TIMES=1: per step, sampling start / end and compute start / end (us)
    static const bool steps_env = std::getenv("A3G_STEP_TIMES") != nullptr;
    std::vector<cudaEvent_t> step_ev;
    const auto host_t0 = std::chrono::steady_clock::now();
    cudaEvent_t tl0 = nullptr;
    const int nss = t.pipe_streams;  // 0: sequential -- sampling on the compute stream, depth 1
    const int narenas = nss == 0 ? 1 : nss + 1;
    for (int i = 1; i < narenas; ++i)
      if (!t.smp[i]) {
        A3G_CUDA(cudaStreamSynchronize(t.s_comp));
        t.smp[i] = new a3g_sampler;
        sampler_alloc(t.smp[i]->st, t.g, t.c, t.max_seeds, t.fanouts.data(), t.L);
      }
    for (uint32_t i = 0; i < K; ++i) {
      const int ar = static_cast<int>(i % narenas);
      a3g_sampler* smp = t.smp[ar];
      cudaStream_t ss = nss == 0 ? t.s_comp : t.s_sx[i % nss];
      if (tl_env && K >= 4 && i == K / 2) {  // trace steps K/2 and K/2+1 (all streams)
        g_tl_on = true;
        A3G_CUDA(cudaEventCreate(&tl0));
        A3G_CUDA(cudaEventRecord(tl0, t.s_comp));
      }
      if (tl_env && K >= 4 && i == K / 2 + 2) g_tl_on = false;
      if (i >= static_cast<uint32_t>(narenas)) A3G_CUDA(cudaStreamWaitEvent(ss, t.ev_consumed[ar], 0));
      cudaEvent_t se[4] = {};
      if (steps_env) {
        for (auto& e : se) A3G_CUDA(cudaEventCreate(&e));
        A3G_CUDA(cudaEventRecord(se[0], ss));
      }
      sample_impl(smp->st, dseeds + off[i], static_cast<uint32_t>(off[i + 1] - off[i]), true, gamma, kind,
                  rng_seeds[i], ss, /*prevalidated=*/!on_device);
      launch_step_stats(t, smp, t.d_stats + static_cast<size_t>(i) * A3G_STEP_STATS, ss);
      A3G_CUDA(cudaEventRecord(t.ev_sampled[ar], ss));
      A3G_CUDA(cudaStreamWaitEvent(t.s_comp, t.ev_sampled[ar], 0));
      if (steps_env) {
        A3G_CUDA(cudaEventRecord(se[1], ss));
        A3G_CUDA(cudaEventRecord(se[2], t.s_comp));
      }
      static const bool skip_compute = std::getenv("A3G_DIAG_SKIP_COMPUTE") != nullptr;  // diagnostics only
      if (!skip_compute) launch_train_compute(t, smp, t.lr, t.d_losses + i, nullptr, t.s_comp, t.timing);
      A3G_CUDA(cudaEventRecord(t.ev_consumed[ar], t.s_comp));
      if (steps_env) {
        A3G_CUDA(cudaEventRecord(se[3], t.s_comp));
        step_ev.insert(step_ev.end(), se, se + 4);
      }
    }
    g_tl_on = false;
    if (steps_env)
      std::fprintf(stderr, "a3g-enqueue %u steps %.1f us\n", K,
                   std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - host_t0).count());
    A3G_CUDA(cudaMemcpyAsync(t.h_losses, t.d_losses, K * 8ull, cudaMemcpyDeviceToHost, t.s_comp));
    A3G_CUDA(cudaEventRecord(t.ev_t1, t.s_comp));
    A3G_CUDA(cudaStreamSynchronize(t.s_comp));
    A3G_CUDA(cudaStreamSynchronize(t.s_samp));
    for (int j = 1; j < TrainerState::kSampStreams; ++j) A3G_CUDA(cudaStreamSynchronize(t.s_sx[j]));
    for (size_t q = 0; q + 3 < step_ev.size(); q += 4) {
      float v[4];
      for (int k = 0; k < 4; ++k) A3G_CUDA(cudaEventElapsedTime(&v[k], t.ev_t0, step_ev[q + k]));
      std::fprintf(stderr, "a3g-step %zu samp %.1f %.1f comp %.1f %.1f\n", q / 4, v[0] * 1e3, v[1] * 1e3,
                   v[2] * 1e3, v[3] * 1e3);
      for (int k = 0; k < 4; ++k) cudaEventDestroy(step_ev[q + k]);
    }
    if (tl0) {  // end time of every traced launch, relative to the first traced step's start
      for (const TlEvent& e : g_tl) {
        float ms = 0;
        cudaEventElapsedTime(&ms, tl0, e.ev);
        std::fprintf(stderr, "a3g-timeline %s %s %.1f\n",
                     e.st == t.s_comp ? "comp" : "samp", e.name, ms * 1e3);
        cudaEventDestroy(e.ev);
      }
      g_tl.clear();
      cudaEventDestroy(tl0);
    }
    t.last_steps = K;
    if (losses_out) std::memcpy(losses_out, t.h_losses, K * 8ull);
    float ms = 0;
    A3G_CUDA(cudaEventElapsedTime(&ms, t.ev_t0, t.ev_t1));
    t.last_total_ms = ms;
    double agg = 0;
    for (size_t i = 0; i + 1 < t.ev_agg.size(); i += 2) {
      float x = 0;
      A3G_CUDA(cudaEventElapsedTime(&x, t.ev_agg[i], t.ev_agg[i + 1]));
      agg += x;
    }
    t.last_agg_launches = t.ev_agg.size() / 2;
    auto avg_pairs = [](const std::vector<cudaEvent_t>& ev) {
      double sum = 0;
      for (size_t i = 0; i + 1 < ev.size(); i += 2) {
        float x = 0;
        A3G_CUDA(cudaEventElapsedTime(&x, ev[i], ev[i + 1]));
        sum += x;
      }
      return ev.size() >= 2 ? sum / static_cast<double>(ev.size() / 2) : 0.0;
    };
    t.last_h1_ms = avg_pairs(t.ev_h1);
    t.last_dw1_ms = avg_pairs(t.ev_dw1);
    t.last_gemm_launches = t.ev_h1.size() / 2;
    t.last_agg_ms = t.last_agg_launches ? agg / t.last_agg_launches : 0;
    unsigned long long words[2] = {0, 0};
    A3G_CUDA(cudaMemcpy(words, t.d_agg_bytes, 16, cudaMemcpyDeviceToHost));
    if (words[1]) raise(A3G_ERR_PARAMETER, "sample_khop: seed out of range");
    const unsigned long long bytes = words[0];
    t.last_agg_bytes = t.last_agg_launches ? static_cast<double>(bytes) / t.last_agg_launches : 0;
  });
}

a3g_status a3g_trainer_step_stats(a3g_trainer* tr, uint64_t* out, uint32_t K) {
  return guard([&] {
    TrainerState& t = tr->st;
    if (K > t.last_steps) raise(A3G_ERR_PARAMETER, "step_stats: more steps than the last train_steps ran");
    if (K == 0) return;
    A3G_CUDA(cudaSetDevice(t.g->device));
    A3G_CUDA(cudaMemcpy(out, t.d_stats, static_cast<size_t>(K) * A3G_STEP_STATS * 8, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < K; ++i) {
      uint64_t* r = out + static_cast<size_t>(i) * A3G_STEP_STATS;
      r[A3G_STAT_MISSES] = r[A3G_STAT_UNIQUE] - r[A3G_STAT_HITS];
    }
  });
}

a3g_status a3g_evaluate_full_graph(a3g_trainer* tr, const uint8_t* test_mask, double* accuracy) {
  return guard([&] {
    TrainerState& t = tr->st;
    A3G_CUDA(cudaSetDevice(t.g->device));
    if (!test_mask) raise(A3G_ERR_PARAMETER, "evaluate_full_graph: test_mask required");
    *accuracy = evaluate_full_graph(t, test_mask);
  });
}

a3g_status a3g_trainer_last_grads(a3g_trainer* tr, double* gw1, double* gw2) {
  return guard([&] {
    TrainerState& t = tr->st;
    A3G_CUDA(cudaSetDevice(t.g->device));
    A3G_CUDA(cudaStreamSynchronize(t.s_comp));
    const size_t FH = static_cast<size_t>(t.F) * t.H, HC = static_cast<size_t>(t.H) * t.C;
    std::vector<float> g(FH + HC);
    A3G_CUDA(cudaMemcpy(g.data(), t.d_gw, g.size() * 4, cudaMemcpyDeviceToHost));
    if (gw1) std::copy(g.begin(), g.begin() + FH, gw1);
    if (gw2) std::copy(g.begin() + FH, g.end(), gw2);
  });
}

a3g_status a3g_trainer_last_forward(a3g_trainer* tr, uint64_t* n_inner, double* logits, double* agg_inner,
                                    double* h1, double* agg_outer) {
  return guard([&] {
    TrainerState& t = tr->st;
    A3G_CUDA(cudaSetDevice(t.g->device));
    A3G_CUDA(cudaStreamSynchronize(t.s_comp));
    SamplerState& s = t.smp[0]->st;  // a3g_train_step uses arena 0
    read_counters(s, t.s_comp);
    const uint64_t ns = s.h_ctr->ucount[0];
    const uint64_t ni = s.L >= 1 ? s.h_ctr->ucount[1] : ns;
    if (n_inner) *n_inner = ni;
    auto fetch = [](double* dst, const float* src, size_t cnt) {
      std::vector<float> tmp(cnt);
      if (cnt) A3G_CUDA(cudaMemcpy(tmp.data(), src, cnt * 4, cudaMemcpyDeviceToHost));
      std::copy(tmp.begin(), tmp.end(), dst);
    };
    if (logits) fetch(logits, t.d_logits, ns * t.C);
    if (h1) fetch(h1, t.d_h1, ni * t.H);
    if (agg_outer) fetch(agg_outer, t.d_agg_outer, ns * t.H);
    if (agg_inner) {
      std::vector<float> tmp(ni * t.pitch);
      if (ni) A3G_CUDA(cudaMemcpy(tmp.data(), t.d_agg_inner, tmp.size() * 4, cudaMemcpyDeviceToHost));
      for (uint64_t r = 0; r < ni; ++r)
        for (uint32_t f = 0; f < t.F; ++f) agg_inner[r * t.F + f] = tmp[r * t.pitch + f];
    }
  });
}

a3g_status a3g_trainer_profile_step(a3g_trainer* tr, const uint32_t* seeds, uint32_t n_seeds, double gamma,
                                    int kind, uint64_t rng_seed, double* stage_ms) {
  return guard([&] {
    TrainerState& t = tr->st;
    A3G_CUDA(cudaSetDevice(t.g->device));
    a3g_sampler* smp = t.smp[0];
    SamplerState& s = smp->st;
    cudaEvent_t ev[5];
    for (auto& e : ev) A3G_CUDA(cudaEventCreate(&e));
    // stage 1: sample_khop (the host seed copy included, as the reference's
    // sample_unit reads host seeds)
    A3G_CUDA(cudaEventRecord(ev[0], t.s_comp));
    sample_impl(s, seeds, n_seeds, false, gamma, kind, rng_seed, t.s_comp);
    A3G_CUDA(cudaEventRecord(ev[1], t.s_comp));
    // stage 2: retrieve_features -- the unique rows gathered into HBM
    read_counters(s, t.s_comp);
    const uint64_t U = s.h_ctr->ucount[s.L];
    const uint64_t need = std::max<uint64_t>(U, 1) * t.F;
    if (need > t.gather_cap) {
      dfree(t.d_gather);
      t.d_gather = dalloc<float>(need);
      t.gather_cap = need;
    }
    A3G_CUDA(cudaEventRecord(ev[2], t.s_comp));
    launch_gather_unique(s, t.d_gather, t.s_comp);
    A3G_CUDA(cudaEventRecord(ev[3], t.s_comp));
    // stage 3: grad_on_batch (lr = 0: the weights are not changed)
    launch_train_compute(t, smp, 0.0, t.d_losses, nullptr, t.s_comp, false);
    A3G_CUDA(cudaEventRecord(ev[4], t.s_comp));
    A3G_CUDA(cudaStreamSynchronize(t.s_comp));
    A3G_CUDA(cudaMemsetAsync(&s.d_ctr->hits, 0, 8, t.s_comp));
    float ms[3];
    A3G_CUDA(cudaEventElapsedTime(&ms[0], ev[0], ev[1]));
    A3G_CUDA(cudaEventElapsedTime(&ms[1], ev[2], ev[3]));
    A3G_CUDA(cudaEventElapsedTime(&ms[2], ev[3], ev[4]));
    for (auto& e : ev) cudaEventDestroy(e);
    for (int i = 0; i < 3; ++i) stage_ms[i] = ms[i];
  });
}

a3g_status a3g_trainer_set_tier_accounting(a3g_trainer* tr, int on) {
  return guard([&] {
    TrainerState& t = tr->st;
    A3G_CUDA(cudaSetDevice(t.g->device));
    A3G_CUDA(cudaStreamSynchronize(t.s_comp));
    if (on && !t.d_tier_seen) {
      const uint64_t words = (t.g->n + 31) / 32;
      t.d_tier_seen = dalloc<uint32_t>(words);
      A3G_CUDA(cudaMemset(t.d_tier_seen, 0, words * 4));
      t.d_tier_rows = dalloc<unsigned long long>(kMaxTiers);
      A3G_CUDA(cudaMemset(t.d_tier_rows, 0, kMaxTiers * 8));
    }
    t.tier_acct = on != 0;
  });
}

a3g_status a3g_trainer_tier_rows(a3g_trainer* tr, uint64_t* rows) {
  return guard([&] {
    TrainerState& t = tr->st;
    A3G_CUDA(cudaSetDevice(t.g->device));
    A3G_CUDA(cudaStreamSynchronize(t.s_comp));
    unsigned long long h[kMaxTiers] = {};
    if (t.d_tier_rows) A3G_CUDA(cudaMemcpy(h, t.d_tier_rows, sizeof h, cudaMemcpyDeviceToHost));
    for (int i = 0; i < kMaxTiers; ++i) rows[i] = h[i];
  });
}

a3g_sampler* a3g_trainer_sampler(a3g_trainer* tr, int slot) {
  a3g_sampler* s = tr->st.smp[static_cast<unsigned>(slot) % TrainerState::kArenas];
  return s ? s : tr->st.smp[0];
}

a3g_status a3g_trainer_timing(a3g_trainer* tr, double* total_ms, double* agg_ms, double* agg_bytes,
                              uint64_t* launches_per_step) {
  return guard([&] {
    TrainerState& t = tr->st;
    if (total_ms) *total_ms = t.last_total_ms;
    if (agg_ms) *agg_ms = t.last_agg_ms;
    if (agg_bytes) *agg_bytes = t.last_agg_bytes;
    // our kernels per step: seeds phase 4 (init, mark, fin count/emit); per
    // layer 6 (classify, item classes, stream, hub merge, fin count/emit);
    // resolve; stats (sampling stream); compute 6 (agg (+fused h1), outer,
    // dh1 scatter, dh1 fix, dW1, reduce (+SGD with one worker)) + the h1 GEMM
    // and its split-K reduce when not fused + scale and SGD with a communicator
    if (launches_per_step)
      *launches_per_step = 4 + 6ull * t.L + (t.L ? 1 : 0) + 1 + 6 + (t.h1_fused ? 0 : 1) +
                           (!t.h1_fused && t.h1_split_used ? 1 : 0) + (t.comm ? 2 : 0) +
                           (t.last_seeds_on_device ? 1 : 0);  // k_check_seeds
  });
}

// ------------------------------------------------------------------- comm
a3g_status a3g_trainer_gemm_timing(a3g_trainer* tr, double* h1_ms, double* dw1_ms, uint64_t* launches) {
  return guard([&] {
    TrainerState& t = tr->st;
    if (h1_ms) *h1_ms = t.last_h1_ms;
    if (dw1_ms) *dw1_ms = t.last_dw1_ms;
    if (launches) *launches = t.last_gemm_launches;
  });
}

a3g_status a3g_comm_unique_id(uint8_t id[128]) {
  return guard([&] { comm_unique_id(id); });
}
a3g_status a3g_comm_create(const uint8_t id[128], int nranks, int rank, int device, a3g_comm** out) {
  return guard([&] { *out = comm_create(id, nranks, rank, device); });
}
a3g_status a3g_comm_create_host(int nranks, int rank, a3g_allreduce_fn fn, void* user, a3g_comm** out) {
  return guard([&] { *out = comm_create_host(nranks, rank, fn, user); });
}
void a3g_comm_destroy(a3g_comm* c) { comm_destroy(c); }

}  // extern "C"
