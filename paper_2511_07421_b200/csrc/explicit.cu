// explicit.cu -- the reference's per-batch model calls on an EXPLICIT batch
// (trainer.cpp:34-239 forward / backward / grad_on_batch, :208-229 sgd_step /
// sync_gradients), for the C++ drop-in: the caller hands a host SampleBatch
// (unique nodes, per-layer (dst_idx, src_idx) edge lists) and the feats array
// it gathered, and the batch runs through the SAME device kernels as the
// stream pipeline (k_agg1, k_outer, k_dh1_scatter/fix, k_dw1_fma, k_reduce).
//
// How an explicit batch becomes a sampler arena (sampler.cuh):
//  * the reference's forward reads inner nodes = unique seeds, then the
//    first-seen layer-0 sources (trainer.cpp:76-89); the batch is relabelled so
//    those come first (new index r < n_inner is inner row r, exactly the
//    layout the sampler produces), the other unique nodes follow in order;
//  * the feats rows are uploaded in the new order into a private feature table
//    (a graph whose node v is new index v), the seed labels into its labels;
//  * layer 0 becomes a padded CSR block over the seeds (row = dst < n_seeds,
//    edge order kept), layer 1 one over the inner rows that own edges (the
//    others fall back to their own row, trainer.cpp:102-107);
//  * edges whose dst the reference skips (layer-0 dst >= n_seeds, layer-1 dst
//    not inner: kSkip, trainer.cpp:36-44, :182-184) are dropped.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "trainer.cuh"

namespace a3g {
namespace {

template <typename T>
T* dalloc_x(size_t n) {
  T* p = nullptr;
  A3G_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  return p;
}

// trainer.cpp:208-211 (kernels::axpy(-lr, g, w)): w[i] += (-lr) * g[i]. The
// first n_fused elements with one fused multiply-add (the AVX2 kernel table
// fuses blocks of four, kernels_avx2.cpp:14-22), the rest with the product
// and the sum rounded separately (its scalar tail, and the scalar table).
__global__ void k_sgd_f64(double* w, const double* g, uint64_t n, uint64_t n_fused, double a) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    w[i] = i < n_fused ? __fma_rn(a, g[i], w[i]) : __dadd_rn(w[i], __dmul_rn(a, g[i]));
}

// trainer.cpp:213-229: out = (sum over k in list order) * (1 / k).
__global__ void k_mean_f64(const double* g, uint32_t k, uint64_t n, double inv, double* out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (uint32_t j = 0; j < k; ++j) s = __dadd_rn(s, g[static_cast<uint64_t>(j) * n + i]);
    out[i] = __dmul_rn(s, inv);
  }
}

}  // namespace
}  // namespace a3g

using namespace a3g;

struct a3g_batch_model {
  int device = 0;
  uint32_t F = 0, H = 0, C = 0;
  // capacities of the private graph / trainer (grown geometrically)
  uint64_t cap_u = 0, cap_s = 0;
  uint32_t cap_f0 = 0, cap_f1 = 0;
  a3g_graph* g = nullptr;
  a3g_cache* c = nullptr;
  a3g_trainer* t = nullptr;
  // the loaded batch (host bookkeeping of the ForwardResult index arrays)
  bool loaded = false;
  uint64_t n_unique = 0, n_seeds = 0, n_inner = 0;
  std::vector<uint32_t> inner_nodes;  // new index r -> original unique index
  std::vector<int32_t> inner_pos;     // original unique index -> inner row, -1
  std::vector<uint32_t> inner_deg, outer_deg;
  bool ran = false;
  double loss = 0.0;

  void release() {
    if (t) a3g_trainer_destroy(t);
    if (c) a3g_cache_destroy(c);
    if (g) a3g_graph_destroy(g);
    t = nullptr;
    c = nullptr;
    g = nullptr;
  }
  ~a3g_batch_model() { release(); }

  // private feature table of cap_u nodes (no edges) + trainer with room for
  // cap_s seeds and fanouts (cap_f0, cap_f1)
  void ensure(uint64_t U, uint64_t S, uint32_t f0, uint32_t f1) {
    if (t && U <= cap_u && S <= cap_s && f0 <= cap_f0 && f1 <= cap_f1) return;
    release();
    auto grow = [](uint64_t need, uint64_t have) { return std::max<uint64_t>(need, have + have / 2); };
    cap_u = grow(std::max<uint64_t>(U, 64), cap_u);
    cap_s = grow(std::max<uint64_t>(S, 16), cap_s);
    cap_f0 = static_cast<uint32_t>(grow(std::max<uint32_t>(f0, 1), cap_f0));
    cap_f1 = static_cast<uint32_t>(grow(std::max<uint32_t>(f1, 1), cap_f1));
    cap_u = std::max<uint64_t>(cap_u, cap_s);
    const std::vector<uint64_t> ro(cap_u + 1, 0);
    // features are written per load; create with none and attach the table here
    A3G_CUDA(cudaSetDevice(device));
    a3g_status st = a3g_graph_create(device, cap_u, 0, F, ro.data(), nullptr, nullptr, A3G_FEAT_F32, nullptr, &g);
    if (st != A3G_OK) raise(st, a3g_last_error());
    const size_t row_bytes = static_cast<size_t>(g->pitch) * 4;
    A3G_CUDA(cudaMalloc(&g->d_feat, cap_u * row_bytes));
    A3G_CUDA(cudaMemset(g->d_feat, 0, cap_u * row_bytes));
    g->view.base[0] = static_cast<const uint8_t*>(g->d_feat);
    g->view.loc = nullptr;
    g->view.row_bytes = static_cast<uint32_t>(row_bytes);
    g->has_features = true;
    st = a3g_cache_from_map(g, nullptr, 1, &c);
    if (st != A3G_OK) raise(st, a3g_last_error());
    const uint32_t fan[2] = {cap_f0, cap_f1};
    st = a3g_trainer_create(g, c, static_cast<uint32_t>(cap_s), fan, 2, H, C, 0.2, 1, &t);
    if (st != A3G_OK) raise(st, a3g_last_error());
  }
};

extern "C" {

a3g_status a3g_batch_model_create(int device, uint32_t F, uint32_t H, uint32_t C, a3g_batch_model** out) {
  return guard([&] {
    if (F < 1 || H < 1 || C < 1) raise(A3G_ERR_PARAMETER, "init_model: dims must be >= 1");
    if (H > 256 || C > 32) raise(A3G_ERR_PARAMETER, "trainer: hidden_dim must be <= 256 and num_classes <= 32");
    auto* m = new a3g_batch_model;
    m->device = device;
    m->F = F;
    m->H = H;
    m->C = C;
    *out = m;
  });
}

void a3g_batch_model_destroy(a3g_batch_model* m) { delete m; }

a3g_status a3g_batch_model_load(a3g_batch_model* m, uint64_t n_unique, uint64_t n_seeds, uint32_t L,
                                const uint64_t* layer_ne, const uint32_t* const* layer_dst,
                                const uint32_t* const* layer_src, const float* feats, const uint32_t* seed_labels,
                                uint64_t* n_inner_out) {
  return guard([&] {
    m->loaded = false;
    m->ran = false;
    if (n_seeds > n_unique) raise(A3G_ERR_PARAMETER, "batch: num_seed_unique > |unique_nodes|");
    if (n_seeds == 0) raise(A3G_ERR_PARAMETER, "batch: no seeds");
    if (n_unique >= (1ull << 32) - 1) raise(A3G_ERR_PARAMETER, "batch: too many unique nodes");
    for (uint32_t l = 0; l < std::min<uint32_t>(L, 2); ++l)
      for (uint64_t e = 0; e < layer_ne[l]; ++e)
        if (layer_dst[l][e] >= n_unique || layer_src[l][e] >= n_unique)
          raise(A3G_ERR_PARAMETER, "batch: edge index out of range");
    const uint64_t U = n_unique, S = n_seeds;
    // ---- inner nodes: seeds, then first-seen layer-0 sources (trainer.cpp:76-89)
    m->inner_pos.assign(U, -1);
    m->inner_nodes.clear();
    for (uint64_t s = 0; s < S; ++s) {
      m->inner_pos[s] = static_cast<int32_t>(s);
      m->inner_nodes.push_back(static_cast<uint32_t>(s));
    }
    const uint64_t e0 = L >= 1 ? layer_ne[0] : 0, e1 = L >= 2 ? layer_ne[1] : 0;
    for (uint64_t e = 0; e < e0; ++e) {
      const uint32_t s = layer_src[0][e];
      if (m->inner_pos[s] < 0) {
        m->inner_pos[s] = static_cast<int32_t>(m->inner_nodes.size());
        m->inner_nodes.push_back(s);
      }
    }
    const uint64_t NI = m->inner_nodes.size();
    // new order: inner rows, then the other unique nodes in index order
    std::vector<uint32_t> new_of(U), old_of;
    old_of.reserve(U);
    for (uint64_t r = 0; r < NI; ++r) old_of.push_back(m->inner_nodes[r]);
    for (uint64_t u = 0; u < U; ++u)
      if (m->inner_pos[u] < 0) old_of.push_back(static_cast<uint32_t>(u));
    for (uint64_t i = 0; i < U; ++i) new_of[old_of[i]] = static_cast<uint32_t>(i);
    // ---- layer 0: padded rows over the seeds (dst < n_seeds, edge order)
    m->outer_deg.assign(S, 0);
    for (uint64_t e = 0; e < e0; ++e)
      if (layer_dst[0][e] < S) ++m->outer_deg[layer_dst[0][e]];
    uint32_t f0 = 1;
    for (uint32_t d : m->outer_deg) f0 = std::max(f0, d);
    // layer 1: rows = inner dsts owning edges, in first-appearance order
    m->inner_deg.assign(NI, 0);
    std::vector<int32_t> row1(NI, -1);
    std::vector<uint32_t> row_dst;  // layer-1 row -> inner row
    for (uint64_t e = 0; e < e1; ++e) {
      const int32_t r = m->inner_pos[layer_dst[1][e]];
      if (r < 0) continue;
      if (row1[r] < 0) {
        row1[r] = static_cast<int32_t>(row_dst.size());
        row_dst.push_back(static_cast<uint32_t>(r));
      }
      ++m->inner_deg[r];
    }
    uint32_t f1 = 1;
    for (uint32_t d : m->inner_deg) f1 = std::max(f1, d);
    // the arena's layer-1 capacity is n_seeds x f0 rows: cover every inner row
    f0 = std::max<uint32_t>(f0, static_cast<uint32_t>((NI + S - 1) / S));
    A3G_CUDA(cudaSetDevice(m->device));
    m->ensure(U, S, f0, f1);
    TrainerState& t = m->t->st;
    SamplerState& s = t.smp[0]->st;
    const uint32_t F0 = s.layer[0].f, F1 = s.layer[1].f;
    std::vector<uint32_t> cnt0(S, 0), sidx0(S * F0, 0);
    for (uint64_t e = 0; e < e0; ++e) {
      const uint32_t d = layer_dst[0][e];
      if (d >= S) continue;
      sidx0[d * F0 + cnt0[d]++] = new_of[layer_src[0][e]];
    }
    const uint64_t R1 = row_dst.size();
    std::vector<uint32_t> cnt1(std::max<uint64_t>(R1, 1), 0), S1(std::max<uint64_t>(R1, 1) * F1, 0);
    for (uint64_t e = 0; e < e1; ++e) {
      const int32_t r = m->inner_pos[layer_dst[1][e]];
      if (r < 0) continue;
      const uint32_t k = static_cast<uint32_t>(row1[r]);
      S1[k * F1 + cnt1[k]++] = new_of[layer_src[1][e]];
    }
    std::vector<int32_t> inv1(NI);
    for (uint64_t r = 0; r < NI; ++r) inv1[r] = row1[r];
    // distinct layer-1 sources (the gather's algorithmic byte count)
    uint64_t distinct = 0;
    {
      std::vector<uint8_t> seen(U, 0);
      for (uint64_t e = 0; e < e1; ++e)
        if (m->inner_pos[layer_dst[1][e]] >= 0 && !seen[layer_src[1][e]]) {
          seen[layer_src[1][e]] = 1;
          ++distinct;
        }
    }
    // ---- upload: features (new order, pitched), labels, arena, counters
    a3g_graph* g = m->g;
    const uint32_t pitch = g->pitch;
    {
      const uint64_t slab = std::max<uint64_t>(1, (32ull << 20) / (pitch * 4ull));
      std::vector<float> stage(slab * pitch, 0.f);
      for (uint64_t v0 = 0; v0 < U; v0 += slab) {
        const uint64_t cnt = std::min<uint64_t>(slab, U - v0);
        for (uint64_t i = 0; i < cnt; ++i)
          std::memcpy(stage.data() + i * pitch, feats + static_cast<uint64_t>(old_of[v0 + i]) * m->F, m->F * 4ull);
        A3G_CUDA(cudaMemcpy(static_cast<float*>(g->d_feat) + v0 * pitch, stage.data(), cnt * pitch * 4ull,
                            cudaMemcpyHostToDevice));
      }
    }
    std::vector<uint32_t> lab(S, 0);
    if (seed_labels) std::copy(seed_labels, seed_labels + S, lab.begin());
    A3G_CUDA(cudaMemcpy(g->d_labels, lab.data(), S * 4, cudaMemcpyHostToDevice));
    std::vector<uint32_t> iota(U);
    std::iota(iota.begin(), iota.end(), 0u);
    A3G_CUDA(cudaMemcpy(s.d_unique, iota.data(), U * 4, cudaMemcpyHostToDevice));
    A3G_CUDA(cudaMemcpy(s.layer[0].cnt, cnt0.data(), S * 4, cudaMemcpyHostToDevice));
    A3G_CUDA(cudaMemcpy(s.layer[0].sidx, sidx0.data(), S * F0 * 4ull, cudaMemcpyHostToDevice));
    A3G_CUDA(cudaMemcpy(s.layer[0].S, sidx0.data(), S * F0 * 4ull, cudaMemcpyHostToDevice));
    if (R1) {
      A3G_CUDA(cudaMemcpy(s.layer[1].cnt, cnt1.data(), R1 * 4, cudaMemcpyHostToDevice));
      A3G_CUDA(cudaMemcpy(s.layer[1].S, S1.data(), R1 * F1 * 4ull, cudaMemcpyHostToDevice));
      A3G_CUDA(cudaMemcpy(s.layer[1].sidx, S1.data(), R1 * F1 * 4ull, cudaMemcpyHostToDevice));
    }
    A3G_CUDA(cudaMemcpy(s.d_inv1, inv1.data(), NI * 4, cudaMemcpyHostToDevice));
    BatchCounters hc{};
    hc.n_seeds = static_cast<uint32_t>(S);
    hc.nfront[0] = static_cast<uint32_t>(S);
    hc.nfront[1] = static_cast<uint32_t>(R1);
    hc.nfront[2] = static_cast<uint32_t>(distinct);
    hc.ucount[0] = static_cast<uint32_t>(S);
    hc.ucount[1] = static_cast<uint32_t>(NI);
    hc.ucount[2] = static_cast<uint32_t>(U);
    hc.edges[0] = static_cast<uint32_t>(e0);
    hc.edges[1] = static_cast<uint32_t>(e1);
    A3G_CUDA(cudaMemcpy(s.d_ctr, &hc, sizeof hc, cudaMemcpyHostToDevice));
    s.has_batch = true;
    s.last_n_seeds = static_cast<uint32_t>(S);
    m->n_unique = U;
    m->n_seeds = S;
    m->n_inner = NI;
    m->loaded = true;
    if (n_inner_out) *n_inner_out = NI;
  });
}

a3g_status a3g_batch_model_run(a3g_batch_model* m, const double* w1, const double* w2, double* loss, double* gw1,
                               double* gw2) {
  return guard([&] {
    if (!m->loaded) raise(A3G_ERR_PARAMETER, "batch model: no batch loaded");
    A3G_CUDA(cudaSetDevice(m->device));
    a3g_status st = a3g_trainer_set_weights(m->t, w1, w2);
    if (st != A3G_OK) raise(st, a3g_last_error());
    TrainerState& t = m->t->st;
    // lr = 0: gradients only (the SGD riding on the reduction leaves W unchanged)
    launch_train_compute(t, t.smp[0], 0.0, t.d_losses, nullptr, t.s_comp, false);
    A3G_CUDA(cudaMemcpyAsync(t.h_losses, t.d_losses, 8, cudaMemcpyDeviceToHost, t.s_comp));
    A3G_CUDA(cudaStreamSynchronize(t.s_comp));
    m->loss = t.h_losses[0];
    m->ran = true;
    if (loss) *loss = m->loss;
    if (gw1 || gw2) {
      st = a3g_trainer_last_grads(m->t, gw1, gw2);
      if (st != A3G_OK) raise(st, a3g_last_error());
    }
  });
}

a3g_status a3g_batch_model_forward(a3g_batch_model* m, uint32_t* inner_nodes, int32_t* inner_pos,
                                   uint32_t* inner_deg, uint32_t* outer_deg, double* agg_inner, double* h1,
                                   double* agg_outer, double* logits) {
  return guard([&] {
    if (!m->ran) raise(A3G_ERR_PARAMETER, "batch model: no forward computed");
    if (inner_nodes) std::copy(m->inner_nodes.begin(), m->inner_nodes.end(), inner_nodes);
    if (inner_pos) std::copy(m->inner_pos.begin(), m->inner_pos.end(), inner_pos);
    if (inner_deg) std::copy(m->inner_deg.begin(), m->inner_deg.end(), inner_deg);
    if (outer_deg) std::copy(m->outer_deg.begin(), m->outer_deg.end(), outer_deg);
    // inner rows are rows [0, n_inner) of the device arrays, in the reference's order
    uint64_t ni = 0;
    std::vector<double> lg(m->t->st.max_seeds * static_cast<uint64_t>(m->C));
    std::vector<double> ao(m->t->st.max_seeds * static_cast<uint64_t>(m->H));
    const a3g_status st = a3g_trainer_last_forward(m->t, &ni, lg.data(), agg_inner, h1, ao.data());
    if (st != A3G_OK) raise(st, a3g_last_error());
    if (ni != m->n_inner) raise(A3G_ERR_CUDA, "batch model: inner row count mismatch");
    if (logits) std::copy(lg.begin(), lg.begin() + m->n_seeds * m->C, logits);
    if (agg_outer) std::copy(ao.begin(), ao.begin() + m->n_seeds * m->H, agg_outer);
  });
}

a3g_status a3g_sgd_step(int device, double* w, const double* g, uint64_t n, uint64_t n_fused, double lr) {
  return guard([&] {
    if (n == 0) return;
    A3G_CUDA(cudaSetDevice(device));
    double* d = dalloc_x<double>(2 * n);
    A3G_CUDA(cudaMemcpy(d, w, n * 8, cudaMemcpyHostToDevice));
    A3G_CUDA(cudaMemcpy(d + n, g, n * 8, cudaMemcpyHostToDevice));
    k_sgd_f64<<<static_cast<int>(std::min<uint64_t>((n + 255) / 256, 1024)), 256>>>(d, d + n, n, std::min(n, n_fused), -lr);
    A3G_LAUNCH_CHECK("k_sgd_f64");
    A3G_CUDA(cudaMemcpy(w, d, n * 8, cudaMemcpyDeviceToHost));
    cudaFree(d);
  });
}

a3g_status a3g_mean_gradients(int device, const double* const* grads, uint32_t k, uint64_t n, double* out) {
  return guard([&] {
    if (k == 0) raise(A3G_ERR_PARAMETER, "sync_gradients: empty gradient list");
    if (n == 0) return;
    A3G_CUDA(cudaSetDevice(device));
    double* d = dalloc_x<double>((static_cast<uint64_t>(k) + 1) * n);
    for (uint32_t j = 0; j < k; ++j)
      A3G_CUDA(cudaMemcpy(d + static_cast<uint64_t>(j) * n, grads[j], n * 8, cudaMemcpyHostToDevice));
    double* o = d + static_cast<uint64_t>(k) * n;
    k_mean_f64<<<static_cast<int>(std::min<uint64_t>((n + 255) / 256, 1024)), 256>>>(d, k, n,
                                                                                       1.0 / static_cast<double>(k), o);
    A3G_LAUNCH_CHECK("k_mean_f64");
    A3G_CUDA(cudaMemcpy(out, o, n * 8, cudaMemcpyDeviceToHost));
    cudaFree(d);
  });
}

}  // extern "C"
