// eval.cu -- full-graph evaluation (proj/src/trainer.cpp:241-303) on sm_100a.
//
// The reference widens every feature row, aggregates the full neighbourhood
// (mean, self-fallback for deg 0), applies ReLU(agg . W1), aggregates again,
// multiplies by W2 and takes the argmax (first maximum) over the test mask.
// On the device the first aggregation is re-associated as mean(X_w . W1)
// (equal in exact arithmetic; fp32 rounding differs from the fp64 reference):
//   k_eval_xw          XW = X . W1            (one pass over the feature store)
//   k_eval_spmm        mean over each CSR row of an n x H table (warp per row;
//                      rows with deg > kEvalChunk are split into chunk items)
//   k_eval_hub_part    chunk partial sums of the split rows
//   k_eval_hub_reduce  adds a split row's partials in chunk order (deterministic)
//   k_eval_argmax      logits = agg2 . W2, first-max argmax, label compare.
// HBM traffic: one read of X plus 2 x m x H x 4 bytes of table gathers, instead
// of m x F x s_f for aggregating raw features.
#include <algorithm>
#include <vector>

#include "trainer.cuh"

namespace a3g {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr uint64_t kEvalChunk = 8192;  // edges per warp item of a split row

template <typename T>
__device__ __forceinline__ float elem(const T* row, uint32_t f);
template <>
__device__ __forceinline__ float elem<float>(const float* row, uint32_t f) {
  return __ldg(row + f);
}
template <>
__device__ __forceinline__ float elem<uint16_t>(const uint16_t* row, uint32_t f) {
  return __uint_as_float(static_cast<uint32_t>(__ldg(row + f)) << 16);
}

// Sum HP per-lane partial vectors across the warp. Returns the total of
// output o_of(lane) (every lane ends with one output; lanes sharing the same
// top log2(HP) bits hold the same output).
template <int HP>
__device__ __forceinline__ float transpose_reduce(float (&p)[HP], int lane, int& o) {
  o = 0;
  int len = HP;
#pragma unroll
  for (int off = 16, lvl = 0; lvl < 5; off >>= 1, ++lvl) {
    if (len > 1) {
      const bool up = lane & off;
      const int half = len / 2;
#pragma unroll
      for (int i = 0; i < HP / 2; ++i) {
        if (i < half) {
          const float send = up ? p[i] : p[i + half];
          const float keep = up ? p[i + half] : p[i];
          p[i] = keep + __shfl_xor_sync(kFull, send, off);
        }
      }
      if (up) o += half;
      len = half;
    } else {
      p[0] += __shfl_xor_sync(kFull, p[0], off);
    }
  }
  return p[0];
}

// XW[v, :] = X[v, :] . W1 (warp per row, lane-strided row read).
template <typename T, int HP>
__global__ void __launch_bounds__(256) k_eval_xw(const __grid_constant__ StoreView view, uint64_t n, uint32_t F,
                                                 uint32_t H, const float* w1, float* xw) {
  extern __shared__ float s_w1[];  // F x HP (zero padded)
  for (uint32_t i = threadIdx.x; i < F * HP; i += blockDim.x) {
    const uint32_t f = i / HP, o = i % HP;
    s_w1[i] = o < H ? w1[f * H + o] : 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t v = gw; v < n; v += nw) {
    const T* row = reinterpret_cast<const T*>(row_ptr(view, static_cast<uint32_t>(v)));
    float p[HP];
#pragma unroll
    for (int o = 0; o < HP; ++o) p[o] = 0.f;
    for (uint32_t f = lane; f < F; f += 32) {
      const float x = elem<T>(row, f);
      const float* w = s_w1 + f * HP;
#pragma unroll
      for (int o = 0; o < HP; ++o) p[o] = fmaf(x, w[o], p[o]);
    }
    int o;
    const float r = transpose_reduce<HP>(p, lane, o);
    if ((lane & (32 / HP - 1)) == 0 && o < static_cast<int>(H)) xw[v * H + o] = r;
  }
}

// Row mean over an n x H table: out[v] = mean_{w in N(v)} tab[w] (self row
// when deg 0), optional ReLU. Lanes: o = lane % HP (column), g = lane / HP
// (edge group). Rows with deg > kEvalChunk are left to the hub kernels.
template <int HP>
__global__ void __launch_bounds__(256) k_eval_spmm(const uint64_t* ro, const uint32_t* col, uint64_t n, uint32_t H,
                                                   const float* tab, int relu, float* out) {
  constexpr int G = 32 / HP;
  const int lane = threadIdx.x & 31;
  const int o = lane % HP, g = lane / HP;
  const bool on = o < static_cast<int>(H);
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t v = gw; v < n; v += nw) {
    const uint64_t b = __ldg(ro + v), e = __ldg(ro + v + 1);
    const uint64_t deg = e - b;
    if (deg > kEvalChunk) continue;
    float acc = 0.f;
    if (deg == 0) {
      acc = on ? tab[v * H + o] : 0.f;  // self-fallback (trainer.cpp:259-260, 276-277)
    } else {
      float a0 = 0.f, a1 = 0.f;
      uint64_t j = b + g;
      for (; j + G < e; j += 2 * G) {
        const uint32_t w0 = __ldg(col + j), w1 = __ldg(col + j + G);
        if (on) {
          a0 += __ldg(tab + static_cast<uint64_t>(w0) * H + o);
          a1 += __ldg(tab + static_cast<uint64_t>(w1) * H + o);
        }
      }
      if (j < e && on) a0 += __ldg(tab + static_cast<uint64_t>(__ldg(col + j)) * H + o);
      acc = a0 + a1;
#pragma unroll
      for (int off = HP; off < 32; off <<= 1) acc += __shfl_xor_sync(kFull, acc, off);
      acc *= 1.f / static_cast<float>(deg);
    }
    if (relu) acc = fmaxf(acc, 0.f);
    if (g == 0 && on) out[v * H + o] = acc;
  }
}

struct HubItem {
  uint32_t row, part;
};

template <int HP>
__global__ void __launch_bounds__(256) k_eval_hub_part(const uint64_t* ro, const uint32_t* col, const HubItem* items,
                                                       uint32_t n_items, uint32_t H, const float* tab, float* part) {
  constexpr int G = 32 / HP;
  const int lane = threadIdx.x & 31;
  const int o = lane % HP, g = lane / HP;
  const bool on = o < static_cast<int>(H);
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = gw; it < n_items; it += nw) {
    const HubItem hi = items[it];
    const uint64_t rb = ro[hi.row], re = ro[hi.row + 1];
    const uint64_t b = rb + static_cast<uint64_t>(hi.part) * kEvalChunk;
    const uint64_t e = min(re, b + kEvalChunk);
    float a0 = 0.f, a1 = 0.f;
    uint64_t j = b + g;
    for (; j + G < e; j += 2 * G) {
      const uint32_t w0 = __ldg(col + j), w1 = __ldg(col + j + G);
      if (on) {
        a0 += __ldg(tab + static_cast<uint64_t>(w0) * H + o);
        a1 += __ldg(tab + static_cast<uint64_t>(w1) * H + o);
      }
    }
    if (j < e && on) a0 += __ldg(tab + static_cast<uint64_t>(__ldg(col + j)) * H + o);
    float acc = a0 + a1;
#pragma unroll
    for (int off = HP; off < 32; off <<= 1) acc += __shfl_xor_sync(kFull, acc, off);
    if (g == 0 && on) part[static_cast<uint64_t>(it) * H + o] = acc;
  }
}

// Split rows: items of row r are contiguous [first[r], first[r+1]).
__global__ void k_eval_hub_reduce(const uint64_t* ro, const uint32_t* hub_rows, const uint32_t* hub_first,
                                  uint32_t n_hubs, uint32_t H, const float* part, int relu, float* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_hubs * H; i += gridDim.x * blockDim.x) {
    const uint32_t h = i / H, o = i % H;
    const uint32_t r = hub_rows[h];
    float acc = 0.f;
    for (uint32_t it = hub_first[h]; it < hub_first[h + 1]; ++it) acc += part[static_cast<uint64_t>(it) * H + o];
    acc *= 1.f / static_cast<float>(ro[r + 1] - ro[r]);
    out[static_cast<uint64_t>(r) * H + o] = relu ? fmaxf(acc, 0.f) : acc;
  }
}

__global__ void __launch_bounds__(256) k_eval_argmax(const float* agg2, uint64_t n, uint32_t H, uint32_t C,
                                                     const float* w2, const uint32_t* labels, const uint8_t* mask,
                                                     unsigned long long* counts) {
  __shared__ float s_w2[32 * 32];
  for (uint32_t i = threadIdx.x; i < H * C; i += blockDim.x) s_w2[i] = w2[i];
  __syncthreads();
  uint32_t correct = 0, total = 0;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (!mask[v]) continue;
    const float* a = agg2 + v * H;
    float best_z = 0.f;
    uint32_t best = 0;
    for (uint32_t c = 0; c < C; ++c) {
      float z = 0.f;
      for (uint32_t j = 0; j < H; ++j) z = fmaf(a[j], s_w2[j * C + c], z);
      if (c == 0 || z > best_z) {  // first maximum (trainer.cpp:292-295)
        best_z = z;
        best = c;
      }
    }
    ++total;
    correct += best == labels[v] ? 1u : 0u;
  }
  correct = __reduce_add_sync(kFull, correct);
  total = __reduce_add_sync(kFull, total);
  if ((threadIdx.x & 31) == 0) {
    if (correct) atomicAdd(counts, static_cast<unsigned long long>(correct));
    if (total) atomicAdd(counts + 1, static_cast<unsigned long long>(total));
  }
}

template <int HP>
void run_eval(TrainerState& t, float* xw, float* h1, float* agg2, float* part, const HubItem* d_items,
              uint32_t n_items, const uint32_t* d_hub_rows, const uint32_t* d_hub_first, uint32_t n_hubs,
              cudaStream_t st) {
  a3g_graph* g = t.g;
  const uint64_t n = g->n;
  const int grid = t.sm_count * 8;
  const size_t smem = static_cast<size_t>(t.F) * HP * sizeof(float);
  if (g->feat_dtype == A3G_FEAT_BF16) {
    A3G_CUDA(cudaFuncSetAttribute(k_eval_xw<uint16_t, HP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    k_eval_xw<uint16_t, HP><<<grid, 256, smem, st>>>(g->view, n, t.F, t.H, t.d_w1, xw);
  } else {
    A3G_CUDA(cudaFuncSetAttribute(k_eval_xw<float, HP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    k_eval_xw<float, HP><<<grid, 256, smem, st>>>(g->view, n, t.F, t.H, t.d_w1, xw);
  }
  A3G_LAUNCH_CHECK("k_eval_xw");
  const float* src[2] = {xw, h1};
  float* dst[2] = {h1, agg2};
  for (int layer = 0; layer < 2; ++layer) {
    const int relu = layer == 0 ? 1 : 0;
    k_eval_spmm<HP><<<grid, 256, 0, st>>>(g->d_ro, g->d_col, n, t.H, src[layer], relu, dst[layer]);
    A3G_LAUNCH_CHECK("k_eval_spmm");
    if (n_items) {
      k_eval_hub_part<HP><<<t.sm_count * 4, 256, 0, st>>>(g->d_ro, g->d_col, d_items, n_items, t.H, src[layer],
                                                           part);
      A3G_LAUNCH_CHECK("k_eval_hub_part");
      k_eval_hub_reduce<<<std::max(1u, (n_hubs * t.H + 255) / 256), 256, 0, st>>>(
          g->d_ro, d_hub_rows, d_hub_first, n_hubs, t.H, part, relu, dst[layer]);
      A3G_LAUNCH_CHECK("k_eval_hub_reduce");
    }
  }
}

}  // namespace

double evaluate_full_graph(TrainerState& t, const uint8_t* test_mask) {
  a3g_graph* g = t.g;
  const uint64_t n = g->n;
  if (t.H > 32 || t.C > 32) raise(A3G_ERR_PARAMETER, "evaluate_full_graph: hidden/classes must be <= 32");
  // split rows (deg > kEvalChunk) and their chunk items, from the host CSR
  std::vector<HubItem> items;
  std::vector<uint32_t> hub_rows, hub_first;
  for (uint64_t v = 0; v < n; ++v) {
    const uint64_t deg = g->h_ro[v + 1] - g->h_ro[v];
    if (deg <= kEvalChunk) continue;
    hub_rows.push_back(static_cast<uint32_t>(v));
    hub_first.push_back(static_cast<uint32_t>(items.size()));
    for (uint32_t p = 0; static_cast<uint64_t>(p) * kEvalChunk < deg; ++p)
      items.push_back(HubItem{static_cast<uint32_t>(v), p});
  }
  hub_first.push_back(static_cast<uint32_t>(items.size()));
  cudaStream_t st = t.s_comp;
  A3G_CUDA(cudaStreamSynchronize(st));
  float *xw = nullptr, *h1 = nullptr, *agg2 = nullptr, *part = nullptr;
  HubItem* d_items = nullptr;
  uint32_t *d_hub_rows = nullptr, *d_hub_first = nullptr;
  uint8_t* d_mask = nullptr;
  unsigned long long* d_counts = nullptr;
  double acc = 0;
  auto cleanup = [&] {
    cudaFree(xw);
    cudaFree(h1);
    cudaFree(agg2);
    cudaFree(part);
    cudaFree(d_items);
    cudaFree(d_hub_rows);
    cudaFree(d_hub_first);
    cudaFree(d_mask);
    cudaFree(d_counts);
  };
  try {
    const size_t tab = std::max<uint64_t>(1, n * t.H) * sizeof(float);
    A3G_CUDA(cudaMalloc(&xw, tab));
    A3G_CUDA(cudaMalloc(&h1, tab));
    A3G_CUDA(cudaMalloc(&agg2, tab));
    A3G_CUDA(cudaMalloc(&part, std::max<size_t>(1, items.size()) * t.H * sizeof(float)));
    A3G_CUDA(cudaMalloc(&d_items, std::max<size_t>(1, items.size()) * sizeof(HubItem)));
    A3G_CUDA(cudaMalloc(&d_hub_rows, std::max<size_t>(1, hub_rows.size()) * 4));
    A3G_CUDA(cudaMalloc(&d_hub_first, hub_first.size() * 4));
    A3G_CUDA(cudaMalloc(&d_mask, std::max<uint64_t>(1, n)));
    A3G_CUDA(cudaMalloc(&d_counts, 16));
    if (!items.empty()) {
      A3G_CUDA(cudaMemcpy(d_items, items.data(), items.size() * sizeof(HubItem), cudaMemcpyHostToDevice));
      A3G_CUDA(cudaMemcpy(d_hub_rows, hub_rows.data(), hub_rows.size() * 4, cudaMemcpyHostToDevice));
    }
    A3G_CUDA(cudaMemcpy(d_hub_first, hub_first.data(), hub_first.size() * 4, cudaMemcpyHostToDevice));
    A3G_CUDA(cudaMemcpy(d_mask, test_mask, n, cudaMemcpyHostToDevice));
    A3G_CUDA(cudaMemset(d_counts, 0, 16));
    const uint32_t ni = static_cast<uint32_t>(items.size()), nh = static_cast<uint32_t>(hub_rows.size());
    const uint32_t HP = t.H <= 1 ? 1 : t.H <= 2 ? 2 : t.H <= 4 ? 4 : t.H <= 8 ? 8 : t.H <= 16 ? 16 : 32;
    switch (HP) {
      case 1: run_eval<1>(t, xw, h1, agg2, part, d_items, ni, d_hub_rows, d_hub_first, nh, st); break;
      case 2: run_eval<2>(t, xw, h1, agg2, part, d_items, ni, d_hub_rows, d_hub_first, nh, st); break;
      case 4: run_eval<4>(t, xw, h1, agg2, part, d_items, ni, d_hub_rows, d_hub_first, nh, st); break;
      case 8: run_eval<8>(t, xw, h1, agg2, part, d_items, ni, d_hub_rows, d_hub_first, nh, st); break;
      case 16: run_eval<16>(t, xw, h1, agg2, part, d_items, ni, d_hub_rows, d_hub_first, nh, st); break;
      default: run_eval<32>(t, xw, h1, agg2, part, d_items, ni, d_hub_rows, d_hub_first, nh, st); break;
    }
    k_eval_argmax<<<t.sm_count * 4, 256, 0, st>>>(agg2, n, t.H, t.C, t.d_w2, g->d_labels, d_mask, d_counts);
    A3G_LAUNCH_CHECK("k_eval_argmax");
    unsigned long long counts[2] = {0, 0};
    A3G_CUDA(cudaMemcpyAsync(counts, d_counts, 16, cudaMemcpyDeviceToHost, st));
    A3G_CUDA(cudaStreamSynchronize(st));
    if (counts[1] == 0) raise(A3G_ERR_CONFIG, "evaluate_full_graph: no test nodes");
    acc = static_cast<double>(counts[0]) / static_cast<double>(counts[1]);
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
  return acc;
}

}  // namespace a3g
