// train.cu -- fused gather + mean aggregation + dense update, forward and
// backward, for the reference's 2-layer mean-GCN (proj/src/trainer.cpp:59-211)
// in fp32 on sm_100a.
//
//   k_agg1        inner rows: gather the layer-1 source rows straight from the
//                 HBM feature store (128-bit loads), mean (self-fallback when
//                 empty, trainer.cpp:93-107), store agg_inner, then
//                 h1 = ReLU(agg_inner . W1) from shared-memory W1
//                 (trainer.cpp:110-113). THE roofline kernel (HBM-bound).
//   k_outer       per seed: agg_outer (trainer.cpp:116-127), logits,
//                 softmax-CE + dlogits (trainer.cpp:153-171),
//                 dagg_outer = dlogits . W2^T (:177-179) and its scatter into
//                 dh1 with 1/deg + fallback (:182-198).
//   k_dw1_partial dW1 = agg_inner^T . (dh1 * [h1>0]) (:200-204), per-block
//                 partials over row ranges.
//   k_reduce      deterministic reduction of the partials, dW2 (:174-175),
//                 mean loss.
//   k_sgd         w -= lr * g (trainer.cpp:208-211).
#include <cmath>

#include <cub/device/device_radix_sort.cuh>

#include "trainer.cuh"

namespace a3g {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kAggThreads = 256;
constexpr int kAggWarps = kAggThreads / 32;

template <typename T>
struct Chunk;
// 16 bytes of a feature row -> EPC floats
template <>
struct Chunk<float> {
  static constexpr int EPC = 4;
  __device__ __forceinline__ static void add(float* acc, uint4 q) {
    acc[0] += __uint_as_float(q.x);
    acc[1] += __uint_as_float(q.y);
    acc[2] += __uint_as_float(q.z);
    acc[3] += __uint_as_float(q.w);
  }
};
template <>
struct Chunk<uint16_t> {  // bf16
  static constexpr int EPC = 8;
  __device__ __forceinline__ static void add(float* acc, uint4 q) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      acc[2 * i] += __uint_as_float(w[i] << 16);
      acc[2 * i + 1] += __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};

struct AggArgs {
  StoreView view;  // feature rows: local HBM / NVLink peer / pinned host (store.cu)
  uint32_t pitch, F, H;
  const uint32_t* unique;
  const int32_t* inv1;
  const uint32_t* cnt1;
  const uint32_t* S1;
  uint32_t f1;
  const uint32_t* n_inner;
  const float* w1;
  float* agg_inner;
  float* h1;
  unsigned long long* bytes;
  int has_layer1;
};

template <typename T, int NCH>
__global__ void __launch_bounds__(kAggThreads) k_agg1(const __grid_constant__ AggArgs a) {
  using Ch = Chunk<T>;
  constexpr int EPC = Ch::EPC;
  extern __shared__ float smem[];
  float* s_w1 = smem;                                   // F x H
  float* s_buf = smem + (static_cast<size_t>(a.F) * a.H + 7) / 8 * 8;  // kAggWarps x pitch, 32B aligned
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < a.F * a.H; i += kAggThreads) s_w1[i] = a.w1[i];
  __syncthreads();
  float* buf = s_buf + static_cast<size_t>(warp) * a.pitch;
  const uint32_t n_inner = *a.n_inner;
  const uint32_t chunks = a.pitch / EPC;  // 16-byte chunks per row
  unsigned long long nbytes = 0;
  const uint32_t gw = blockIdx.x * kAggWarps + warp, nw = gridDim.x * kAggWarps;
  const uint32_t H = a.H, F = a.F;
  const bool pow2 = H <= 32 && (32 % H) == 0;
  for (uint32_t r = gw; r < n_inner; r += nw) {
    const int32_t k = a.has_layer1 ? __ldg(a.inv1 + r) : -1;
    const uint32_t c = k >= 0 ? __ldg(a.cnt1 + k) : 0u;
    float acc[NCH][EPC];
#pragma unroll
    for (int i = 0; i < NCH; ++i)
#pragma unroll
      for (int e = 0; e < EPC; ++e) acc[i][e] = 0.f;
    float scale = 1.f;
    if (c == 0) {  // self-fallback: own features (trainer.cpp:102-107)
      const uint4* row = reinterpret_cast<const uint4*>(row_ptr(a.view, __ldg(a.unique + r)));
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const uint32_t q = lane + 32 * i;
        if (q < chunks) Ch::add(acc[i], __ldg(row + q));
      }
      nbytes += static_cast<unsigned long long>(F) * sizeof(T) + 4;
    } else {
      const uint32_t* srcs = a.S1 + static_cast<uint64_t>(k) * a.f1;
      uint32_t t = 0;
      for (; t + 1 < c; t += 2) {
        const uint4* r0 = reinterpret_cast<const uint4*>(row_ptr(a.view, __ldg(srcs + t)));
        const uint4* r1 = reinterpret_cast<const uint4*>(row_ptr(a.view, __ldg(srcs + t + 1)));
        uint4 x0[NCH], x1[NCH];
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const uint32_t q = lane + 32 * i;
          if (q < chunks) {
            x0[i] = __ldg(r0 + q);
            x1[i] = __ldg(r1 + q);
          }
        }
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const uint32_t q = lane + 32 * i;
          if (q < chunks) {
            Ch::add(acc[i], x0[i]);
            Ch::add(acc[i], x1[i]);
          }
        }
      }
      if (t < c) {
        const uint4* r0 = reinterpret_cast<const uint4*>(row_ptr(a.view, __ldg(srcs + t)));
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const uint32_t q = lane + 32 * i;
          if (q < chunks) Ch::add(acc[i], __ldg(r0 + q));
        }
      }
      scale = 1.f / static_cast<float>(c);
      nbytes += static_cast<unsigned long long>(c) * (static_cast<unsigned long long>(F) * sizeof(T) + 4) + 8;
    }
    // agg_inner row (pitched f32) + smem copy for the GEMM
    float4* out = reinterpret_cast<float4*>(a.agg_inner + static_cast<uint64_t>(r) * a.pitch);
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const uint32_t q = lane + 32 * i;
      if (q < chunks) {
#pragma unroll
        for (int e = 0; e < EPC; e += 4) {
          const float4 v = make_float4(acc[i][e] * scale, acc[i][e + 1] * scale, acc[i][e + 2] * scale,
                                       acc[i][e + 3] * scale);
          out[q * (EPC / 4) + e / 4] = v;
          reinterpret_cast<float4*>(buf)[q * (EPC / 4) + e / 4] = v;
        }
      }
    }
    __syncwarp();
    // h1 = ReLU(agg . W1)
    if (pow2) {
      const uint32_t G = 32 / H, o = lane % H, g = lane / H;
      const uint32_t KF = (F + G - 1) / G;
      const uint32_t f0 = g * KF, f1e = min(F, f0 + KF);
      float sum = 0.f;
      for (uint32_t f = f0; f < f1e; ++f) sum = fmaf(buf[f], s_w1[f * H + o], sum);
      for (uint32_t off = H; off < 32; off <<= 1) sum += __shfl_xor_sync(kFull, sum, off);
      if (g == 0) a.h1[static_cast<uint64_t>(r) * H + o] = fmaxf(sum, 0.f);
    } else {
      for (uint32_t o = lane; o < H; o += 32) {
        float sum = 0.f;
        for (uint32_t f = 0; f < F; ++f) sum = fmaf(buf[f], s_w1[f * H + o], sum);
        a.h1[static_cast<uint64_t>(r) * H + o] = fmaxf(sum, 0.f);
      }
    }
    nbytes += static_cast<unsigned long long>(F) * 4 + static_cast<unsigned long long>(H) * 4;
    __syncwarp();
  }
  if (lane == 0 && nbytes) atomicAdd(a.bytes, nbytes);
}

// Per-step statistics (a3g_trainer_step_stats): batch sizes from the sampler's
// counters and the cache hit/miss count over unique_nodes (lookup,
// cache.cpp:48-68: any-device presence is a hit).
__global__ void k_step_stats(const BatchCounters* ctr, const uint32_t* unique, const uint32_t* bits, int bitmode,
                             uint32_t L, unsigned long long* out) {
  const uint32_t U = ctr->ucount[L];
  const int lane = threadIdx.x & 31;
  uint32_t hits = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < U; i += gridDim.x * blockDim.x) {
    const uint32_t v = unique[i];
    hits += (bitmode == 1 || (bitmode == 2 && ((__ldg(bits + (v >> 5)) >> (v & 31)) & 1u))) ? 1u : 0u;
  }
  hits = __reduce_add_sync(kFull, hits);
  if (lane == 0 && hits) atomicAdd(out + A3G_STAT_HITS, static_cast<unsigned long long>(hits));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t E = 0;
    for (uint32_t l = 0; l < L; ++l) E += ctr->edges[l];
    out[A3G_STAT_UNIQUE] = U;
    out[A3G_STAT_EDGES] = E;
    out[A3G_STAT_INNER] = L >= 1 ? ctr->ucount[1] : ctr->ucount[0];
    out[A3G_STAT_SEEDS] = ctr->ucount[0];
    // misses = U - hits, derived on the host (a3g_trainer_step_stats)
  }
}

struct OuterArgs {
  const float* h1;
  const uint32_t* cnt0;
  const uint32_t* sidx0;
  uint32_t f0;
  const uint32_t* ns;
  const uint32_t* unique;
  const uint32_t* labels;
  const float* w2;
  uint32_t H, C;
  float* agg_outer;
  float* logits;
  float* dlogits;
  float* loss_s;
  float* dagg;     // [cap_seeds x H] per-edge dh1 contribution of seed s
  uint32_t* keys;  // [cap_seeds x (f0 + 1)] dh1 row of each scatter entry (kInv: none)
  uint32_t* vals;  // seed of each scatter entry
  uint32_t cap_seeds;
  int has_layer0;
};

__global__ void __launch_bounds__(256) k_outer(OuterArgs a) {
  const int lane = threadIdx.x & 31;
  const uint32_t ns = *a.ns;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t H = a.H, C = a.C;
  const float inv_ns = 1.f / static_cast<float>(ns);
  for (uint32_t s = gw; s < ns; s += nw) {
    const uint32_t c0 = a.has_layer0 ? a.cnt0[s] : 0u;
    const uint32_t* srcs = a.sidx0 + static_cast<uint64_t>(s) * a.f0;
    float ag = 0.f;
    if (lane < H) {
      if (c0 == 0) {
        ag = a.h1[static_cast<uint64_t>(s) * H + lane];
      } else {
        for (uint32_t t = 0; t < c0; ++t) ag += a.h1[static_cast<uint64_t>(srcs[t]) * H + lane];
        ag *= 1.f / static_cast<float>(c0);
      }
      a.agg_outer[static_cast<uint64_t>(s) * H + lane] = ag;
    }
    // logits (trainer.cpp:129-131)
    float myz = -INFINITY;
    for (uint32_t cc = 0; cc < C; ++cc) {
      float p = lane < H ? ag * a.w2[lane * C + cc] : 0.f;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(kFull, p, off);
      if (lane == static_cast<int>(cc)) myz = p;
    }
    float mx = myz;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, off));
    const float e = lane < static_cast<int>(C) ? expf(myz - mx) : 0.f;
    float den = e;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) den += __shfl_xor_sync(kFull, den, off);
    const uint32_t y = a.labels[a.unique[s]];
    const float zy = __shfl_sync(kFull, myz, y & 31);
    const float d = lane < static_cast<int>(C)
                        ? (e / den - (static_cast<uint32_t>(lane) == y ? 1.f : 0.f)) * inv_ns
                        : 0.f;
    if (lane < static_cast<int>(C)) {
      a.logits[static_cast<uint64_t>(s) * C + lane] = myz;
      a.dlogits[static_cast<uint64_t>(s) * C + lane] = d;
    }
    if (lane == 0) a.loss_s[s] = -(zy - mx - logf(den));
    // dagg_outer = dlogits . W2^T (trainer.cpp:177-179), pre-scaled by the
    // outer mean's 1/deg: the contribution of each of the seed's edges
    float dg = 0.f;
    for (uint32_t cc = 0; cc < C; ++cc) {
      const float dc = __shfl_sync(kFull, d, cc);
      if (lane < H) dg = fmaf(dc, a.w2[lane * C + cc], dg);
    }
    if (lane < H) a.dagg[static_cast<uint64_t>(s) * H + lane] = c0 == 0 ? dg : (1.f / static_cast<float>(c0)) * dg;
    // scatter entries (dh1 row <- seed s), sorted stably by row next: edge
    // entries in edge order, then the self-fallback entry (trainer.cpp:182-198)
    const uint64_t e0 = static_cast<uint64_t>(s) * a.f0;
    for (uint32_t t = lane; t < a.f0; t += 32) {
      a.keys[e0 + t] = t < c0 ? srcs[t] : kInv;
      a.vals[e0 + t] = s;
    }
    if (lane == 0) {
      const uint64_t fb = static_cast<uint64_t>(a.cap_seeds) * a.f0 + s;
      a.keys[fb] = c0 == 0 ? s : kInv;
      a.vals[fb] = s;
    }
  }
  // pad the unused tail of the entry arrays (rows ns .. cap_seeds)
  const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(ns) * a.f0 + gt; i < static_cast<uint64_t>(a.cap_seeds) * a.f0; i += nt)
    a.keys[i] = kInv;
  for (uint64_t i = static_cast<uint64_t>(a.cap_seeds) * a.f0 + ns + gt;
       i < static_cast<uint64_t>(a.cap_seeds) * (a.f0 + 1); i += nt)
    a.keys[i] = kInv;
}

// dh1[r] = sum of the contributions of the sorted entries with key r, in
// order (edges in edge order, then the fallback): deterministic, no atomics.
__global__ void __launch_bounds__(256) k_dh1_gather(const uint32_t* keys, const uint32_t* vals, uint64_t n_entries,
                                                    const float* dagg, uint32_t H, float* dh1) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = gw; i < n_entries; i += nw) {
    const uint32_t r = keys[i];
    if (r == kInv) break;  // sorted: the padding is last
    if (i > 0 && keys[i - 1] == r) continue;  // not the head of its run
    float acc = 0.f;
    for (uint64_t j = i; j < n_entries && keys[j] == r; ++j)
      if (lane < static_cast<int>(H)) acc += dagg[static_cast<uint64_t>(vals[j]) * H + lane];
    if (lane < static_cast<int>(H)) dh1[static_cast<uint64_t>(r) * H + lane] = acc;
  }
}

struct Dw1Args {
  const float* agg_inner;
  const float* h1;
  const float* dh1;
  const uint32_t* n_inner;
  uint32_t pitch, F, H;
  float* part;
};

template <int HT, int NCOL>
__global__ void __launch_bounds__(256) k_dw1_partial(Dw1Args a) {
  __shared__ float s_dh[32][HT];
  const uint32_t n = *a.n_inner;
  const uint32_t per = (n + gridDim.x - 1) / gridDim.x;
  const uint32_t r_beg = blockIdx.x * per, r_end = min(n, r_beg + per);
  float acc[NCOL][HT];
#pragma unroll
  for (int c = 0; c < NCOL; ++c)
#pragma unroll
    for (int j = 0; j < HT; ++j) acc[c][j] = 0.f;
  const uint32_t H = a.H;
  for (uint32_t r0 = r_beg; r0 < r_end; r0 += 32) {
    for (uint32_t i = threadIdx.x; i < 32 * HT; i += blockDim.x) {
      const uint32_t rr = r0 + i / HT, j = i % HT;
      float v = 0.f;
      if (rr < r_end && j < H) {
        const uint64_t o = static_cast<uint64_t>(rr) * H + j;
        v = a.h1[o] > 0.f ? a.dh1[o] : 0.f;  // relu_mask (trainer.cpp:200)
      }
      s_dh[i / HT][j] = v;
    }
    __syncthreads();
    const uint32_t nr = min(32u, r_end - r0);
    for (uint32_t i = 0; i < nr; ++i) {
      const float* arow = a.agg_inner + static_cast<uint64_t>(r0 + i) * a.pitch;
#pragma unroll
      for (int c = 0; c < NCOL; ++c) {
        const uint32_t f = threadIdx.x + 256 * c;
        const float x = f < a.F ? arow[f] : 0.f;
#pragma unroll
        for (int j = 0; j < HT; ++j) acc[c][j] = fmaf(x, s_dh[i][j], acc[c][j]);
      }
    }
    __syncthreads();
  }
  float* out = a.part + static_cast<uint64_t>(blockIdx.x) * a.F * H;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) {
    const uint32_t f = threadIdx.x + 256 * c;
    if (f < a.F)
#pragma unroll
      for (int j = 0; j < HT; ++j)
        if (j < static_cast<int>(H)) out[static_cast<uint64_t>(f) * H + j] = acc[c][j];
  }
}

struct ReduceArgs {
  const float* part;
  uint32_t nparts;
  const float* agg_outer;
  const float* dlogits;
  const float* loss_s;
  const uint32_t* ns;
  uint32_t F, H, C;
  float* gw;  // [F*H | H*C | n | loss_mean*n]
};

__global__ void k_reduce(ReduceArgs a) {
  const uint32_t FH = a.F * a.H, HC = a.H * a.C;
  const uint32_t ns = *a.ns;
  if (blockIdx.x == gridDim.x - 1) {  // mean loss, fixed-order tree
    __shared__ float s_l[256];
    float x = 0.f;
    for (uint32_t s = threadIdx.x; s < ns; s += blockDim.x) x += a.loss_s[s];
    s_l[threadIdx.x] = x;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) s_l[threadIdx.x] += s_l[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      a.gw[FH + HC] = static_cast<float>(ns);
      a.gw[FH + HC + 1] = s_l[0];  // sum of per-seed losses = mean * n
    }
    return;
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < FH + HC;
       i += (gridDim.x - 1) * blockDim.x) {
    float s = 0.f;
    if (i < FH) {
      for (uint32_t p = 0; p < a.nparts; ++p) s += a.part[static_cast<uint64_t>(p) * FH + i];
    } else {
      const uint32_t q = i - FH, j = q / a.C, c = q % a.C;
      for (uint32_t t = 0; t < ns; ++t)
        s = fmaf(a.agg_outer[static_cast<uint64_t>(t) * a.H + j], a.dlogits[static_cast<uint64_t>(t) * a.C + c], s);
    }
    a.gw[i] = s;
  }
}

// grads are local means; with a communicator gw holds n_k-weighted sums and
// sync == true divides by the summed n (trainer.cpp:213-229 generalised to
// unequal shards).
__global__ void k_scale_for_sync(float* gw, uint32_t n_total) {
  const float n = gw[n_total];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_total; i += gridDim.x * blockDim.x)
    gw[i] *= n;
}

__global__ void k_sgd(float* w1, float* w2, float* gw, uint32_t FH, uint32_t HC, float lr, int synced,
                      double* loss_slot) {
  const float n = gw[FH + HC];
  const float inv = synced ? 1.f / n : 1.f;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < FH + HC; i += gridDim.x * blockDim.x) {
    const float g = gw[i] * inv;
    if (synced) gw[i] = g;
    if (i < FH)
      w1[i] -= lr * g;
    else
      w2[i - FH] -= lr * g;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && loss_slot) *loss_slot = static_cast<double>(gw[FH + HC + 1]) / n;
}

template <typename T>
void launch_agg(TrainerState& t, const AggArgs& aa, int nch, cudaStream_t st) {
  const int grid = t.sm_count * 2;
  const size_t smem = t.agg_smem;
#define A3G_AGG_CASE(N)                                                                          \
  case N:                                                                                        \
    A3G_CUDA(cudaFuncSetAttribute(k_agg1<T, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                  static_cast<int>(smem)));                                      \
    k_agg1<T, N><<<grid, kAggThreads, smem, st>>>(aa);                                           \
    break;
  switch (nch) {
    A3G_AGG_CASE(1)
    A3G_AGG_CASE(2)
    A3G_AGG_CASE(3)
    A3G_AGG_CASE(4)
    A3G_AGG_CASE(5)
    A3G_AGG_CASE(6)
    A3G_AGG_CASE(8)
    A3G_AGG_CASE(16)
    default:
      raise(A3G_ERR_PARAMETER, "feature row too wide for k_agg1");
  }
#undef A3G_AGG_CASE
  A3G_LAUNCH_CHECK("k_agg1");
}

template <int HT>
void launch_dw1_h(const Dw1Args& da, int ncol, uint32_t nparts, cudaStream_t st) {
  switch (ncol) {
    case 1: k_dw1_partial<HT, 1><<<nparts, 256, 0, st>>>(da); break;
    case 2: k_dw1_partial<HT, 2><<<nparts, 256, 0, st>>>(da); break;
    case 3: k_dw1_partial<HT, 3><<<nparts, 256, 0, st>>>(da); break;
    case 4: k_dw1_partial<HT, 4><<<nparts, 256, 0, st>>>(da); break;
    case 5: case 6: case 7: case 8: k_dw1_partial<HT, 8><<<nparts, 256, 0, st>>>(da); break;
    default: raise(A3G_ERR_PARAMETER, "feat_dim too large for k_dw1_partial");
  }
  A3G_LAUNCH_CHECK("k_dw1_partial");
}

}  // namespace

// nccl glue lives in comm.cpp
void comm_allreduce_sum(a3g_comm* comm, float* buf, size_t count, cudaStream_t st);

void launch_train_compute(TrainerState& t, a3g_sampler* smp, double lr, double* d_loss_slot,
                          unsigned long long* d_stats, cudaStream_t st, bool record_timing) {
  SamplerState& s = smp->st;
  a3g_graph* g = t.g;
  BatchCounters* ctr = s.d_ctr;
  A3G_CUDA(cudaMemsetAsync(t.d_dh1, 0, t.cap_inner * t.H * sizeof(float), st));
  if (d_stats) {
    const a3g_cache* c = t.c;
    const int bitmode = c->all_cached ? 1 : (c->none_cached ? 0 : 2);
    k_step_stats<<<t.sm_count, 256, 0, st>>>(ctr, s.d_unique, c->d_bits, bitmode, s.L, d_stats);
    A3G_LAUNCH_CHECK("k_step_stats");
  }
  // ---- gather + aggregation + GEMM1 (forward, inner rows)
  AggArgs aa{};
  aa.view = g->view;
  aa.pitch = g->pitch;
  aa.F = t.F;
  aa.H = t.H;
  aa.unique = s.d_unique;
  aa.inv1 = s.d_inv1;
  aa.has_layer1 = s.L >= 2;
  aa.cnt1 = s.L >= 2 ? s.layer[1].cnt : nullptr;
  aa.S1 = s.L >= 2 ? s.layer[1].S : nullptr;
  aa.f1 = s.L >= 2 ? s.layer[1].f : 0;
  aa.n_inner = s.L >= 1 ? &ctr->ucount[1] : &ctr->ucount[0];
  aa.w1 = t.d_w1;
  aa.agg_inner = t.d_agg_inner;
  aa.h1 = t.d_h1;
  aa.bytes = t.d_agg_bytes;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (record_timing) {
    A3G_CUDA(cudaEventCreate(&e0));
    A3G_CUDA(cudaEventCreate(&e1));
    A3G_CUDA(cudaEventRecord(e0, st));
  }
  if (g->feat_dtype == A3G_FEAT_BF16) {
    const int nch = static_cast<int>((g->pitch / 8 + 31) / 32);
    launch_agg<uint16_t>(t, aa, nch == 7 ? 8 : (nch > 8 && nch <= 16 ? 16 : nch), st);
  } else {
    const int nch = static_cast<int>((g->pitch / 4 + 31) / 32);
    launch_agg<float>(t, aa, nch == 7 ? 8 : (nch > 8 && nch <= 16 ? 16 : nch), st);
  }
  if (record_timing) {
    A3G_CUDA(cudaEventRecord(e1, st));
    t.ev_agg.push_back(e0);
    t.ev_agg.push_back(e1);
  }
  // ---- outer aggregation, logits, loss, dlogits, scatter to dh1
  OuterArgs oa{};
  oa.h1 = t.d_h1;
  oa.has_layer0 = s.L >= 1;
  oa.cnt0 = s.L >= 1 ? s.layer[0].cnt : nullptr;
  oa.sidx0 = s.L >= 1 ? s.layer[0].sidx : nullptr;
  oa.f0 = s.L >= 1 ? s.layer[0].f : 0;
  oa.ns = &ctr->ucount[0];
  oa.unique = s.d_unique;
  oa.labels = g->d_labels;
  oa.w2 = t.d_w2;
  oa.H = t.H;
  oa.C = t.C;
  oa.agg_outer = t.d_agg_outer;
  oa.logits = t.d_logits;
  oa.dlogits = t.d_dlogits;
  oa.loss_s = t.d_loss_s;
  oa.dagg = t.d_dagg;
  oa.keys = t.d_keys[0];
  oa.vals = t.d_vals[0];
  oa.cap_seeds = t.max_seeds;
  if (oa.f0 == 0) oa.f0 = 1;  // no layer: fallback entries only (keys of the edge part are all kInv)
  k_outer<<<std::max(1, static_cast<int>((t.max_seeds + 7) / 8)), 256, 0, st>>>(oa);
  A3G_LAUNCH_CHECK("k_outer");
  // ---- deterministic scatter into dh1: stable radix sort of the entries by row
  {
    size_t tmp = t.sort_tmp_bytes;
    A3G_CUDA(cub::DeviceRadixSort::SortPairs(t.d_sort_tmp, tmp, t.d_keys[0], t.d_keys[1], t.d_vals[0], t.d_vals[1],
                                             static_cast<int>(t.n_entries), 0, 32, st));
    k_dh1_gather<<<t.sm_count * 2, 256, 0, st>>>(t.d_keys[1], t.d_vals[1], t.n_entries, t.d_dagg, t.H, t.d_dh1);
    A3G_LAUNCH_CHECK("k_dh1_gather");
  }
  // ---- dW1 partials
  Dw1Args da{};
  da.agg_inner = t.d_agg_inner;
  da.h1 = t.d_h1;
  da.dh1 = t.d_dh1;
  da.n_inner = aa.n_inner;
  da.pitch = g->pitch;
  da.F = t.F;
  da.H = t.H;
  da.part = t.d_part;
  const int ncol = static_cast<int>((t.F + 255) / 256);
  if (t.H <= 16)
    launch_dw1_h<16>(da, ncol, t.nparts, st);
  else
    launch_dw1_h<32>(da, ncol, t.nparts, st);
  // ---- reduce -> grads, loss
  ReduceArgs ra{};
  ra.part = t.d_part;
  ra.nparts = t.nparts;
  ra.agg_outer = t.d_agg_outer;
  ra.dlogits = t.d_dlogits;
  ra.loss_s = t.d_loss_s;
  ra.ns = &ctr->ucount[0];
  ra.F = t.F;
  ra.H = t.H;
  ra.C = t.C;
  ra.gw = t.d_gw;
  const uint32_t FH = t.F * t.H, HC = t.H * t.C;
  const int rgrid = static_cast<int>(std::min<uint32_t>(t.sm_count, (FH + HC + 255) / 256)) + 1;
  k_reduce<<<rgrid, 256, 0, st>>>(ra);
  A3G_LAUNCH_CHECK("k_reduce");
  const bool synced = t.comm != nullptr;
  if (synced) {
    k_scale_for_sync<<<t.sm_count, 256, 0, st>>>(t.d_gw, FH + HC);
    A3G_LAUNCH_CHECK("k_scale_for_sync");
    comm_allreduce_sum(t.comm, t.d_gw, FH + HC + 2, st);
  }
  k_sgd<<<t.sm_count, 256, 0, st>>>(t.d_w1, t.d_w2, t.d_gw, FH, HC, static_cast<float>(lr), synced ? 1 : 0,
                                    d_loss_slot);
  A3G_LAUNCH_CHECK("k_sgd");
}

}  // namespace a3g

namespace a3g {
size_t dh1_sort_temp_bytes(uint64_t n_entries) {
  size_t bytes = 0;
  A3G_CUDA(cub::DeviceRadixSort::SortPairs(static_cast<void*>(nullptr), bytes, static_cast<const uint32_t*>(nullptr),
                                           static_cast<uint32_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                           static_cast<uint32_t*>(nullptr), static_cast<int>(n_entries), 0, 32));
  return bytes;
}
}  // namespace a3g
