// train.cu -- one training step of the reference's 2-layer mean-GCN
// (proj/src/trainer.cpp:59-211) on sm_100a, after the sampler:
//
//   k_step_stats  batch sizes + cache hit/miss count over unique_nodes.
//   k_agg1        inner rows: gather the layer-1 source rows through the
//                 feature store (128-bit loads, several rows in flight), mean
//                 (self-fallback when empty, trainer.cpp:93-107) -> agg_inner.
//                 THE roofline kernel (HBM-bound).
//   k_h1_tc       h1 = ReLU(agg_inner . W1) on tcgen05 (gemm_tc.cu).
//   k_outer       per seed: agg_outer (trainer.cpp:116-127), logits,
//                 softmax-CE + dlogits (:153-171), dagg_outer = dlogits . W2^T
//                 (:177-179) pre-scaled by 1/deg, and the scatter entries.
//   k_dh1_scatter dh1 = the outer aggregation's scatter (:182-198) as 64-bit
//                 fixed-point integer atomics (order-independent: deterministic).
//   k_dw1_tc      dW1 = agg_inner^T . (dh1 * [h1>0]) on tcgen05 (:200-204).
//   k_reduce      fixed-order reduction of the dW1 partials, dW2 (:174-175),
//                 mean loss.
//   k_sgd         w -= lr * g (trainer.cpp:208-211).
#include <cmath>
#include <cstdlib>

#include "ptx.cuh"
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
  const uint32_t* n_distinct;  // distinct layer-1 sources (nfront[2]), or null
  float* agg_inner;
  unsigned long long* bytes;
  int has_layer1;
  const float* w1;  // [F][H] (fused h1 epilogue, HB > 0)
  float* h1;        // [n_inner][H] relu(agg_inner . W1)
};

// Gather + mean of the layer-1 source rows of every inner row (trainer.cpp:
// 93-107). Each warp streams its source rows through a ring of S row
// buffers in shared memory with cp.async (LDGSTS): every lane copies its own
// 16-byte chunks of a row (chunk q = lane + 32 i) and later sums exactly those
// chunks, so the pipeline needs no barriers -- per-lane cp.async groups, one
// per source row, with S - 1 rows in flight behind the one being summed,
// across row boundaries. No registers are held by in-flight loads: 24 warps
// x 3 rows (~175 KB for 2.4 KB rows) are in flight per SM, and the
// random-row gather runs at HBM (or NVLink / PCIe, store.cu) bandwidth
// rather than load latency. Sum in edge order, then x (1/c): the reference's
// scale(1.0/deg) (trainer.cpp:41-54).
__device__ __forceinline__ void ldgsts16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void ldgsts_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ldgsts_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// h1 = relu(x . W1) for NR finished inner rows at once (x pre-scaled, the
// lane's chunks): one pass over the lane's W1 words serves all NR rows, so
// the shared-memory W1 traffic per row is 1/NR. Group g owns outputs
// [g HG, (g+1) HG); per-lane partials, then a recursive-halving reduce over
// the group's lanes (fixed order).
template <int NCH, int EPC, int LPR, int HG, int NR>
__device__ __forceinline__ void h1_rows(const float (&x)[NR][NCH][EPC], const uint32_t (&rows)[NR],
                                        const float* w1s, uint32_t chunks, uint32_t g, uint32_t gl, uint32_t H,
                                        float* h1) {
  float p[NR][HG];
#pragma unroll
  for (int r = 0; r < NR; ++r)
#pragma unroll
    for (int h = 0; h < HG; ++h) p[r][h] = 0.f;
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const uint32_t q = gl + LPR * i;
    if (q < chunks) {
#pragma unroll
      for (int e = 0; e < EPC; ++e) {
#pragma unroll
        for (int h4 = 0; h4 < HG / 4; ++h4) {
          const float4 w = reinterpret_cast<const float4*>(w1s)[((g * (HG / 4) + h4) * EPC + e) * chunks + q];
#pragma unroll
          for (int r = 0; r < NR; ++r) {
            p[r][4 * h4] = fmaf(x[r][i][e], w.x, p[r][4 * h4]);
            p[r][4 * h4 + 1] = fmaf(x[r][i][e], w.y, p[r][4 * h4 + 1]);
            p[r][4 * h4 + 2] = fmaf(x[r][i][e], w.z, p[r][4 * h4 + 2]);
            p[r][4 * h4 + 3] = fmaf(x[r][i][e], w.w, p[r][4 * h4 + 3]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    uint32_t hidx = 0;
    int o = LPR / 2;
#pragma unroll
    for (int n = HG; n > 1; n >>= 1, o >>= 1) {
      const bool upper = (gl & static_cast<uint32_t>(o)) != 0;
#pragma unroll
      for (int j = 0; j < n / 2; ++j) {
        const float send = upper ? p[r][j] : p[r][j + n / 2];
        const float keep = upper ? p[r][j + n / 2] : p[r][j];
        p[r][j] = keep + __shfl_xor_sync(kFull, send, o);
      }
      if (upper) hidx += n / 2;
    }
    for (; o > 0; o >>= 1) p[r][0] += __shfl_xor_sync(kFull, p[r][0], o);
    const uint32_t h = g * HG + hidx;
    if ((gl & static_cast<uint32_t>(LPR / HG - 1)) == 0 && h < H)
      h1[static_cast<uint64_t>(rows[r]) * H + h] = fmaxf(p[r][0], 0.f);
  }
}

// PAIR (with HB > 0): the h1 epilogue waits for the warp's next finished row
// and serves both from one pass over W1 (half the shared-memory W1 reads).
template <typename T, int NCH, int WARPS, int S, int LPR, int HB, bool PAIR = false>
__global__ void __launch_bounds__(WARPS * 32, 1) k_agg1(const __grid_constant__ AggArgs a) {
  // LPR lanes per source row: short rows (<= 16 chunks) are copied RPI at a
  // time by lane groups; each group sums its own rows, the groups' partial
  // sums are added at the end of an inner row (fixed order: deterministic)
  using Ch = Chunk<T>;
  constexpr int EPC = Ch::EPC;
  constexpr int RPI = 32 / LPR;
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t g = lane / LPR, gl = lane % LPR;
  const uint32_t rb = a.view.row_bytes;
  const uint32_t ring = ptx::smem_u32(smem) + static_cast<uint32_t>(warp) * S * RPI * rb;
  const uint8_t* ring_p = smem + static_cast<size_t>(warp) * S * RPI * rb;
  const uint32_t n_inner = *a.n_inner;
  const uint32_t chunks = a.pitch / EPC;  // 16-byte chunks per row
  const uint32_t gw = blockIdx.x * WARPS + warp, nw = gridDim.x * WARPS;
  // fused h1 epilogue (HB > 0): W1 zero-padded after the rings, laid out
  // [h/4][e][q][h%4] (feature f = q EPC + e of chunk q) so that the lanes of
  // a group, reading consecutive chunks q, hit consecutive 16-byte words
  float* w1s = reinterpret_cast<float*>(smem + static_cast<size_t>(WARPS) * S * RPI * rb);
  if constexpr (HB > 0) {
    for (uint32_t i = threadIdx.x; i < chunks * EPC * HB; i += WARPS * 32) {
      const uint32_t j = i & 3, q = (i >> 2) % chunks, e = (i >> 2) / chunks % EPC, h = (i >> 2) / chunks / EPC * 4 + j;
      const uint32_t f = q * EPC + e;
      w1s[i] = (f < a.F && h < a.H) ? __ldg(a.w1 + static_cast<size_t>(f) * a.H + h) : 0.f;
    }
    __syncthreads();
  }
  const uint32_t nrows = gw < n_inner ? (n_inner - gw + nw - 1) / nw : 0;  // this warp's rows gw + j*nw
  unsigned long long nbytes = 0;
  // producer: row j, source t; lanes hold the (layer row, count) of rows
  // 32*batch + lane and the current row's source ids; lane s holds the
  // (row, count|last, groups) record of ring slot s for the consumer
  uint32_t pj = 0, pt = 0, pc = 0, batch = ~0u, src_lane = 0;
  int32_t meta_k = -1, pk = -1;
  uint32_t meta_c = 0;
  bool row_ready = false;
  uint32_t slot_row = 0, slot_c = 0, slot_n = 0;
  uint32_t issued = 0, consumed = 0;
  float acc[NCH][EPC];
#pragma unroll
  for (int i = 0; i < NCH; ++i)
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[i][e] = 0.f;
  constexpr int HG = HB > 0 ? HB / RPI : 4;
  float prev[PAIR ? 1 : 1][NCH][EPC];  // PAIR: the finished row awaiting its partner
  uint32_t prev_row[1] = {0};
  bool have_prev = false;
  for (;;) {
    // ---- producer: fill the ring
    while (issued - consumed < S && pj < nrows) {
      const uint32_t r = gw + pj * nw;
      if (!row_ready) {
        if ((pj >> 5) != batch) {
          batch = pj >> 5;
          const uint32_t rr = gw + (batch * 32 + lane) * nw;
          meta_k = -1;
          meta_c = 0;
          if (batch * 32 + lane < nrows && a.has_layer1) {
            meta_k = __ldg(a.inv1 + rr);
            meta_c = meta_k >= 0 ? __ldg(a.cnt1 + meta_k) : 0u;
          }
        }
        pk = __shfl_sync(kFull, meta_k, pj & 31);
        pc = __shfl_sync(kFull, meta_c, pj & 31);
        src_lane = lane < static_cast<int>(pc) ? __ldg(a.S1 + static_cast<uint64_t>(pk) * a.f1 + lane) : 0u;
        nbytes += pc ? static_cast<unsigned long long>(pc) * 4 + 8 : static_cast<unsigned long long>(a.F) * sizeof(T) + 4;
        row_ready = true;
      }
      const uint32_t total = pc ? pc : 1u;           // sources of this row (fallback: own row)
      const uint32_t ngrp = min(static_cast<uint32_t>(RPI), total - pt);
      const uint32_t t = pt + g;
      uint32_t v = __shfl_sync(kFull, src_lane, t & 31);
      if (pc == 0) v = __ldg(a.unique + r);  // self-fallback: own features (trainer.cpp:102-107)
      else if (t >= 32 && t < pc) v = __ldg(a.S1 + static_cast<uint64_t>(pk) * a.f1 + t);  // fanout > 32
      const uint32_t slot = issued % S;
      const bool last = pt + ngrp >= total;
      if (g < ngrp) {
        const uint8_t* src = row_ptr(a.view, v);
        const uint32_t dst = ring + (slot * RPI + g) * rb;
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
          const uint32_t q = gl + LPR * i;
          if (q < chunks) ldgsts16(dst + q * 16, src + q * 16);
        }
      }
      ldgsts_commit();
      if (lane == static_cast<int>(slot)) {
        slot_row = r;
        slot_c = pc | (last ? 0x80000000u : 0u);
        slot_n = ngrp;
      }
      ++issued;
      if (last) {
        ++pj;
        pt = 0;
        row_ready = false;
      } else {
        pt += ngrp;
      }
    }
    if (consumed == issued) break;
    // ---- consumer: the oldest slot (this lane's chunks of its group's row)
    if (issued - consumed == S)
      ldgsts_wait<S - 1>();
    else
      ldgsts_wait<0>();
    const uint32_t slot = consumed % S;
    const uint32_t sn = __shfl_sync(kFull, slot_n, slot);
    if (g < sn) {
      const uint4* row = reinterpret_cast<const uint4*>(ring_p + static_cast<size_t>(slot * RPI + g) * rb);
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const uint32_t q = gl + LPR * i;
        if (q < chunks) Ch::add(acc[i], row[q]);
      }
    }
    const uint32_t srow = __shfl_sync(kFull, slot_row, slot);
    const uint32_t sc = __shfl_sync(kFull, slot_c, slot);
    ++consumed;
    if (sc & 0x80000000u) {
      if (RPI > 1) {
#pragma unroll
        for (int off = LPR; off < 32; off <<= 1)
#pragma unroll
          for (int i = 0; i < NCH; ++i)
#pragma unroll
            for (int e = 0; e < EPC; ++e) acc[i][e] += __shfl_xor_sync(kFull, acc[i][e], off);
      }
      const uint32_t c = sc & 0x7fffffffu;
      const float scale = c ? 1.f / static_cast<float>(c) : 1.f;
      float4* out = reinterpret_cast<float4*>(a.agg_inner + static_cast<uint64_t>(srow) * a.pitch);
      if constexpr (HB > 0) {
        if constexpr (PAIR) {
          if (!have_prev) {
#pragma unroll
            for (int i = 0; i < NCH; ++i)
#pragma unroll
              for (int e = 0; e < EPC; ++e) prev[0][i][e] = acc[i][e] * scale;
            prev_row[0] = srow;
            have_prev = true;
          } else {
            float xx[2][NCH][EPC];
#pragma unroll
            for (int i = 0; i < NCH; ++i)
#pragma unroll
              for (int e = 0; e < EPC; ++e) {
                xx[0][i][e] = prev[0][i][e];
                xx[1][i][e] = acc[i][e] * scale;
              }
            const uint32_t rr[2] = {prev_row[0], srow};
            h1_rows<NCH, EPC, LPR, HG, 2>(xx, rr, w1s, chunks, g, gl, a.H, a.h1);
            have_prev = false;
          }
        } else {
          float xx[1][NCH][EPC];
#pragma unroll
          for (int i = 0; i < NCH; ++i)
#pragma unroll
            for (int e = 0; e < EPC; ++e) xx[0][i][e] = acc[i][e] * scale;
          const uint32_t rr[1] = {srow};
          h1_rows<NCH, EPC, LPR, HG, 1>(xx, rr, w1s, chunks, g, gl, a.H, a.h1);
        }
      }
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const uint32_t q = gl + LPR * i;
        if (g == 0 && q < chunks) {
#pragma unroll
          for (int e = 0; e < EPC; e += 4)
            out[q * (EPC / 4) + e / 4] = make_float4(acc[i][e] * scale, acc[i][e + 1] * scale,
                                                     acc[i][e + 2] * scale, acc[i][e + 3] * scale);
        }
#pragma unroll
        for (int e = 0; e < EPC; ++e) acc[i][e] = 0.f;
      }
      nbytes += static_cast<unsigned long long>(a.F) * 4 + (HB > 0 ? a.H * 4ull : 0ull);  // agg_inner (+h1) row
    }
  }
  if constexpr (HB > 0 && PAIR) {
    if (have_prev) h1_rows<NCH, EPC, LPR, HG, 1>(prev, prev_row, w1s, chunks, g, gl, a.H, a.h1);
  }
  // algorithmic feature bytes: every DISTINCT layer-1 source row once -- the
  // layer-2 frontier is exactly the first-seen set of layer-1 sources
  // (sampler.cpp:128-131); duplicates are re-reads the caches may absorb
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.n_distinct)
    nbytes += *a.n_distinct * static_cast<unsigned long long>(a.F) * sizeof(T);
  if (lane == 0 && nbytes) atomicAdd(a.bytes, nbytes);
}

// Long rows (one row per warp step, LPR 32): the same gather + mean + fused
// h1 epilogue with each source row moved by ONE TMA bulk copy
// (cp.async.bulk, completion on the slot's mbarrier) that lane 0 issues,
// instead of per-lane 16-byte LDGSTS with their per-chunk address and
// predicate work. The slot's (row, count|last) record travels through shared
// memory beside it (written before the arrive, read after the wait), so the
// per-source-row work is one shuffle + one bulk issue on the producer side and
// one barrier poll + the lane's chunk sums on the consumer side. The warp's
// __syncwarp before each refill orders every lane's reads of the slots being
// reused before lane 0's next copy into them (consumer release).
// source id of a layer-1 slot beyond the first 32 (out of line: rare)
__device__ __noinline__ uint32_t agg_src_far(const uint32_t* S1, int32_t pk, uint32_t f1, uint32_t t) {
  return __ldg(S1 + static_cast<uint64_t>(pk) * f1 + t);
}

template <typename T, int NCH, int WARPS, int S, int HB, bool PAIR, bool IDENT>
__global__ void __launch_bounds__(WARPS * 32, 1) k_agg1_tma(const __grid_constant__ AggArgs a) {
  static_assert((S & (S - 1)) == 0, "ring depth must be a power of two");
  using Ch = Chunk<T>;
  constexpr int EPC = Ch::EPC;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[WARPS * S];
  __shared__ uint2 smeta[WARPS * S];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t rb = a.view.row_bytes;  // == chunks * 16
  const uint32_t n_inner = *a.n_inner;
  const uint32_t chunks = a.pitch / EPC;
  const uint32_t gw = blockIdx.x * WARPS + warp, nw = gridDim.x * WARPS;
  float* w1s = reinterpret_cast<float*>(smem + static_cast<size_t>(WARPS) * S * rb);
  for (int i = threadIdx.x; i < WARPS * S; i += WARPS * 32) ptx::mbar_init(&bars[i], 1);
  ptx::fence_mbar_init();
  if constexpr (HB > 0) {
    // W1 [F][H] -> [h/4][e][q][h%4] (feature f = q EPC + e), zero padded to
    // the pitch and to HB outputs; source order (f, h): no divisions
    for (uint32_t i = threadIdx.x; i < a.pitch * HB; i += WARPS * 32) {
      const uint32_t f = i / HB, h = i % HB, q = f / EPC, e = f % EPC;
      w1s[(((h >> 2) * EPC + e) * chunks + q) * 4 + (h & 3)] =
          (f < a.F && h < a.H) ? __ldg(a.w1 + static_cast<size_t>(f) * a.H + h) : 0.f;
    }
  }
  __syncthreads();
  // the warp's ring, barriers and slot records as shared-window addresses
  const uint32_t ring_s = ptx::smem_u32(smem) + static_cast<uint32_t>(warp) * S * rb;
  const uint32_t bar_s = ptx::smem_u32(bars) + static_cast<uint32_t>(warp) * S * 8;
  const uint32_t meta_s = ptx::smem_u32(smeta) + static_cast<uint32_t>(warp) * S * 8;
  const uint32_t lane_s = ring_s + static_cast<uint32_t>(lane) * 16;  // this lane's chunk q = lane of slot 0
  const uint32_t nrows = gw < n_inner ? (n_inner - gw + nw - 1) / nw : 0;
  const uint8_t* base0 = a.view.base[0];
  unsigned long long nbytes = 0;
  uint32_t pj = 0, pt = 0, pc = 0, batch = ~0u, src_lane = 0, r = 0;
  int32_t meta_k = -1, pk = -1;
  uint32_t meta_c = 0;
  bool row_ready = false;
  uint32_t issued = 0, consumed = 0;
  float acc[NCH][EPC];
#pragma unroll
  for (int i = 0; i < NCH; ++i)
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[i][e] = 0.f;
  constexpr int HG = HB > 0 ? HB : 4;
  float prev[1][NCH][EPC];
  uint32_t prev_row[1] = {0};
  bool have_prev = false;
  for (;;) {
    __syncwarp();  // consumer release of the slots refilled below
    while (issued - consumed < S && pj < nrows) {
      if (!row_ready) {
        r = gw + pj * nw;
        if ((pj >> 5) != batch) {
          batch = pj >> 5;
          const uint32_t rr = gw + (batch * 32 + lane) * nw;
          meta_k = -1;
          meta_c = 0;
          if (batch * 32 + lane < nrows && a.has_layer1) {
            meta_k = __ldg(a.inv1 + rr);
            meta_c = meta_k >= 0 ? __ldg(a.cnt1 + meta_k) : 0u;
          }
        }
        pk = __shfl_sync(kFull, meta_k, pj & 31);
        pc = __shfl_sync(kFull, meta_c, pj & 31);
        src_lane = lane < static_cast<int>(pc) ? __ldg(a.S1 + static_cast<uint64_t>(pk) * a.f1 + lane) : 0u;
        if (pc == 0) src_lane = __ldg(a.unique + r);  // self-fallback: own features (trainer.cpp:102-107)
        nbytes += pc ? static_cast<unsigned long long>(pc) * 4 + 8 : static_cast<unsigned long long>(a.F) * sizeof(T) + 4;
        row_ready = true;
      }
      uint32_t v = __shfl_sync(kFull, src_lane, pt & 31);
      if (pt >= 32) [[unlikely]]
        v = agg_src_far(a.S1, pk, a.f1, pt);  // fanout > 32
      const bool last = pt + 1 >= (pc ? pc : 1u);
      if (lane == 0) {
        const uint32_t slot = issued & (S - 1);
        ptx::sts_v2(meta_s + slot * 8, r, pc | (last ? 0x80000000u : 0u));
        const uint8_t* src = IDENT ? base0 + static_cast<uint64_t>(v) * rb : row_ptr(a.view, v);
        ptx::mbar_arrive_expect_tx_s(bar_s + slot * 8, rb);
        ptx::bulk_g2s_s(ring_s + slot * rb, src, rb, bar_s + slot * 8);
      }
      ++issued;
      if (last) {
        ++pj;
        pt = 0;
        row_ready = false;
      } else {
        ++pt;
      }
    }
    if (consumed == issued) break;
    const uint32_t slot = consumed & (S - 1);
    ptx::mbar_wait_s(bar_s + slot * 8, (consumed / S) & 1u);
    const uint2 md = ptx::lds_v2(meta_s + slot * 8);
    const uint32_t row_s = lane_s + slot * rb;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const uint32_t q = lane + 32 * i;
      if (q < chunks) Ch::add(acc[i], ptx::lds_v4(row_s + 512 * i));
    }
    ++consumed;
    if (md.y & 0x80000000u) {
      const uint32_t srow = md.x, c = md.y & 0x7fffffffu;
      const float scale = c ? 1.f / static_cast<float>(c) : 1.f;
      float4* out = reinterpret_cast<float4*>(a.agg_inner + static_cast<uint64_t>(srow) * a.pitch);
      if constexpr (HB > 0) {
        if constexpr (PAIR) {
          if (!have_prev) {
#pragma unroll
            for (int i = 0; i < NCH; ++i)
#pragma unroll
              for (int e = 0; e < EPC; ++e) prev[0][i][e] = acc[i][e] * scale;
            prev_row[0] = srow;
            have_prev = true;
          } else {
            float xx[2][NCH][EPC];
#pragma unroll
            for (int i = 0; i < NCH; ++i)
#pragma unroll
              for (int e = 0; e < EPC; ++e) {
                xx[0][i][e] = prev[0][i][e];
                xx[1][i][e] = acc[i][e] * scale;
              }
            const uint32_t rr[2] = {prev_row[0], srow};
            // two passes of HG/2 outputs: half the partial sums live at once (no
            // spills, fewer rematerialised addresses; the butterfly order per output
            // is unchanged, so h1 is bit-identical): k_agg1 alone 0.595 -> 0.617
            h1_rows<NCH, EPC, 32, HG / 2, 2>(xx, rr, w1s, chunks, 0, lane, a.H, a.h1);
            h1_rows<NCH, EPC, 32, HG / 2, 2>(xx, rr, w1s, chunks, 1, lane, a.H, a.h1);
            have_prev = false;
          }
        } else {
          float xx[1][NCH][EPC];
#pragma unroll
          for (int i = 0; i < NCH; ++i)
#pragma unroll
            for (int e = 0; e < EPC; ++e) xx[0][i][e] = acc[i][e] * scale;
          const uint32_t rr[1] = {srow};
          h1_rows<NCH, EPC, 32, HG, 1>(xx, rr, w1s, chunks, 0, lane, a.H, a.h1);
        }
      }
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        const uint32_t q = lane + 32 * i;
        if (q < chunks) {
#pragma unroll
          for (int e = 0; e < EPC; e += 4)
            out[q * (EPC / 4) + e / 4] = make_float4(acc[i][e] * scale, acc[i][e + 1] * scale,
                                                     acc[i][e + 2] * scale, acc[i][e + 3] * scale);
        }
#pragma unroll
        for (int e = 0; e < EPC; ++e) acc[i][e] = 0.f;
      }
      nbytes += static_cast<unsigned long long>(a.F) * 4 + (HB > 0 ? a.H * 4ull : 0ull);  // agg_inner (+h1) row
    }
  }
  if constexpr (HB > 0 && PAIR) {
    if (have_prev) h1_rows<NCH, EPC, 32, HG, 1>(prev, prev_row, w1s, chunks, 0, lane, a.H, a.h1);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.n_distinct)
    nbytes += *a.n_distinct * static_cast<unsigned long long>(a.F) * sizeof(T);
  if (lane == 0 && nbytes) atomicAdd(a.bytes, nbytes);
}

// dW1 = agg_inner^T . G, G = dh1 * [h1 > 0] (trainer.cpp:203-204), on the
// CUDA cores: an HBM-bound skinny product (N = H <= 32) -- one pass over
// agg_inner at full bandwidth beats staging 3-term bf16 operands for tcgen05
// (the k_dw1_tc path, A3G_TC_GEMMS=1). CTA = 128 features x kDw1Rows rows:
// the agg tile streams through a cp.async ring of kDw1Stages x kDw1Stage rows
// (no registers held by loads in flight), thread = one feature column with
// HB accumulators, the CTA's G rows staged once in shared memory. Rows are
// summed in order and the splits reduced in order by k_reduce
// (deterministic); empty splits write zero partials.
constexpr uint32_t kDw1Rows = 128;
constexpr uint32_t kDw1Stage = 16;
constexpr uint32_t kDw1Stages = 4;

size_t dw1_smem(int HB) { return (kDw1Stages * kDw1Stage * 128 + kDw1Rows * HB) * sizeof(float); }

template <int HB>
__global__ void __launch_bounds__(128) k_dw1_fma(const float* __restrict__ agg, uint32_t pitch, uint32_t F, uint32_t H,
                                                 const uint32_t* n_inner, const float* __restrict__ h1,
                                                 const float* __restrict__ dh1, float* part) {
  extern __shared__ __align__(16) float dsm[];
  float* ring = dsm;                                     // [stages][kDw1Stage][128]
  float* sg = dsm + kDw1Stages * kDw1Stage * 128;        // [kDw1Rows][HB]
  const uint32_t n = *n_inner;
  const uint32_t r0 = blockIdx.y * kDw1Rows;
  const uint32_t nr = r0 < n ? min(kDw1Rows, n - r0) : 0u;
  const uint32_t f0 = blockIdx.x * 128;
  const uint32_t nst = (nr + kDw1Stage - 1) / kDw1Stage;
  // stage s: rows [s kDw1Stage, +kDw1Stage) x 32 chunks of 16 B, 4 per thread
  auto issue = [&](uint32_t st) {
    if (st < nst) {
      const uint32_t base = ptx::smem_u32(ring + (st % kDw1Stages) * kDw1Stage * 128);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t idx = threadIdx.x + 128 * k, rr = idx >> 5, c = idx & 31;
        const uint32_t r = st * kDw1Stage + rr;
        if (r < nr && f0 + 4 * c < pitch)
          ldgsts16(base + (rr * 128 + 4 * c) * 4, agg + static_cast<uint64_t>(r0 + r) * pitch + f0 + 4 * c);
      }
    }
    ldgsts_commit();
  };
#pragma unroll
  for (uint32_t st = 0; st < kDw1Stages - 1; ++st) issue(st);
  {
    // G tile: every load issued before any is used (a serial loop here would
    // pay one memory latency per element)
    constexpr int PER = kDw1Rows * HB / 128;
    float gh[PER], gd[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint32_t i = threadIdx.x + 128 * k, r = i / HB, h = i % HB;
      gh[k] = 0.f;
      gd[k] = 0.f;
      if (r < nr && h < H) {
        const uint64_t q = static_cast<uint64_t>(r0 + r) * H + h;
        gh[k] = __ldg(h1 + q);
        gd[k] = __ldg(dh1 + q);
      }
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) sg[threadIdx.x + 128 * k] = gh[k] > 0.f ? gd[k] : 0.f;
  }
  float acc[HB];
#pragma unroll
  for (int h = 0; h < HB; ++h) acc[h] = 0.f;
  for (uint32_t st = 0; st < nst; ++st) {
    ldgsts_wait<kDw1Stages - 2>();
    __syncthreads();
    const float* tile = ring + (st % kDw1Stages) * kDw1Stage * 128;
    const uint32_t rows = min(kDw1Stage, nr - st * kDw1Stage);
#pragma unroll 4
    for (uint32_t rr = 0; rr < rows; ++rr) {
      const float x = tile[rr * 128 + threadIdx.x];
      const float4* gr = reinterpret_cast<const float4*>(sg + (st * kDw1Stage + rr) * HB);
#pragma unroll
      for (int h4 = 0; h4 < HB / 4; ++h4) {
        const float4 gv = gr[h4];
        acc[4 * h4] = fmaf(x, gv.x, acc[4 * h4]);
        acc[4 * h4 + 1] = fmaf(x, gv.y, acc[4 * h4 + 1]);
        acc[4 * h4 + 2] = fmaf(x, gv.z, acc[4 * h4 + 2]);
        acc[4 * h4 + 3] = fmaf(x, gv.w, acc[4 * h4 + 3]);
      }
    }
    __syncthreads();  // the slot is refilled next
    issue(st + kDw1Stages - 1);
  }
  const uint32_t f = f0 + threadIdx.x;
  if (f < F) {
    float* out = part + static_cast<uint64_t>(blockIdx.y) * F * H + static_cast<uint64_t>(f) * H;
#pragma unroll
    for (int h = 0; h < HB; ++h)
      if (static_cast<uint32_t>(h) < H) out[h] = acc[h];
  }
}

// Per-step statistics (a3g_trainer_step_stats): batch sizes from the sampler's
// counters and the cache hit/miss count over unique_nodes (lookup,
// cache.cpp:48-68: any-device presence is a hit).
__global__ void k_step_stats(const BatchCounters* ctr, const uint32_t* unique, const uint32_t* bits, int bitmode,
                             uint32_t L, unsigned long long* out, unsigned long long* err) {
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
    out[A3G_STAT_BAD_SEEDS] = ctr->bad_seeds;
    out[A3G_STAT_POSITIONS] = ctr->positions;
    if (ctr->bad_seeds && err) atomicOr(err, 1ull);
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
  uint32_t* amax;  // max |dagg| (float bits), the fixed-point scale of the dh1 scatter
  int has_layer0;
};

// One warp per seed; lane l owns hidden units l, l + 32, ... (H <= 32 * kOuterHB:
// 1 unit per lane up to H = 32, 8 up to H = 256).
template <int kOuterHB>
__global__ void __launch_bounds__(256) k_outer(OuterArgs a) {
  const int lane = threadIdx.x & 31;
  const uint32_t ns = *a.ns;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t H = a.H, C = a.C;
  const uint32_t nh = (H + 31) / 32;  // hidden units per lane in use
  const float inv_ns = 1.f / static_cast<float>(ns);
  for (uint32_t s = gw; s < ns; s += nw) {
    const uint32_t c0 = a.has_layer0 ? a.cnt0[s] : 0u;
    const uint32_t* srcs = a.sidx0 + static_cast<uint64_t>(s) * a.f0;
    // outer mean of h1 over the seed's layer-0 sources, or its own row
    // (trainer.cpp:115-127): sum in edge order, then x (1/deg)
    float ag[kOuterHB];
#pragma unroll
    for (int k = 0; k < kOuterHB; ++k) ag[k] = 0.f;
    if (c0 == 0) {
#pragma unroll
      for (int k = 0; k < kOuterHB; ++k) {
        const uint32_t h = lane + 32 * k;
        if (static_cast<uint32_t>(k) < nh && h < H) ag[k] = a.h1[static_cast<uint64_t>(s) * H + h];
      }
    } else {
      for (uint32_t t = 0; t < c0; ++t) {
        const float* row = a.h1 + static_cast<uint64_t>(srcs[t]) * H;
#pragma unroll
        for (int k = 0; k < kOuterHB; ++k) {
          const uint32_t h = lane + 32 * k;
          if (static_cast<uint32_t>(k) < nh && h < H) ag[k] += row[h];
        }
      }
      const float inv = 1.f / static_cast<float>(c0);
#pragma unroll
      for (int k = 0; k < kOuterHB; ++k) ag[k] *= inv;
    }
#pragma unroll
    for (int k = 0; k < kOuterHB; ++k) {
      const uint32_t h = lane + 32 * k;
      if (static_cast<uint32_t>(k) < nh && h < H) a.agg_outer[static_cast<uint64_t>(s) * H + h] = ag[k];
    }
    // logits (trainer.cpp:129-131)
    float myz = -INFINITY;
    for (uint32_t cc = 0; cc < C; ++cc) {
      float p = 0.f;
#pragma unroll
      for (int k = 0; k < kOuterHB; ++k) {
        const uint32_t h = lane + 32 * k;
        if (static_cast<uint32_t>(k) < nh && h < H) p = fmaf(ag[k], a.w2[h * C + cc], p);
      }
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
    float dg[kOuterHB];
#pragma unroll
    for (int k = 0; k < kOuterHB; ++k) dg[k] = 0.f;
    for (uint32_t cc = 0; cc < C; ++cc) {
      const float dc = __shfl_sync(kFull, d, cc);
#pragma unroll
      for (int k = 0; k < kOuterHB; ++k) {
        const uint32_t h = lane + 32 * k;
        if (static_cast<uint32_t>(k) < nh && h < H) dg[k] = fmaf(dc, a.w2[h * C + cc], dg[k]);
      }
    }
    float amax = 0.f;
#pragma unroll
    for (int k = 0; k < kOuterHB; ++k) {
      const uint32_t h = lane + 32 * k;
      if (static_cast<uint32_t>(k) < nh && h < H) {
        const float v = c0 == 0 ? dg[k] : (1.f / static_cast<float>(c0)) * dg[k];
        a.dagg[static_cast<uint64_t>(s) * H + h] = v;
        amax = fmaxf(amax, fabsf(v));
      }
    }
    amax = fmaxf(amax, __shfl_xor_sync(kFull, amax, 16));
    amax = fmaxf(amax, __shfl_xor_sync(kFull, amax, 8));
    amax = fmaxf(amax, __shfl_xor_sync(kFull, amax, 4));
    amax = fmaxf(amax, __shfl_xor_sync(kFull, amax, 2));
    amax = fmaxf(amax, __shfl_xor_sync(kFull, amax, 1));
    if (lane == 0) atomicMax(a.amax, __float_as_uint(amax));  // non-negative floats order like their bits
  }
}

// Fixed-point scale of the dh1 scatter: the step has at most ns * max(f0, 1)
// contributions in total (one per layer-0 slot, or one self-fallback per
// seed) -- a row can receive all of them when duplicate CSR edges
// (from_edges / A3G1 accept them) make one source fill every slot -- each
// bounded by amax, so no row sum reaches 2^62.
__device__ __forceinline__ double fx_scale(uint32_t amax_bits, uint32_t ns, uint32_t f0) {
  const float amax = __uint_as_float(amax_bits);
  if (!(amax > 0.f)) return 1.0;
  const int e = ilogb(static_cast<double>(amax) * (static_cast<double>(ns) * (f0 > 1 ? f0 : 1) + 1.0)) + 1;
  return ldexp(1.0, 62 - e);
}

// Scatter through the outer mean aggregation into dh1 (trainer.cpp:182-198):
// dh1[src] += dagg[s] for every layer-0 edge (s -> src), dh1[s] += dagg[s]
// for self-fallback seeds -- as 64-bit fixed-point integer atomics, which add
// associatively: the result is independent of the order (deterministic) and
// more precise than an fp32 sum.
__global__ void __launch_bounds__(256) k_dh1_scatter(const float* dagg, const uint32_t* amax, const uint32_t* ns_p,
                                                     const uint32_t* cnt0, const uint32_t* sidx0, uint32_t f0,
                                                     int has_layer0, uint32_t H, unsigned long long* fx) {
  const uint32_t ns = *ns_p;
  const double scale = fx_scale(*amax, ns, has_layer0 ? f0 : 1u);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < static_cast<uint64_t>(ns) * H;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = static_cast<uint32_t>(i / H), h = static_cast<uint32_t>(i - static_cast<uint64_t>(s) * H);
    const unsigned long long q = static_cast<unsigned long long>(llrint(static_cast<double>(dagg[i]) * scale));
    const uint32_t c0 = has_layer0 ? cnt0[s] : 0u;
    if (c0 == 0) {
      atomicAdd(fx + static_cast<uint64_t>(s) * H + h, q);
    } else {
      const uint32_t* srcs = sidx0 + static_cast<uint64_t>(s) * f0;
      for (uint32_t t = 0; t < c0; ++t) atomicAdd(fx + static_cast<uint64_t>(srcs[t]) * H + h, q);
    }
  }
}

// dh1 = fixed point / scale (rows < n_inner); clears the accumulator for the next step.
__global__ void k_dh1_fix(unsigned long long* fx, const uint32_t* amax, const uint32_t* ns_p, uint32_t f0,
                          const uint32_t* n_inner, uint32_t H, float* dh1) {
  const double inv = 1.0 / fx_scale(*amax, *ns_p, f0);
  const uint64_t total = static_cast<uint64_t>(*n_inner) * H;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    dh1[i] = static_cast<float>(static_cast<double>(static_cast<long long>(fx[i])) * inv);
    fx[i] = 0ull;
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
  // fused SGD (single worker: no gradient exchange between reduce and step)
  float* w1;
  float* w2;
  float lr;
  double* loss_slot;
  int sgd;
};

// blocks [0, nb1): dW1 = sum of the row-split partials (fixed order);
// blocks [nb1, nb1 + H*C): one dW2 entry each, agg_outer^T . dlogits as a
// fixed-shape block tree (trainer.cpp:174-175); last block: the loss sum.
__global__ void __launch_bounds__(256) k_reduce(ReduceArgs a, uint32_t nb1) {
  __shared__ float s_l[256];
  const uint32_t FH = a.F * a.H, HC = a.H * a.C;
  const uint32_t ns = *a.ns;
  if (blockIdx.x < nb1) {
    // 32 consecutive entries per block, the partials strided over 8 thread
    // rows (coalesced), then the 8 row sums in order: a fixed-shape tree
    const uint32_t j = threadIdx.x & 31, k = threadIdx.x >> 5;
    const uint32_t i = blockIdx.x * 32 + j;
    float x = 0.f;
    if (i < FH)
      for (uint32_t p = k; p < a.nparts; p += 8) x += a.part[static_cast<uint64_t>(p) * FH + i];
    s_l[threadIdx.x] = x;
    __syncthreads();
    if (k == 0 && i < FH) {
      float t = s_l[j];
#pragma unroll
      for (int r = 1; r < 8; ++r) t += s_l[j + 32 * r];
      a.gw[i] = t;
      if (a.sgd) a.w1[i] -= a.lr * t;
    }
    return;
  }
  const uint32_t q = blockIdx.x - nb1;
  float x = 0.f;
  if (q < HC) {
    const uint32_t j = q / a.C, c = q % a.C;
    for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x)
      x = fmaf(a.agg_outer[static_cast<uint64_t>(t) * a.H + j], a.dlogits[static_cast<uint64_t>(t) * a.C + c], x);
  } else {
    for (uint32_t t = threadIdx.x; t < ns; t += blockDim.x) x += a.loss_s[t];
  }
  s_l[threadIdx.x] = x;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s_l[threadIdx.x] += s_l[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (q < HC) {
      a.gw[FH + q] = s_l[0];
      if (a.sgd) a.w2[q] -= a.lr * s_l[0];
    } else {
      a.gw[FH + HC] = static_cast<float>(ns);
      a.gw[FH + HC + 1] = s_l[0];  // sum of per-seed losses = mean * n
      if (a.sgd && a.loss_slot) *a.loss_slot = static_cast<double>(s_l[0]) / static_cast<float>(ns);
    }
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

template <typename T, int N, int W, int S, int LPR, int HB, bool PAIR = false>
void launch_agg_cfg(TrainerState& t, const AggArgs& aa, cudaStream_t st) {
  const size_t ring = static_cast<size_t>(W) * S * (32 / LPR) * aa.view.row_bytes;
  const size_t smem = ring + (HB > 0 ? static_cast<size_t>(aa.pitch) * HB * 4 : 0);
  if (smem > 227 * 1024) raise(A3G_ERR_PARAMETER, "feature row too wide for k_agg1's shared-memory ring");
  const int grid = t.sm_count * (smem * 2 <= 227 * 1024 && W <= 32 ? 2 : 1);
  A3G_CUDA(cudaFuncSetAttribute(k_agg1<T, N, W, S, LPR, HB, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  k_agg1<T, N, W, S, LPR, HB, PAIR><<<grid, W * 32, smem, st>>>(aa);
}

// The paired h1 epilogue (two rows per pass over W1) needs ~128 registers:
// 16-warp CTAs. Default for long rows (LPR 32: C2 k_agg1 0.528 -> 0.541 of
// HBM alone); short rows (LPR 8) measured slower (C3 0.347 -> 0.301).
// A3G_AGG_PAIR=0 disables it, =16 forces it (A/B), =24 (spills) for sweeps.
static int agg_pair(int lpr) {
  static const int v = [] {
    const char* e = std::getenv("A3G_AGG_PAIR");
    return e ? std::atoi(e) : -1;
  }();
  if (v < 0) return lpr == 32 ? 16 : 0;
  return v == 16 || v == 24 ? v : 0;
}

// 24 warps per CTA (more warps beat a deeper ring: r01 sweep 8x8 63 us,
// 16x4 53 us, 24x3 51 us on C2); ring depth from the row size.
static int agg_warps() {
  static const int v = [] {
    const char* e = std::getenv("A3G_AGG_WARPS");
    return e && std::atoi(e) == 16 ? 16 : 24;
  }();
  return v;
}

// TMA bulk-copy gather for long rows (default; A3G_AGG_TMA=0 selects the
// per-lane LDGSTS kernel for A/B).
static bool agg_tma() {
  static const bool v = [] {
    const char* e = std::getenv("A3G_AGG_TMA");
    return !(e && std::atoi(e) == 0);
  }();
  return v;
}

template <typename T, int N, int HB>
bool launch_agg_tma(TrainerState& t, const AggArgs& aa, cudaStream_t st) {
  constexpr int W = N <= 8 ? 16 : 8;
  constexpr int S = N <= 5 ? 4 : 2;
  const size_t ring = static_cast<size_t>(W) * S * aa.view.row_bytes;
  const size_t smem = ring + (HB > 0 ? static_cast<size_t>(aa.pitch) * HB * 4 : 0);
  const size_t stat = static_cast<size_t>(W) * S * (sizeof(uint64_t) + sizeof(uint2));
  if (smem + stat > 227 * 1024) return false;
  if (aa.view.loc == nullptr) {
    A3G_CUDA(cudaFuncSetAttribute(k_agg1_tma<T, N, W, S, HB, (HB > 0), true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_agg1_tma<T, N, W, S, HB, (HB > 0), true><<<t.sm_count, W * 32, smem, st>>>(aa);
  } else {
    A3G_CUDA(cudaFuncSetAttribute(k_agg1_tma<T, N, W, S, HB, (HB > 0), false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_agg1_tma<T, N, W, S, HB, (HB > 0), false><<<t.sm_count, W * 32, smem, st>>>(aa);
  }
  return true;
}

template <typename T, int N, int LPR, int HB>
void launch_agg_n(TrainerState& t, const AggArgs& aa, cudaStream_t st) {
  if constexpr (LPR == 32) {
    if (agg_tma() && launch_agg_tma<T, N, HB>(t, aa, st)) return;
  }
  if constexpr (HB > 0) {
    if (agg_pair(LPR) == 16) {
      const uint64_t ps = 16ull * (32 / LPR) * aa.view.row_bytes;
      if (ps * 4 + static_cast<uint64_t>(aa.pitch) * HB * 4 <= 227 * 1024)
        launch_agg_cfg<T, N, 16, 4, LPR, HB, true>(t, aa, st);
      else
        launch_agg_cfg<T, N, 16, 3, LPR, HB, true>(t, aa, st);
      return;
    }
    if (agg_pair(LPR) == 24) {
      launch_agg_cfg<T, N, 24, 3, LPR, HB, true>(t, aa, st);
      return;
    }
  }
  if (agg_warps() == 16) {  // smaller CTA footprint (co-residence with sampling CTAs)
    const uint64_t ps = 16ull * (32 / LPR) * aa.view.row_bytes;
    if (ps * 6 <= 120 * 1024)
      launch_agg_cfg<T, N, 16, 6, LPR, HB>(t, aa, st);
    else if (ps * 4 <= 120 * 1024)
      launch_agg_cfg<T, N, 16, 4, LPR, HB>(t, aa, st);
    else
      launch_agg_cfg<T, N, 16, 3, LPR, HB>(t, aa, st);
    return;
  }
  const uint64_t per_slot = 24ull * (32 / LPR) * aa.view.row_bytes;
  const uint64_t w1_bytes = HB > 0 ? static_cast<uint64_t>(aa.pitch) * HB * 4 : 0;
  if (per_slot * 3 + w1_bytes > 227 * 1024) {
    // wide rows (up to the 8 KB the chunk layout covers): 8 warps x 2 ring
    // slots stream them instead of refusing the width
    launch_agg_cfg<T, N, 8, 2, LPR, HB>(t, aa, st);
    return;
  }
  if (per_slot * 8 <= 176 * 1024)
    launch_agg_cfg<T, N, 24, 8, LPR, HB>(t, aa, st);
  else if (per_slot * 6 <= 176 * 1024)
    launch_agg_cfg<T, N, 24, 6, LPR, HB>(t, aa, st);
  else if (per_slot * 4 <= 176 * 1024)
    launch_agg_cfg<T, N, 24, 4, LPR, HB>(t, aa, st);
  else
    launch_agg_cfg<T, N, 24, 3, LPR, HB>(t, aa, st);
}

template <typename T, int HB>
void launch_agg_h(TrainerState& t, const AggArgs& aa, uint32_t chunks, cudaStream_t st) {
  if (chunks <= 8) {
    launch_agg_n<T, 1, 8, HB>(t, aa, st);
  } else if (chunks <= 16) {
    launch_agg_n<T, 2, 8, HB>(t, aa, st);
  } else if (chunks <= 32) {  // 4 rows per warp step (100-d f32 rows: 106 -> 61 us at C3; LPR 16: 67 us)
    launch_agg_n<T, 4, 8, HB>(t, aa, st);
  } else {
    switch ((chunks + 31) / 32) {
      case 1: launch_agg_n<T, 1, 32, HB>(t, aa, st); break;
      case 2: launch_agg_n<T, 2, 32, HB>(t, aa, st); break;
      case 3: launch_agg_n<T, 3, 32, HB>(t, aa, st); break;
      case 4: launch_agg_n<T, 4, 32, HB>(t, aa, st); break;
      case 5: launch_agg_n<T, 5, 32, HB>(t, aa, st); break;
      case 6: launch_agg_n<T, 6, 32, HB>(t, aa, st); break;
      case 7: case 8: launch_agg_n<T, 8, 32, HB>(t, aa, st); break;
      case 9: case 10: case 11: case 12: case 13: case 14: case 15: case 16:
        launch_agg_n<T, 16, 32, HB>(t, aa, st);
        break;
      default:
        raise(A3G_ERR_PARAMETER, "feature row too wide for k_agg1");
    }
  }
}

// rows of <= 32 chunks (16 B) go 4 rows per warp step (LPR 8): short rows
// are issue-bound, not bandwidth-bound. H <= 16 with W1 fitting beside the
// ring fuses h1 = relu(agg . W1) into the epilogue (returns true); otherwise
// the tcgen05 GEMM computes h1 afterwards.
template <typename T>
bool launch_agg(TrainerState& t, AggArgs aa, uint32_t chunks, cudaStream_t st) {
  const bool fuse = !t.tc_gemms && t.H <= 16 && static_cast<size_t>(aa.pitch) * 16 * 4 <= 48 * 1024;
  if (fuse)
    launch_agg_h<T, 16>(t, aa, chunks, st);
  else
    launch_agg_h<T, 0>(t, aa, chunks, st);
  A3G_LAUNCH_DONE("k_agg1", st);
  return fuse;
}

}  // namespace

// Per-resource accounting of the gather (a3g_trainer_set_tier_accounting):
// the distinct feature rows k_agg1 reads -- every layer-1 source of an inner
// row, or the row itself on the self-fallback -- by the tier they live in
// (StoreView loc: HBM shard r < 15, pinned host 15; identity layout: 0).
// Off by default; the bench's roofline leg turns it on, and it runs after
// k_agg1's timing events.
__global__ void k_tier_rows(const uint32_t* unique, const int32_t* inv1, const uint32_t* cnt1, const uint32_t* S1,
                            uint32_t f1, const uint32_t* n_inner_p, int has_layer1, const uint32_t* loc,
                            uint32_t* seen, unsigned long long* tier_rows) {
  const uint32_t n_inner = *n_inner_p;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_inner; r += gridDim.x * blockDim.x) {
    const int32_t k = has_layer1 ? inv1[r] : -1;
    const uint32_t c = k >= 0 ? cnt1[k] : 0u;
    for (uint32_t t = 0; t < (c ? c : 1u); ++t) {
      const uint32_t v = c ? S1[static_cast<uint64_t>(k) * f1 + t] : unique[r];
      const uint32_t bit = 1u << (v & 31);
      if (!(atomicOr(seen + (v >> 5), bit) & bit))
        atomicAdd(tier_rows + (loc ? (__ldg(loc + v) >> kLocShift) : 0u), 1ull);
    }
  }
}

// nccl glue lives in comm.cpp
void comm_allreduce_sum(a3g_comm* comm, float* buf, size_t count, cudaStream_t st);

// per-step statistics of a sampled batch (a3g_trainer_step_stats); the
// pipeline runs it on the batch's sampling stream, off the compute chain
void launch_step_stats(TrainerState& t, a3g_sampler* smp, unsigned long long* d_stats, cudaStream_t st) {
  SamplerState& s = smp->st;
  const a3g_cache* c = t.c;
  const int bitmode = c->all_cached ? 1 : (c->none_cached ? 0 : 2);
  k_step_stats<<<t.sm_count, 256, 0, st>>>(s.d_ctr, s.d_unique, c->d_bits, bitmode, s.L, d_stats,
                                           t.d_agg_bytes + 1);
  A3G_LAUNCH_DONE("k_step_stats", st);
}

void launch_train_compute(TrainerState& t, a3g_sampler* smp, double lr, double* d_loss_slot,
                          unsigned long long* d_stats, cudaStream_t st, bool record_timing) {
  SamplerState& s = smp->st;
  a3g_graph* g = t.g;
  BatchCounters* ctr = s.d_ctr;
  if (d_stats) launch_step_stats(t, smp, d_stats, st);
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
  aa.n_distinct = s.L >= 2 ? &ctr->nfront[2] : nullptr;
  aa.agg_inner = t.d_agg_inner;
  aa.bytes = t.d_agg_bytes;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (record_timing) {
    e0 = pool_event(t);
    e1 = pool_event(t);
    A3G_CUDA(cudaEventRecord(e0, st));
  }
  aa.w1 = t.d_w1;
  aa.h1 = t.d_h1;
  bool fused;
  if (g->feat_dtype == A3G_FEAT_BF16)
    fused = launch_agg<uint16_t>(t, aa, g->pitch / 8, st);
  else
    fused = launch_agg<float>(t, aa, g->pitch / 4, st);
  t.h1_fused = fused;
  if (record_timing) {
    A3G_CUDA(cudaEventRecord(e1, st));
    t.ev_agg.push_back(e0);
    t.ev_agg.push_back(e1);
  }
  if (t.tier_acct) {
    k_tier_rows<<<t.sm_count * 2, 256, 0, st>>>(s.d_unique, s.d_inv1, aa.cnt1, aa.S1, aa.f1, aa.n_inner,
                                                aa.has_layer1, g->view.loc, t.d_tier_seen, t.d_tier_rows);
    A3G_LAUNCH_DONE("k_tier_rows", st);
    A3G_CUDA(cudaMemsetAsync(t.d_tier_seen, 0, (g->n + 31) / 32 * 4, st));
  }
  if (!fused) {
    cudaEvent_t g0 = nullptr, g1 = nullptr;
    if (record_timing) {
      g0 = pool_event(t);
      g1 = pool_event(t);
      A3G_CUDA(cudaEventRecord(g0, st));
    }
    launch_h1_tc(t, t.d_agg_inner, aa.n_inner, t.d_h1, st);
    if (record_timing) {
      A3G_CUDA(cudaEventRecord(g1, st));
      t.ev_h1.push_back(g0);
      t.ev_h1.push_back(g1);
    }
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
  oa.amax = t.d_amax;
  A3G_CUDA(cudaMemsetAsync(t.d_amax, 0, sizeof(uint32_t), st));
  if (t.H <= 32)
    k_outer<1><<<std::max(1, static_cast<int>((t.max_seeds + 7) / 8)), 256, 0, st>>>(oa);
  else
    k_outer<8><<<std::max(1, static_cast<int>((t.max_seeds + 7) / 8)), 256, 0, st>>>(oa);
  A3G_LAUNCH_DONE("k_outer", st);
  // ---- deterministic scatter into dh1 (fixed-point integer atomics)
  k_dh1_scatter<<<t.sm_count * 2, 256, 0, st>>>(t.d_dagg, t.d_amax, oa.ns, oa.cnt0, oa.sidx0, oa.f0, oa.has_layer0,
                                                t.H, t.d_dh1_fx);
  A3G_LAUNCH_DONE("k_dh1_scatter", st);
  k_dh1_fix<<<t.sm_count * 2, 256, 0, st>>>(t.d_dh1_fx, t.d_amax, oa.ns, oa.has_layer0 ? oa.f0 : 1u, aa.n_inner,
                                            t.H, t.d_dh1);
  A3G_LAUNCH_DONE("k_dh1_fix", st);
  // ---- dW1 = agg_inner^T . (dh1 * [h1 > 0]), partials per row split
  uint32_t nparts;
  if (t.tc_gemms || t.H > 32) {
    nparts = t.tc_splits;
    cudaEvent_t g0 = nullptr, g1 = nullptr;
    if (record_timing) {
      g0 = pool_event(t);
      g1 = pool_event(t);
      A3G_CUDA(cudaEventRecord(g0, st));
    }
    launch_dw1_tc(t, t.d_agg_inner, aa.n_inner, t.d_h1, t.d_dh1, t.d_part, nparts, st);
    if (record_timing) {
      A3G_CUDA(cudaEventRecord(g1, st));
      t.ev_dw1.push_back(g0);
      t.ev_dw1.push_back(g1);
    }
  } else {
    nparts = t.dw1_splits;
    const dim3 grid((t.F + 127) / 128, nparts);
    if (t.H <= 16) {
      static std::atomic<uint64_t> attr16{0};
      smem_attr_once(attr16, reinterpret_cast<const void*>(k_dw1_fma<16>), dw1_smem(16));
      k_dw1_fma<16><<<grid, 128, dw1_smem(16), st>>>(t.d_agg_inner, t.pitch, t.F, t.H, aa.n_inner, t.d_h1, t.d_dh1,
                                                      t.d_part);
    } else {
      static std::atomic<uint64_t> attr32{0};
      smem_attr_once(attr32, reinterpret_cast<const void*>(k_dw1_fma<32>), dw1_smem(32));
      k_dw1_fma<32><<<grid, 128, dw1_smem(32), st>>>(t.d_agg_inner, t.pitch, t.F, t.H, aa.n_inner, t.d_h1, t.d_dh1,
                                                      t.d_part);
    }
    A3G_LAUNCH_DONE("k_dw1_fma", st);
  }
  // ---- reduce -> grads, loss
  ReduceArgs ra{};
  ra.part = t.d_part;
  ra.nparts = nparts;
  ra.agg_outer = t.d_agg_outer;
  ra.dlogits = t.d_dlogits;
  ra.loss_s = t.d_loss_s;
  ra.ns = &ctr->ucount[0];
  ra.F = t.F;
  ra.H = t.H;
  ra.C = t.C;
  ra.gw = t.d_gw;
  const uint32_t FH = t.F * t.H, HC = t.H * t.C;
  const uint32_t nb1 = (FH + 31) / 32;
  const bool synced = t.comm != nullptr;
  ra.w1 = t.d_w1;
  ra.w2 = t.d_w2;
  ra.lr = static_cast<float>(lr);
  ra.loss_slot = d_loss_slot;
  ra.sgd = synced ? 0 : 1;  // one worker: the SGD step rides on the reduction
  k_reduce<<<nb1 + HC + 1, 256, 0, st>>>(ra, nb1);
  A3G_LAUNCH_DONE("k_reduce", st);
  if (!synced) return;
  {
    k_scale_for_sync<<<t.sm_count, 256, 0, st>>>(t.d_gw, FH + HC);
    A3G_LAUNCH_DONE("k_scale_for_sync", st);
    comm_allreduce_sum(t.comm, t.d_gw, FH + HC + 2, st);
  }
  k_sgd<<<t.sm_count, 256, 0, st>>>(t.d_w1, t.d_w2, t.d_gw, FH, HC, static_cast<float>(lr), synced ? 1 : 0,
                                    d_loss_slot);
  A3G_LAUNCH_DONE("k_sgd", st);
}

}  // namespace a3g

