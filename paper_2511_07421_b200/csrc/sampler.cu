// sampler.cu -- locality-aware k-hop sampler for sm_100a.
//
// Replaces sampling::sample_khop (proj/src/sampler.cpp:89-137) with the exact
// same output: weighted reservoir (Algo 2, sampler.cpp:9-42) or Algorithm R
// (sampler.cpp:44-58) per frontier node with the reference's counter RNG keyed
// by hash2(step_seed, hash2(layer, node)) (sampler.cpp:117), global first-seen
// relabelling (Interner, sampler.cpp:72-85) and per-layer first-seen frontiers
// (sampler.cpp:113-131).
//
// Per layer:
//   k_sample_rows   warp per frontier row (dynamic chunks of rows). deg <= m:
//                   copy; m < deg <= kSeg: in-warp exact replay (slot = lane,
//                   ballot of keys > current min, 4-chunk prefetch); deg > kSeg
//                   ("hubs", up to n-1 neighbours): registered for splitting.
//   k_hub_segments  warp per kSeg-long segment of a hub row: local replay from
//                   an empty reservoir, emitting every local insertion
//                   ("record") and the segment's exact m-th largest key tau_s.
//                   Every global insertion is a local record of its segment.
//   k_hub_merge     block per hub: records of segment s with key <= max_{s'<s}
//                   tau_{s'} can never beat the global minimum and are dropped
//                   in parallel; warp 0 replays the survivors in order, which
//                   reproduces the sequential slot history exactly.
//   k_fin_count / k_fin_emit: first-seen dedup + relabel (tagged atomicMax of
//                   the first position, tile partials, ballot scans).
// Counts stay on the device: no host sync inside a batch.
#include <cmath>

#include "sampler.cuh"

namespace a3g {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kRowChunk = 4;  // rows claimed per atomic by a warp
constexpr int kPrefetch = 4;  // 32-key chunks loaded ahead per replay step

__device__ __forceinline__ void warp_argmin(double& k, int& idx) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double ok = __shfl_xor_sync(kFull, k, off);
    const int oi = __shfl_xor_sync(kFull, idx, off);
    if (ok < k || (ok == k && oi < idx)) {
      k = ok;
      idx = oi;
    }
  }
}

__device__ __forceinline__ void mark_first(uint64_t* first, uint32_t v, uint32_t tag, uint32_t pos) {
  atomicMax(reinterpret_cast<unsigned long long*>(first + v),
            (static_cast<unsigned long long>(tag) << 32) | static_cast<unsigned long long>(~pos));
}

// Lower bound in u-space below which a gamma-weighted key pow(u, 1/gamma)
// cannot exceed thr (conservative by a 1e-6 relative margin).
__device__ __forceinline__ double gamma_lo(double thr, double gamma) {
  if (gamma > 1e8) return 0.0;
  return pow(thr, gamma) * (1.0 - 1e-6);
}

struct SampleArgs {
  const uint64_t* ro;
  const uint32_t* col;
  const uint32_t* bits;
  const uint32_t* front;
  const uint32_t* nrows;  // device count of frontier rows
  uint32_t* cnt;
  uint32_t* S;
  uint64_t* first;
  uint32_t* work;
  double* scratch;  // [cap_rows*f] keys, only for f > 32 serial path
  HubArena hub;
  uint32_t* hub_count;
  uint32_t* seg_count;
  uint64_t seed;
  double gamma, inv_gamma;
  uint32_t f, layer, tag;
  int kind;   // A3G_SAMPLER_*
  int wmode;  // 0: all weights 1; 1: all gamma; 2: bitmap
};

__device__ __forceinline__ bool is_gamma(const SampleArgs& a, uint32_t v) {
  return a.wmode == 1 || (a.wmode == 2 && ((__ldg(a.bits + (v >> 5)) >> (v & 31)) & 1u));
}

// Weight of neighbour j (node v): assign_weights (sampler.cpp:60-68).
struct BitmapWeight {
  const SampleArgs* a;
  __device__ __forceinline__ bool unit(uint32_t v, uint64_t) const { return !is_gamma(*a, v); }
  __device__ __forceinline__ double inv_w(uint32_t, uint64_t) const { return a->inv_gamma; }
};
struct ListWeight {  // explicit weights (test hook a3g_weighted_reservoir)
  const double* w;
  __device__ __forceinline__ bool unit(uint32_t, uint64_t j) const { return w[j] == 1.0; }
  __device__ __forceinline__ double inv_w(uint32_t, uint64_t j) const { return 1.0 / w[j]; }
};

// Reservoir state of one warp: slot = lane (m <= 32), lanes >= m hold +inf.
struct WState {
  double my_key;
  uint32_t my_id;
  double thr;  // current minimum key (keys[min_pos])
  int mp;      // min_pos: first slot holding the minimum (std::min_element)
};

struct NoEmit {
  __device__ __forceinline__ void operator()(uint32_t, double, int) const {}
};

// Fill slots [0, nf) from positions j0 + lane (sampler.cpp:30-33); every fill
// is an insertion. Draw number of position j is c0 + j + 1.
template <typename WF, typename Emit>
__device__ __forceinline__ void fill_slots(const uint32_t* nb, uint64_t j0, uint32_t nf, uint64_t key,
                                           uint64_t c0, int lane, const WF& wf, WState& s, const Emit& emit) {
  s.my_key = INFINITY;
  s.my_id = 0;
  if (lane < static_cast<int>(nf)) {
    const uint64_t j = j0 + lane;
    const uint32_t v = __ldg(nb + j);
    const double u = unit_of(draw(key, c0 + j + 1));
    s.my_key = wf.unit(v, j) ? u : pow(u, wf.inv_w(v, j));
    s.my_id = v;
    emit(v, s.my_key, lane);
  }
  s.thr = s.my_key;
  s.mp = lane;
  warp_argmin(s.thr, s.mp);
}

// Replay positions [jb, je) against a full reservoir (sampler.cpp:34-39):
// a key replaces slot min_pos iff strictly greater than keys[min_pos]; then
// min_pos = first minimum. Chunks of 32 keys, kPrefetch chunks in flight.
// With a single non-unit weight (use_filter) a gamma-key is only evaluated
// (pow) when u >= thr^gamma*(1-1e-6): below that, pow(u,1/gamma) < thr for any
// <= 2-ulp pow, so no decision can change.
template <typename WF, typename Emit>
__device__ __forceinline__ void replay_range(const uint32_t* nb, uint64_t jb, uint64_t je, uint64_t key,
                                             uint64_t c0, int lane, const WF& wf, bool use_filter,
                                             double gamma, WState& s, const Emit& emit) {
  double lo = use_filter ? gamma_lo(s.thr, gamma) : 0.0;
  for (uint64_t b = jb; b < je; b += 32 * kPrefetch) {
    uint32_t v[kPrefetch];
    double kk[kPrefetch];
#pragma unroll
    for (int q = 0; q < kPrefetch; ++q) {
      const uint64_t j = b + q * 32 + lane;
      v[q] = j < je ? __ldg(nb + j) : 0u;
    }
#pragma unroll
    for (int q = 0; q < kPrefetch; ++q) {
      const uint64_t j = b + q * 32 + lane;
      kk[q] = -1.0;
      if (j < je) {
        const double u = unit_of(draw(key, c0 + j + 1));
        if (wf.unit(v[q], j)) {
          kk[q] = u;
        } else if (u >= lo) {
          kk[q] = pow(u, wf.inv_w(v[q], j));
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kPrefetch; ++q) {
      unsigned mask = __ballot_sync(kFull, kk[q] > s.thr);
      if (mask) {
        while (mask) {
          const int src = __ffs(mask) - 1;
          const double kv = __shfl_sync(kFull, kk[q], src);
          const uint32_t iv = __shfl_sync(kFull, v[q], src);
          if (lane == s.mp) {
            s.my_key = kv;
            s.my_id = iv;
          }
          emit(iv, kv, src);
          s.thr = s.my_key;
          s.mp = lane;
          warp_argmin(s.thr, s.mp);
          mask &= __ballot_sync(kFull, kk[q] > s.thr) & ~((2u << src) - 1u);
        }
        if (use_filter) lo = gamma_lo(s.thr, gamma);
      }
    }
  }
}

// Weighted reservoir of one whole row by one warp, m <= 32 < deg.
template <typename WF>
__device__ __forceinline__ uint32_t weighted_row_warp(const uint32_t* nb, uint64_t deg, uint32_t m,
                                                      uint64_t key, int lane, const WF& wf,
                                                      bool use_filter, double gamma, uint64_t c0 = 0) {
  WState s;
  fill_slots(nb, 0, m, key, c0, lane, wf, s, NoEmit{});
  replay_range(nb, m, deg, key, c0, lane, wf, use_filter, gamma, s, NoEmit{});
  return s.my_id;
}

// Algorithm R (sampler.cpp:44-58) by one warp over positions [jb, je), jb >=
// m: slot r of position j is replaced iff r = next_below(j+1) < m (draw number
// c0 + j - m + 1); candidates applied in position order.
__device__ __forceinline__ void uniform_range(const uint32_t* nb, uint64_t jb, uint64_t je, uint32_t m,
                                              uint64_t key, int lane, uint64_t c0, uint32_t& my_id) {
  for (uint64_t b = jb; b < je; b += 32) {
    const uint64_t j = b + lane;
    const bool valid = j < je;
    uint32_t r = kInv, v = 0;
    if (valid) {
      r = static_cast<uint32_t>(__umul64hi(draw(key, c0 + j - m + 1), j + 1));
      if (r < m) v = __ldg(nb + j);
    }
    unsigned mask = __ballot_sync(kFull, valid && r < m);
    while (mask) {
      const int src = __ffs(mask) - 1;
      const uint32_t slot = __shfl_sync(kFull, r, src);
      const uint32_t iv = __shfl_sync(kFull, v, src);
      if (lane == static_cast<int>(slot)) my_id = iv;
      mask &= mask - 1;
    }
  }
}

__device__ __forceinline__ uint32_t uniform_row_warp(const uint32_t* nb, uint64_t deg, uint32_t m,
                                                     uint64_t key, int lane, uint64_t c0 = 0) {
  uint32_t my_id = lane < static_cast<int>(m) ? __ldg(nb + lane) : 0u;
  uniform_range(nb, m, deg, m, key, lane, c0, my_id);
  return my_id;
}

// Thread-serial exact reservoir for rows with f > 32 (rare; e.g. exhaustive
// fanouts). Writes the row's slots and keys directly.
__device__ void serial_row(const SampleArgs& a, const uint32_t* nb, uint64_t deg, uint64_t key,
                           uint32_t* out, double* keys) {
  const uint32_t m = a.f;
  if (a.kind == A3G_SAMPLER_UNIFORM) {
    for (uint64_t j = 0; j < deg; ++j) {
      if (j < m) {
        out[j] = nb[j];
      } else {
        const uint64_t r = __umul64hi(draw(key, j - m + 1), j + 1);
        if (r < m) out[r] = nb[j];
      }
    }
    return;
  }
  uint32_t cnt = 0, mp = 0;
  for (uint64_t j = 0; j < deg; ++j) {
    const uint32_t v = nb[j];
    const double u = unit_of(draw(key, j + 1));
    const double k = is_gamma(a, v) ? pow(u, a.inv_gamma) : u;
    if (cnt < m) {
      out[cnt] = v;
      keys[cnt] = k;
      ++cnt;
      if (k < keys[mp]) mp = cnt - 1;
    } else if (k > keys[mp]) {
      out[mp] = v;
      keys[mp] = k;
      mp = 0;
      for (uint32_t t = 1; t < cnt; ++t)
        if (keys[t] < keys[mp]) mp = t;
    }
  }
}

// Whole row by one warp (m <= 32 < deg); writes slots + first-position marks.
__device__ __forceinline__ void row_by_warp(const SampleArgs& a, const uint32_t* nb, uint64_t deg, uint64_t key,
                                            uint32_t k, int lane) {
  const uint32_t m = a.f;
  uint32_t my_id;
  if (a.kind == A3G_SAMPLER_UNIFORM) {
    my_id = uniform_row_warp(nb, deg, m, key, lane);
  } else {
    const BitmapWeight wf{&a};
    my_id = weighted_row_warp(nb, deg, m, key, lane, wf, a.wmode != 0, a.gamma);
  }
  const uint64_t row0 = static_cast<uint64_t>(k) * m;
  if (lane < static_cast<int>(m)) {
    a.S[row0 + lane] = my_id;
    mark_first(a.first, my_id, a.tag, static_cast<uint32_t>(row0 + lane));
  }
  if (lane == 0) a.cnt[k] = m;
}

__global__ void __launch_bounds__(256) k_sample_rows(SampleArgs a) {
  const int lane = threadIdx.x & 31;
  const uint32_t nrows = *a.nrows;
  const uint32_t m = a.f;
  for (;;) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(a.work, kRowChunk);
    base = __shfl_sync(kFull, base, 0);
    if (base >= nrows) break;
    const uint32_t rend = min(base + kRowChunk, nrows);
    for (uint32_t k = base; k < rend; ++k) {
      const uint32_t dst = __ldg(a.front + k);
      const uint64_t beg = __ldg(a.ro + dst), deg = __ldg(a.ro + dst + 1) - beg;
      const uint32_t* nb = a.col + beg;
      const uint64_t row0 = static_cast<uint64_t>(k) * m;
      if (deg <= m) {  // fill phase only: output = neighbour list (sampler.cpp:30-33)
        for (uint32_t t = lane; t < deg; t += 32) {
          const uint32_t v = __ldg(nb + t);
          a.S[row0 + t] = v;
          mark_first(a.first, v, a.tag, static_cast<uint32_t>(row0 + t));
        }
        if (lane == 0) a.cnt[k] = static_cast<uint32_t>(deg);
        continue;
      }
      const uint64_t key = hash2(a.seed, hash2(a.layer, dst));  // sampler.cpp:117
      if (m > 32) {
        if (lane == 0) serial_row(a, nb, deg, key, a.S + row0, a.scratch + row0);
        __syncwarp();
        for (uint32_t t = lane; t < m; t += 32)
          mark_first(a.first, a.S[row0 + t], a.tag, static_cast<uint32_t>(row0 + t));
        if (lane == 0) a.cnt[k] = m;
        continue;
      }
      if (deg > kSeg) {  // hub: register for the segmented path
        const uint32_t nseg = static_cast<uint32_t>((deg + kSeg - 1) / kSeg);
        uint32_t h = 0, s0 = 0;
        if (lane == 0) {
          h = atomicAdd(a.hub_count, 1u);
          s0 = atomicAdd(a.seg_count, nseg);
          const bool ok = h < a.hub.hub_cap && s0 + static_cast<uint64_t>(nseg) <= a.hub.seg_cap;
          if (h < a.hub.hub_cap) {
            a.hub.row[h] = k;
            a.hub.seg0[h] = s0;
            a.hub.nseg[h] = ok ? nseg : 0u;  // 0 = handled here (capacity exceeded)
          }
          if (!ok) h = kInv;
        }
        h = __shfl_sync(kFull, h, 0);
        s0 = __shfl_sync(kFull, s0, 0);
        if (h != kInv) {
          for (uint32_t i = lane; i < nseg; i += 32) a.hub.seg_hub[s0 + i] = h;
          continue;
        }
      }
      row_by_warp(a, nb, deg, key, k, lane);
    }
  }
}

// Local replay of one hub segment [sb, se) from an empty reservoir; records =
// every local insertion (id, key) in order; tau = segment's m-th largest key.
struct SegEmit {
  uint32_t* rid;
  double* rkey;
  uint32_t* cnt;  // warp-uniform counter (register, by reference)
  uint32_t cap;
  int lane;
  __device__ __forceinline__ void operator()(uint32_t id, double key, int src) const {
    const uint32_t c = *cnt;
    if (lane == src && c < cap) {
      rid[c] = id;
      rkey[c] = key;
    }
    *cnt = c + 1;
  }
};
struct FillEmit {  // fills: lane i writes record i (records 0..nf-1)
  uint32_t* rid;
  double* rkey;
  uint32_t cap;
  __device__ __forceinline__ void operator()(uint32_t id, double key, int lane) const {
    if (static_cast<uint32_t>(lane) < cap) {
      rid[lane] = id;
      rkey[lane] = key;
    }
  }
};

__global__ void __launch_bounds__(256) k_hub_segments(SampleArgs a) {
  const int lane = threadIdx.x & 31;
  const uint32_t nhub = min(*a.hub_count, a.hub.hub_cap);
  const uint32_t nseg_total = min(*a.seg_count, a.hub.seg_cap);
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t m = a.f;
  for (uint32_t s = gw; s < nseg_total; s += nw) {
    const uint32_t h = a.hub.seg_hub[s];
    if (h >= nhub) continue;  // stale entry
    const uint32_t s0 = a.hub.seg0[h], ns = a.hub.nseg[h];
    if (s < s0 || s >= s0 + ns) continue;
    const uint32_t k = a.hub.row[h];
    const uint32_t dst = a.front[k];
    const uint64_t beg = a.ro[dst], deg = a.ro[dst + 1] - beg;
    const uint32_t* nb = a.col + beg;
    const uint64_t key = hash2(a.seed, hash2(a.layer, dst));
    const uint64_t sb = static_cast<uint64_t>(s - s0) * kSeg, se = min(deg, sb + kSeg);
    if (a.kind == A3G_SAMPLER_UNIFORM) {
      // last position per slot within the segment (positions >= m)
      uint32_t last = kInv;  // lane = slot
      const uint64_t jb = sb > m ? sb : static_cast<uint64_t>(m);
      for (uint64_t b = jb; b < se; b += 32) {
        const uint64_t j = b + lane;
        uint32_t r = kInv;
        if (j < se) r = static_cast<uint32_t>(__umul64hi(draw(key, j - m + 1), j + 1));
        unsigned mask = __ballot_sync(kFull, j < se && r < m);
        while (mask) {
          const int src = __ffs(mask) - 1;
          const uint32_t slot = __shfl_sync(kFull, r, src);
          if (lane == static_cast<int>(slot)) last = static_cast<uint32_t>(b + src);
          mask &= mask - 1;
        }
      }
      a.hub.slot_last[static_cast<uint64_t>(s) * 32 + lane] = last;
      continue;
    }
    const BitmapWeight wf{&a};
    uint32_t* rid = a.hub.rec_id + static_cast<uint64_t>(s) * kRecCap;
    double* rkey = a.hub.rec_key + static_cast<uint64_t>(s) * kRecCap;
    const uint32_t nf = static_cast<uint32_t>(se - sb < m ? se - sb : m);
    WState st;
    fill_slots(nb, sb, nf, key, 0, lane, wf, st, FillEmit{rid, rkey, kRecCap});
    uint32_t cnt = nf;
    double tau = -1.0;
    if (se - sb >= m) {
      SegEmit em{rid, rkey, &cnt, kRecCap, lane};
      replay_range(nb, sb + m, se, key, 0, lane, wf, a.wmode != 0, a.gamma, st, em);
      tau = st.thr;
    }
    if (lane == 0) {
      a.hub.rec_cnt[s] = cnt;
      a.hub.tau[s] = tau;
    }
  }
}

constexpr int kMergeWarps = 8;

__global__ void __launch_bounds__(kMergeWarps * 32) k_hub_merge(SampleArgs a) {
  __shared__ uint32_t s_id[kMergeWarps][kRecCap];
  __shared__ double s_key[kMergeWarps][kRecCap];
  __shared__ uint32_t s_n[kMergeWarps];
  __shared__ double s_lrun;
  __shared__ int s_overflow;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nhub = min(*a.hub_count, a.hub.hub_cap);
  const uint32_t m = a.f;
  for (uint32_t h = blockIdx.x; h < nhub; h += gridDim.x) {
    const uint32_t ns = a.hub.nseg[h];
    if (ns == 0) continue;  // processed by k_sample_rows
    const uint32_t s0 = a.hub.seg0[h], k = a.hub.row[h];
    const uint32_t dst = a.front[k];
    const uint64_t beg = a.ro[dst], deg = a.ro[dst + 1] - beg;
    const uint32_t* nb = a.col + beg;
    const uint64_t key = hash2(a.seed, hash2(a.layer, dst));
    const uint64_t row0 = static_cast<uint64_t>(k) * m;
    if (a.kind == A3G_SAMPLER_UNIFORM) {
      if (warp == 0) {
        uint32_t my_id = lane < static_cast<int>(m) ? nb[lane] : 0u;
        for (int s = static_cast<int>(ns) - 1; s >= 0; --s) {
          const uint32_t last = a.hub.slot_last[static_cast<uint64_t>(s0 + s) * 32 + lane];
          if (last != kInv) {
            my_id = nb[last];
            break;
          }
        }
        if (lane < static_cast<int>(m)) {
          a.S[row0 + lane] = my_id;
          mark_first(a.first, my_id, a.tag, static_cast<uint32_t>(row0 + lane));
        }
        if (lane == 0) a.cnt[k] = m;
      }
      __syncthreads();
      continue;
    }
    if (threadIdx.x == 0) {
      s_lrun = -1.0;
      int of = 0;
      for (uint32_t s = 0; s < ns; ++s) of |= a.hub.rec_cnt[s0 + s] > kRecCap;
      s_overflow = of;
    }
    __syncthreads();
    if (s_overflow) {  // a segment's records overflowed: exact whole-row replay
      if (warp == 0) row_by_warp(a, nb, deg, key, k, lane);
      __syncthreads();
      continue;
    }
    // global fill = records 0..m-1 of segment 0 (positions 0..m-1)
    WState st;
    if (warp == 0) {
      const uint64_t rb = static_cast<uint64_t>(s0) * kRecCap;
      st.my_key = lane < static_cast<int>(m) ? a.hub.rec_key[rb + lane] : INFINITY;
      st.my_id = lane < static_cast<int>(m) ? a.hub.rec_id[rb + lane] : 0u;
      st.thr = st.my_key;
      st.mp = lane;
      warp_argmin(st.thr, st.mp);
    }
    for (uint32_t w0 = 0; w0 < ns; w0 += kMergeWarps) {
      // filter: records of segment s with key <= L_s = max_{s'<s} tau_s' are dropped
      const uint32_t s = w0 + warp;
      uint32_t n_keep = 0;
      if (s < ns) {
        double L = s_lrun;
        for (uint32_t t = w0; t < s; ++t) L = fmax(L, a.hub.tau[s0 + t]);
        const uint64_t rb = static_cast<uint64_t>(s0 + s) * kRecCap;
        const uint32_t rc = a.hub.rec_cnt[s0 + s];
        for (uint32_t i0 = (s == 0 ? m : 0); i0 < rc; i0 += 32) {
          const uint32_t i = i0 + lane;
          double kv = -1.0;
          uint32_t iv = 0;
          if (i < rc) {
            kv = a.hub.rec_key[rb + i];
            iv = a.hub.rec_id[rb + i];
          }
          const bool keep = i < rc && kv > L;
          const unsigned bm = __ballot_sync(kFull, keep);
          if (keep) {
            const uint32_t o = n_keep + __popc(bm & ((1u << lane) - 1u));
            s_id[warp][o] = iv;
            s_key[warp][o] = kv;
          }
          n_keep += __popc(bm);
        }
      }
      if (lane == 0) s_n[warp] = n_keep;
      __syncthreads();
      if (warp == 0) {
        for (int wr = 0; wr < kMergeWarps && w0 + wr < ns; ++wr) {
          const uint32_t n = s_n[wr];
          for (uint32_t i0 = 0; i0 < n; i0 += 32) {
            const uint32_t i = i0 + lane;
            const double kk = i < n ? s_key[wr][i] : -1.0;
            const uint32_t v = i < n ? s_id[wr][i] : 0u;
            unsigned mask = __ballot_sync(kFull, kk > st.thr);
            while (mask) {
              const int src = __ffs(mask) - 1;
              const double kv = __shfl_sync(kFull, kk, src);
              const uint32_t iv = __shfl_sync(kFull, v, src);
              if (lane == st.mp) {
                st.my_key = kv;
                st.my_id = iv;
              }
              st.thr = st.my_key;
              st.mp = lane;
              warp_argmin(st.thr, st.mp);
              mask &= __ballot_sync(kFull, kk > st.thr) & ~((2u << src) - 1u);
            }
          }
        }
        if (lane == 0) {
          double L = s_lrun;
          for (uint32_t t = w0; t < min(ns, w0 + kMergeWarps); ++t) L = fmax(L, a.hub.tau[s0 + t]);
          s_lrun = L;
        }
      }
      __syncthreads();
    }
    if (warp == 0) {
      if (lane < static_cast<int>(m)) {
        a.S[row0 + lane] = st.my_id;
        mark_first(a.first, st.my_id, a.tag, static_cast<uint32_t>(row0 + lane));
      }
      if (lane == 0) a.cnt[k] = m;
    }
    __syncthreads();
  }
}

// Test hook: one explicit neighbour list with arbitrary positive weights
// (sampler.hpp:50-56), single warp; rows with m > 32 run thread-serial.
__global__ void k_reservoir_list(const uint32_t* nb, const double* w, uint64_t deg, uint32_t m,
                                 uint64_t key, uint64_t c0, int kind, uint32_t* out, double* keys) {
  const int lane = threadIdx.x & 31;
  if (deg <= m) {
    for (uint64_t t = lane; t < deg; t += 32) out[t] = nb[t];
    return;
  }
  if (m <= 32) {
    uint32_t id;
    if (kind == A3G_SAMPLER_UNIFORM) {
      id = uniform_row_warp(nb, deg, m, key, lane, c0);
    } else {
      const ListWeight wf{w};
      id = weighted_row_warp(nb, deg, m, key, lane, wf, false, 1.0, c0);
    }
    if (lane < static_cast<int>(m)) out[lane] = id;
    return;
  }
  if (lane != 0) return;
  if (kind == A3G_SAMPLER_UNIFORM) {
    for (uint64_t j = 0; j < deg; ++j) {
      if (j < m) {
        out[j] = nb[j];
      } else {
        const uint64_t r = __umul64hi(draw(key, c0 + j - m + 1), j + 1);
        if (r < m) out[r] = nb[j];
      }
    }
    return;
  }
  uint32_t cnt = 0, mp = 0;
  for (uint64_t j = 0; j < deg; ++j) {
    const double u = unit_of(draw(key, c0 + j + 1));
    const double k = w[j] == 1.0 ? u : pow(u, 1.0 / w[j]);
    if (cnt < m) {
      out[cnt] = nb[j];
      keys[cnt] = k;
      ++cnt;
      if (k < keys[mp]) mp = cnt - 1;
    } else if (k > keys[mp]) {
      out[mp] = nb[j];
      keys[mp] = k;
      mp = 0;
      for (uint32_t t = 1; t < cnt; ++t)
        if (keys[t] < keys[mp]) mp = t;
    }
  }
}

// Seeds phase marking: every seed position p marks first[seed[p]].
__global__ void k_mark_list(const uint32_t* ids, uint32_t n, uint64_t* first, uint32_t tag) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x)
    mark_first(first, ids[p], tag, p);
}

__global__ void k_init_counters(BatchCounters* c, uint32_t n_seeds) {
  uint32_t* w = reinterpret_cast<uint32_t*>(c);
  for (uint32_t i = threadIdx.x; i < sizeof(BatchCounters) / 4; i += blockDim.x) w[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) c->n_seeds = n_seeds;
}

// ------------------------------------------------------------ finalize -----
constexpr int kFinThreads = 256;
constexpr int kFinRounds = 8;
constexpr int kFinTile = kFinThreads * kFinRounds;

struct FinArgs {
  const uint32_t* S;
  const uint32_t* cnt;  // nullptr: every position < nrows*f valid (seeds)
  const uint32_t* nrows;
  const uint64_t* first;
  uint64_t* gidx;
  uint4* blk;
  const uint32_t* uprev;  // nullptr -> 0
  uint32_t* unique;
  uint32_t* next_front;      // nullptr: last layer (frontier not needed)
  uint32_t* next_front_idx;
  int32_t* inv;              // layer-0 only: unique idx -> next-frontier row
  uint32_t* out_nfront;
  uint32_t* out_u;
  uint32_t* out_e;
  uint32_t f, tag, gtag;
};

struct Flags {
  bool valid, first, isnew;
  uint32_t v;
};

__device__ __forceinline__ Flags fin_flags(const FinArgs& a, uint64_t P, uint64_t p) {
  Flags fl{false, false, false, 0};
  if (p >= P) return fl;
  if (a.cnt) {
    const uint64_t row = p / a.f;
    const uint32_t slot = static_cast<uint32_t>(p - row * a.f);
    if (slot >= __ldg(a.cnt + row)) return fl;
  }
  fl.valid = true;
  fl.v = __ldg(a.S + p);
  const uint64_t want = (static_cast<uint64_t>(a.tag) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(p));
  fl.first = a.first[fl.v] == want;
  if (fl.first) fl.isnew = static_cast<uint32_t>(a.gidx[fl.v] >> 32) != a.gtag;
  return fl;
}

__global__ void __launch_bounds__(kFinThreads) k_fin_count(FinArgs a) {
  const uint64_t P = static_cast<uint64_t>(*a.nrows) * a.f;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kFinTile;
  if (base >= P) return;
  __shared__ uint32_t s_cnt[3];
  if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  uint32_t cv = 0, cf = 0, cn = 0;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < kFinRounds; ++r) {
    const Flags fl = fin_flags(a, P, base + r * kFinThreads + threadIdx.x);
    cv += __popc(__ballot_sync(kFull, fl.valid));
    cf += __popc(__ballot_sync(kFull, fl.first));
    cn += __popc(__ballot_sync(kFull, fl.isnew));
  }
  if (lane == 0) {
    atomicAdd(&s_cnt[0], cv);
    atomicAdd(&s_cnt[1], cf);
    atomicAdd(&s_cnt[2], cn);
  }
  __syncthreads();
  if (threadIdx.x == 0) a.blk[blockIdx.x] = make_uint4(s_cnt[0], s_cnt[1], s_cnt[2], 0);
}

__global__ void __launch_bounds__(kFinThreads) k_fin_emit(FinArgs a) {
  const uint64_t P = static_cast<uint64_t>(*a.nrows) * a.f;
  const uint32_t nblk = static_cast<uint32_t>((P + kFinTile - 1) / kFinTile);
  if (blockIdx.x >= nblk) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ uint32_t s_red[3][kFinThreads / 32];
  __shared__ uint32_t s_w[2][kFinThreads / 32];
  // exclusive prefix of the tile partials (and, for block 0, the totals)
  const uint32_t lim = blockIdx.x == 0 ? nblk : blockIdx.x;
  uint32_t pv = 0, pf = 0, pn = 0;
  for (uint32_t t = threadIdx.x; t < lim; t += kFinThreads) {
    const uint4 q = a.blk[t];
    pv += q.x;
    pf += q.y;
    pn += q.z;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    pv += __shfl_xor_sync(kFull, pv, off);
    pf += __shfl_xor_sync(kFull, pf, off);
    pn += __shfl_xor_sync(kFull, pn, off);
  }
  if (lane == 0) {
    s_red[0][warp] = pv;
    s_red[1][warp] = pf;
    s_red[2][warp] = pn;
  }
  __syncthreads();
  pv = pf = pn = 0;
  for (int w = 0; w < kFinThreads / 32; ++w) {
    pv += s_red[0][w];
    pf += s_red[1][w];
    pn += s_red[2][w];
  }
  const uint32_t uprev = a.uprev ? *a.uprev : 0u;
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      *a.out_e = pv;
      *a.out_nfront = pf;
      *a.out_u = uprev + pn;
    }
    pv = pf = pn = 0;  // block 0's own prefix is zero
  }
  __syncthreads();
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kFinTile;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t run_f = pf, run_n = pn;
  for (int r = 0; r < kFinRounds; ++r) {
    const Flags fl = fin_flags(a, P, base + r * kFinThreads + threadIdx.x);
    const unsigned bf = __ballot_sync(kFull, fl.first);
    const unsigned bn = __ballot_sync(kFull, fl.isnew);
    if (lane == 0) {
      s_w[0][warp] = __popc(bf);
      s_w[1][warp] = __popc(bn);
    }
    __syncthreads();
    uint32_t of = run_f, on = run_n, tf = 0, tn = 0;
    for (int w = 0; w < kFinThreads / 32; ++w) {
      if (w < warp) {
        of += s_w[0][w];
        on += s_w[1][w];
      }
      tf += s_w[0][w];
      tn += s_w[1][w];
    }
    if (fl.first) {
      const uint32_t nf = of + __popc(bf & lt);
      uint32_t idx;
      if (fl.isnew) {
        idx = uprev + on + __popc(bn & lt);
        a.unique[idx] = fl.v;
        a.gidx[fl.v] = (static_cast<uint64_t>(a.gtag) << 32) | idx;
      } else {
        idx = static_cast<uint32_t>(a.gidx[fl.v]);
      }
      if (a.next_front) {
        a.next_front[nf] = fl.v;
        a.next_front_idx[nf] = idx;
        if (a.inv) a.inv[idx] = static_cast<int32_t>(nf);
      }
    }
    run_f += tf;
    run_n += tn;
    __syncthreads();
  }
}

// srcidx of every valid slot of layer blockIdx.y.
struct ResolveArgs {
  const uint32_t* S[kMaxLayers];
  const uint32_t* cnt[kMaxLayers];
  uint32_t* sidx[kMaxLayers];
  const uint32_t* nrows[kMaxLayers];
  uint32_t f[kMaxLayers];
  const uint64_t* gidx;
};

__global__ void k_resolve(ResolveArgs a) {
  const int l = blockIdx.y;
  const uint32_t f = a.f[l];
  const uint64_t P = static_cast<uint64_t>(*a.nrows[l]) * f;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < P;
       p += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t row = p / f;
    if (p - row * f < a.cnt[l][row]) a.sidx[l][p] = static_cast<uint32_t>(a.gidx[a.S[l][p]]);
  }
}

// retrieve_features gather (cache.cpp:70-87): f32 rows, F contiguous.
template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) {
  return x;
}
template <>
__device__ __forceinline__ float to_f32<uint16_t>(uint16_t x) {
  return __uint_as_float(static_cast<uint32_t>(x) << 16);
}

template <typename T>
__global__ void k_gather_unique(const T* feat, uint32_t pitch, uint32_t F, const uint32_t* unique,
                                const uint32_t* ucount, const uint32_t* bits, int bitmode,
                                float* out, BatchCounters* ctr) {
  const uint32_t U = *ucount;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t hits = 0, seen = 0;
  for (uint32_t i = gw; i < U; i += nw) {
    const uint32_t v = unique[i];
    const T* src = feat + static_cast<uint64_t>(v) * pitch;
    float* dst = out + static_cast<uint64_t>(i) * F;
    for (uint32_t c = lane; c < F; c += 32) dst[c] = to_f32<T>(src[c]);
    if (lane == 0) {
      ++seen;
      const bool hit = bitmode == 1 || (bitmode == 2 && ((bits[v >> 5] >> (v & 31)) & 1u));
      hits += hit ? 1u : 0u;
    }
  }
  if (lane == 0 && seen) {
    atomicAdd(&ctr->hits, hits);
    atomicAdd(&ctr->misses, seen - hits);
  }
}

}  // namespace

// ------------------------------------------------------------ host side ----
void launch_sample(SamplerState& s, uint32_t n_seeds, double gamma, int kind, uint64_t rng_seed,
                   cudaStream_t st) {
  a3g_graph* g = s.g;
  a3g_cache* c = s.c;
  BatchCounters* ctr = s.d_ctr;
  k_init_counters<<<1, 64, 0, st>>>(ctr, n_seeds);
  A3G_LAUNCH_CHECK("k_init_counters");
  if (s.cap_inner) A3G_CUDA(cudaMemsetAsync(s.d_inv1, 0xff, s.cap_inner * sizeof(int32_t), st));
  ++s.gtag;
  // ---- seeds phase (sampler.cpp:100-105)
  const uint32_t tag0 = ++s.tag;
  k_mark_list<<<(n_seeds + 255) / 256, 256, 0, st>>>(s.d_seeds, n_seeds, s.d_first, tag0);
  A3G_LAUNCH_CHECK("k_mark_list");
  {
    FinArgs fa{};
    fa.S = s.d_seeds;
    fa.cnt = nullptr;
    fa.nrows = &ctr->n_seeds;
    fa.first = s.d_first;
    fa.gidx = s.d_gidx;
    fa.blk = s.d_blk;
    fa.uprev = nullptr;
    fa.unique = s.d_unique;
    fa.next_front = s.L ? s.layer[0].front : nullptr;
    fa.next_front_idx = s.L ? s.layer[0].front_idx : nullptr;
    fa.inv = nullptr;
    fa.out_nfront = &ctr->nfront[0];
    fa.out_u = &ctr->ucount[0];
    fa.out_e = &ctr->pad;  // seeds: valid count unused
    fa.f = 1;
    fa.tag = tag0;
    fa.gtag = s.gtag;
    const uint32_t nb = (n_seeds + kFinTile - 1) / kFinTile;
    k_fin_count<<<nb, kFinThreads, 0, st>>>(fa);
    k_fin_emit<<<nb, kFinThreads, 0, st>>>(fa);
    A3G_LAUNCH_CHECK("seed finalize");
  }
  // ---- layers (sampler.cpp:107-135)
  int wmode = 0;
  if (kind == A3G_SAMPLER_WEIGHTED && gamma != 1.0) {
    if (c->all_cached)
      wmode = 1;
    else if (!c->none_cached)
      wmode = 2;
  }
  const int sample_blocks = s.sm_count * 4;
  for (uint32_t l = 0; l < s.L; ++l) {
    LayerArena& la = s.layer[l];
    const uint32_t tag = ++s.tag;
    SampleArgs sa{};
    sa.ro = g->d_ro;
    sa.col = g->d_col;
    sa.bits = c->d_bits;
    sa.front = la.front;
    sa.nrows = &ctr->nfront[l];
    sa.cnt = la.cnt;
    sa.S = la.S;
    sa.first = s.d_first;
    sa.work = &ctr->work[l];
    sa.scratch = la.scratch;
    sa.hub = s.hub;
    sa.hub_count = &ctr->hubs[l];
    sa.seg_count = &ctr->segs[l];
    sa.seed = rng_seed;
    sa.gamma = gamma;
    sa.inv_gamma = 1.0 / gamma;
    sa.f = la.f;
    sa.layer = l;
    sa.tag = tag;
    sa.kind = kind;
    sa.wmode = wmode;
    k_sample_rows<<<sample_blocks, 256, 0, st>>>(sa);
    A3G_LAUNCH_CHECK("k_sample_rows");
    if (la.f <= 32) {
      k_hub_segments<<<s.sm_count * 8, 256, 0, st>>>(sa);
      A3G_LAUNCH_CHECK("k_hub_segments");
      k_hub_merge<<<s.sm_count * 2, kMergeWarps * 32, 0, st>>>(sa);
      A3G_LAUNCH_CHECK("k_hub_merge");
    }
    FinArgs fa{};
    fa.S = la.S;
    fa.cnt = la.cnt;
    fa.nrows = &ctr->nfront[l];
    fa.first = s.d_first;
    fa.gidx = s.d_gidx;
    fa.blk = s.d_blk;
    fa.uprev = &ctr->ucount[l];
    fa.unique = s.d_unique;
    fa.next_front = (l + 1 < s.L) ? s.layer[l + 1].front : nullptr;
    fa.next_front_idx = (l + 1 < s.L) ? s.layer[l + 1].front_idx : nullptr;
    fa.inv = (l == 0 && s.L >= 2) ? s.d_inv1 : nullptr;
    fa.out_nfront = &ctr->nfront[l + 1];
    fa.out_u = &ctr->ucount[l + 1];
    fa.out_e = &ctr->edges[l];
    fa.f = la.f;
    fa.tag = tag;
    fa.gtag = s.gtag;
    const uint32_t nb = static_cast<uint32_t>((la.cap_rows * la.f + kFinTile - 1) / kFinTile);
    k_fin_count<<<nb, kFinThreads, 0, st>>>(fa);
    k_fin_emit<<<nb, kFinThreads, 0, st>>>(fa);
    A3G_LAUNCH_CHECK("layer finalize");
  }
  if (s.L) {
    ResolveArgs ra{};
    for (uint32_t l = 0; l < s.L; ++l) {
      ra.S[l] = s.layer[l].S;
      ra.cnt[l] = s.layer[l].cnt;
      ra.sidx[l] = s.layer[l].sidx;
      ra.nrows[l] = &ctr->nfront[l];
      ra.f[l] = s.layer[l].f;
    }
    ra.gidx = s.d_gidx;
    k_resolve<<<dim3(s.sm_count * 2, s.L), 256, 0, st>>>(ra);
    A3G_LAUNCH_CHECK("k_resolve");
  }
}

void launch_gather_unique(SamplerState& s, float* out, cudaStream_t st) {
  a3g_graph* g = s.g;
  a3g_cache* c = s.c;
  const int bitmode = c->all_cached ? 1 : (c->none_cached ? 0 : 2);
  const uint32_t* uc = &s.d_ctr->ucount[s.L];
  if (g->feat_dtype == A3G_FEAT_BF16)
    k_gather_unique<uint16_t><<<s.sm_count * 4, 256, 0, st>>>(
        static_cast<const uint16_t*>(g->d_feat), g->pitch, g->F, s.d_unique, uc, c->d_bits, bitmode,
        out, s.d_ctr);
  else
    k_gather_unique<float><<<s.sm_count * 4, 256, 0, st>>>(static_cast<const float*>(g->d_feat),
                                                            g->pitch, g->F, s.d_unique, uc,
                                                            c->d_bits, bitmode, out, s.d_ctr);
  A3G_LAUNCH_CHECK("k_gather_unique");
}

void launch_reservoir_list(const uint32_t* d_nb, const double* d_w, uint64_t deg, uint32_t m,
                           uint64_t key, uint64_t c0, int kind, uint32_t* d_out, double* d_keys,
                           cudaStream_t st) {
  k_reservoir_list<<<1, 32, 0, st>>>(d_nb, d_w, deg, m, key, c0, kind, d_out, d_keys);
  A3G_LAUNCH_CHECK("k_reservoir_list");
}

}  // namespace a3g
