// reservoir.cuh -- warp-level exact replays of the reference reservoirs
// (proj/src/sampler.cpp:9-58) used by the sampler kernels.
//
// A reservoir of m <= 32 slots lives in one warp (slot = lane). Keys of 32
// neighbours are evaluated at once; a ballot of keys beating the current
// minimum selects the only positions that can be inserted; they are applied in
// neighbour order, each followed by a warp argmin (ties -> lowest slot, as
// std::min_element). This reproduces the sequential slot history exactly.
//
// Key policies (how keys are represented and compared):
//   PolUnit      all weights 1 (gamma == 1 or nothing cached): k = u exactly, so
//                keys compare as the 53-bit integers x >> 11 (no FP64 at all).
//   PolGammaAll  every neighbour cached: k = u^(1/gamma) is monotone in u, so
//                keys compare as integers too; only near-ties (within `tie`
//                integer ulps, where pow may round two u to one k) are decided
//                with the exact pow, like the reference (probability ~1e-15).
//   PolMixed     cached and uncached neighbours (bitmap), or explicit weights:
//                1-space doubles; a gamma-key is evaluated (pow) only when
//                u >= thr^gamma*(1-1e-6), below which pow(u,1/gamma) < thr for
//                any <= 2-ulp pow.
#pragma once

#include <cmath>

#include "a3g_internal.cuh"

namespace a3g {
namespace rsv {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kPrefetch = 4;  // 32-key chunks in flight per replay step

__device__ __forceinline__ double u_of(uint64_t k53) { return static_cast<double>(k53) * 0x1.0p-53; }

__device__ __forceinline__ void argmin_f64(double& k, int& idx) {
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
// Warp argmin of 64-bit order keys, ties -> lowest lane (std::min_element):
// two redux.sync.min.u32 (high then low word) + one ballot -- a short
// dependency chain instead of five rounds of 64-bit shuffles.
__device__ __forceinline__ void argmin_bits(uint64_t b, uint64_t& mn, int& mp) {
  const uint32_t hi = static_cast<uint32_t>(b >> 32), lo = static_cast<uint32_t>(b);
  const uint32_t mh = __reduce_min_sync(kFull, hi);
  const uint32_t ml = __reduce_min_sync(kFull, hi == mh ? lo : 0xffffffffu);
  mn = (static_cast<uint64_t>(mh) << 32) | ml;
  mp = __ffs(__ballot_sync(kFull, b == mn)) - 1;
}

__device__ __forceinline__ double gamma_lo(double thr, double gamma) {
  if (gamma > 1e8) return 0.0;
  return pow(thr, gamma) * (1.0 - 1e-6);
}

struct PolUnit {
  using K = uint64_t;
  static constexpr bool kNearTies = false;
  static constexpr uint64_t tie = 0;
  __device__ __forceinline__ K inf() const { return ~0ull; }
  __device__ __forceinline__ K fill_key(uint64_t x, uint32_t, uint64_t) const { return x >> 11; }
  __device__ __forceinline__ bool eval(uint64_t x, uint32_t, uint64_t, K thr, K& k) const {
    k = x >> 11;
    return k > thr;
  }
  __device__ __forceinline__ bool gt(K a, K b) const { return a > b; }
  __device__ __forceinline__ bool cheap_gt(K a, K b) const { return a > b; }
  __device__ __forceinline__ void on_thr(K) {}
  __device__ __forceinline__ void argmin(K& thr, int& mp, K my, int) const { argmin_bits(my, thr, mp); }
  // record filter of the hub merge: may a record with key k beat a minimum >= L?
  __device__ __forceinline__ bool keep(K k, K L) const { return k > L; }
};

struct PolGammaAll {
  using K = uint64_t;
  static constexpr bool kNearTies = true;
  double inv_g;
  uint64_t tie;
  __device__ __forceinline__ K inf() const { return ~0ull; }
  __device__ __forceinline__ K fill_key(uint64_t x, uint32_t, uint64_t) const { return x >> 11; }
  __device__ __forceinline__ bool eval(uint64_t x, uint32_t, uint64_t, K thr, K& k) const {
    k = x >> 11;
    return k > thr;
  }
  __device__ __forceinline__ bool gt(K a, K b) const {
    return a > b && (a - b > tie || pow(u_of(a), inv_g) > pow(u_of(b), inv_g));
  }
  __device__ __forceinline__ bool cheap_gt(K a, K b) const { return a > b; }
  __device__ __forceinline__ void on_thr(K) {}
  __device__ __forceinline__ void argmin(K& thr, int& mp, K my, int lane) const {
    argmin_bits(my, thr, mp);
    // another slot within `tie` of the minimum may hold an equal k: decide
    // with the exact keys (std::min_element semantics)
    if (__ballot_sync(kFull, my != ~0ull && my != thr && my - thr <= tie)) {
      double kf = my != ~0ull ? pow(u_of(my), inv_g) : INFINITY;
      int i = lane;
      argmin_f64(kf, i);
      mp = i;
      thr = __shfl_sync(kFull, my, i);
    }
  }
  __device__ __forceinline__ bool keep(K k, K L) const { return k + tie > L; }
};

// Weight of neighbour (v, j): assign_weights (sampler.cpp:60-68).
struct BitmapW {
  const uint32_t* bits;  // nullptr: every neighbour weighted gamma
  double inv_gamma;
  __device__ __forceinline__ bool unit(uint32_t v, uint64_t) const {
    return bits ? !((__ldg(bits + (v >> 5)) >> (v & 31)) & 1u) : false;
  }
  __device__ __forceinline__ double inv_w(uint32_t, uint64_t) const { return inv_gamma; }
};
struct ListW {  // explicit weights (test hook a3g_weighted_reservoir)
  const double* w;
  __device__ __forceinline__ bool unit(uint32_t, uint64_t j) const { return w[j] == 1.0; }
  __device__ __forceinline__ double inv_w(uint32_t, uint64_t j) const { return 1.0 / w[j]; }
};

template <typename WF>
struct PolMixed {
  using K = double;
  WF wf;
  bool use_filter;
  double gamma;
  double lo;
  __device__ __forceinline__ K inf() const { return INFINITY; }
  __device__ __forceinline__ K fill_key(uint64_t x, uint32_t v, uint64_t j) const {
    const double u = unit_of(x);
    return wf.unit(v, j) ? u : pow(u, wf.inv_w(v, j));
  }
  __device__ __forceinline__ bool eval(uint64_t x, uint32_t v, uint64_t j, K thr, K& k) const {
    const double u = unit_of(x);
    if (wf.unit(v, j)) {
      k = u;
    } else if (!use_filter || u >= lo) {
      k = pow(u, wf.inv_w(v, j));
    } else {
      return false;
    }
    return k > thr;
  }
  __device__ __forceinline__ bool gt(K a, K b) const { return a > b; }
  __device__ __forceinline__ bool cheap_gt(K a, K b) const { return a > b; }
  __device__ __forceinline__ void on_thr(K thr) {
    if (use_filter) lo = gamma_lo(thr, gamma);
  }
  __device__ __forceinline__ void argmin(K& thr, int& mp, K my, int) const {
    // keys are >= 0 (or +inf): their IEEE bit patterns order like the values
    uint64_t mn;
    argmin_bits(static_cast<uint64_t>(__double_as_longlong(my)), mn, mp);
    thr = __longlong_as_double(static_cast<long long>(mn));
  }
  __device__ __forceinline__ bool keep(K k, K L) const { return k > L; }
};

template <typename K>
struct WState {
  K my_key;
  uint32_t my_id;
  K thr;  // keys[min_pos]
  int mp; // min_pos
};

// Emit interface: (node id, key, lane holding it, row position). Hub-segment
// records store the position; the merge translates the final slots to ids.
struct NoEmit {
  template <typename K>
  __device__ __forceinline__ void operator()(uint32_t, K, int, uint64_t) const {}
};

// Fill slots [0, nf) with positions j0 + lane (sampler.cpp:30-33). The draw of
// position j is number c0 + j + 1 of stream `key` (rng.hpp:43-46).
template <typename P, typename Emit>
__device__ __forceinline__ void fill_slots(const uint32_t* nb, uint64_t j0, uint32_t nf, uint64_t key,
                                           uint64_t c0, int lane, const P& pol, WState<typename P::K>& s,
                                           const Emit& emit) {
  s.my_key = pol.inf();
  s.my_id = 0;
  if (lane < static_cast<int>(nf)) {
    const uint64_t j = j0 + lane;
    const uint32_t v = nb[j];
    s.my_key = pol.fill_key(mix64(key + (c0 + j + 1) * kPhi), v, j);
    s.my_id = v;
    emit(v, s.my_key, lane, j);
  }
  pol.argmin(s.thr, s.mp, s.my_key, lane);
}

// Replay positions [jb, je) against a full reservoir (sampler.cpp:34-39).
template <typename P, typename Emit>
__device__ __forceinline__ void replay_range(const uint32_t* nb, uint64_t jb, uint64_t je, uint64_t key,
                                             uint64_t c0, int lane, P& pol, WState<typename P::K>& s,
                                             const Emit& emit) {
  using K = typename P::K;
  pol.on_thr(s.thr);
  uint64_t ctr = key + (c0 + jb + lane + 1) * kPhi;  // stream position of lane's first key
  constexpr uint64_t kStep = 32ull * kPhi;
  for (uint64_t b = jb; b < je; b += 32 * kPrefetch, ctr += kPrefetch * kStep) {
    uint32_t v[kPrefetch];
    K kk[kPrefetch];
    bool cand[kPrefetch];
#pragma unroll
    for (int q = 0; q < kPrefetch; ++q) {
      const uint64_t j = b + q * 32 + lane;
      v[q] = j < je ? nb[j] : 0u;  // nb: global or a TMA-staged shared-memory piece
    }
#pragma unroll
    for (int q = 0; q < kPrefetch; ++q) {
      const uint64_t j = b + q * 32 + lane;
      cand[q] = j < je && pol.eval(mix64(ctr + q * kStep), v[q], j, s.thr, kk[q]);
    }
#pragma unroll
    for (int q = 0; q < kPrefetch; ++q) {
      unsigned mask = __ballot_sync(kFull, cand[q] && pol.cheap_gt(kk[q], s.thr));
      if (mask) {
        bool changed = false;
        while (mask) {
          const int src = __ffs(mask) - 1;
          const K kv = __shfl_sync(kFull, kk[q], src);
          const uint32_t iv = __shfl_sync(kFull, v[q], src);
          if (pol.gt(kv, s.thr)) {
            if (lane == s.mp) {
              s.my_key = kv;
              s.my_id = iv;
            }
            emit(iv, kv, src, b + q * 32 + src);
            pol.argmin(s.thr, s.mp, s.my_key, lane);
            changed = true;
            mask &= __ballot_sync(kFull, cand[q] && pol.cheap_gt(kk[q], s.thr));
          }
          mask &= ~((2u << src) - 1u);
        }
        if (changed) pol.on_thr(s.thr);
      }
    }
  }
}

// Weighted reservoir of a whole row by one warp (m <= 32 < deg).
template <typename P>
__device__ __forceinline__ uint32_t weighted_row_warp(const uint32_t* nb, uint64_t deg, uint32_t m, uint64_t key,
                                                      int lane, P& pol, uint64_t c0 = 0) {
  WState<typename P::K> s;
  fill_slots(nb, 0, m, key, c0, lane, pol, s, NoEmit{});
  replay_range(nb, m, deg, key, c0, lane, pol, s, NoEmit{});
  return s.my_id;
}

// Algorithm R (sampler.cpp:44-58) by one warp over positions [jb, je), jb >= m:
// slot r of position j is replaced iff r = next_below(j+1) < m (draw number
// c0 + j - m + 1); applied in position order.
__device__ __forceinline__ void uniform_range(const uint32_t* nb, uint64_t jb, uint64_t je, uint32_t m,
                                              uint64_t key, int lane, uint64_t c0, uint32_t& my_id) {
  for (uint64_t b = jb; b < je; b += 32) {
    const uint64_t j = b + lane;
    const bool valid = j < je;
    uint32_t r = kInv, v = 0;
    if (valid) {
      r = static_cast<uint32_t>(__umul64hi(draw(key, c0 + j - m + 1), j + 1));
      if (r < m) v = nb[j];
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

__device__ __forceinline__ uint32_t uniform_row_warp(const uint32_t* nb, uint64_t deg, uint32_t m, uint64_t key,
                                                     int lane, uint64_t c0 = 0) {
  uint32_t my_id = lane < static_cast<int>(m) ? nb[lane] : 0u;
  uniform_range(nb, m, deg, m, key, lane, c0, my_id);
  return my_id;
}

}  // namespace rsv
}  // namespace a3g
