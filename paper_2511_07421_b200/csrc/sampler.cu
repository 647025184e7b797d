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
//   k_classify      frontier rows -> work items: deg <= m rows are copied
//                   (fill only, sampler.cpp:30-33); m < deg <= seg rows are one
//                   item; deg > seg rows ("hubs", up to n-1 neighbours) are
//                   split into seg-long segment items + a merge entry in the
//                   small (<= 8 segments) or big hub work list.
//   k_item_class    items bucketed by length class (longest claimed first).
//   k_stream_grp    integer-key policies (all weights 1 or all gamma, and
//                   Algorithm R): lane groups of next_pow2(m) lanes, one item
//                   per group, keys hashed from positions only; candidates
//                   replayed in order per group (exact slot history).
//   k_stream_grp_mixed  bitmap-weighted keys (partial cache, gamma > 1): the
//                   same lane groups with fp64 keys (the neighbour id of every
//                   position decides its weight).
//   segments        replay locally from an empty reservoir, emitting every
//                   local insertion ("record", row position + key) and the
//                   segment's exact m-th largest key tau_s: every global
//                   insertion is a local record of its segment.
//   k_hub_merge     big hubs: block per hub, parallel filter of all records
//                   against L_s = max_{s'<s} tau_{s'} (a lower bound of the
//                   running minimum), then an exact replay of the survivors;
//                   small hubs: warp per hub, claimed dynamically.
//   k_fin_count / k_fin_emit: first-seen dedup + relabel (tagged atomicMax of
//                   the first position, tile partials, ballot scans).
// Counts stay on the device: no host sync inside a batch.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include <cub/device/device_radix_sort.cuh>

#include "ptx.cuh"
#include "reservoir.cuh"
#include "sampler.cuh"

namespace a3g {
namespace {

using rsv::kFull;
constexpr int kRowChunk = 4;  // rows claimed per atomic by a warp
constexpr uint32_t kMergeFilterWarpsC = 8;  // hub size class boundary (== kMergeFilterWarps)

__device__ __forceinline__ void mark_first(uint64_t* first, uint32_t v, uint32_t tag, uint32_t pos) {
  atomicMax(reinterpret_cast<unsigned long long*>(first + v),
            (static_cast<unsigned long long>(tag) << 32) | static_cast<unsigned long long>(~pos));
}

struct SampleArgs {
  const uint64_t* ro;
  const uint32_t* col;
  const uint32_t* bits;
  const uint32_t* ebits;  // per-edge cached bits (partial caches), or null
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
  uint32_t* big_count;    // hubs with > kMergeFilterWarps segments (k_hub_merge)
  uint32_t* cls_count;    // [8] stream items per length class (k_item_class)
  uint32_t* small_count;  // hubs with 1..kMergeFilterWarps segments (merge_small_hub)
  uint32_t* item_count;
  uint32_t* item_work;
  unsigned long long* positions;  // BatchCounters::positions
  uint64_t seed;
  double gamma, inv_gamma;
  uint64_t tie;
  uint32_t f, layer, tag;
  uint32_t seg;  // hub segment length (SamplerState::seg)
  int split_cls;  // >= 0: items of length class >= split_cls go to the lane-group kernel, the rest lane-per-item
  int kind;   // A3G_SAMPLER_*
  int wmode;  // 0: all weights 1; 1: all gamma; 2: bitmap
};

// Prefilter word of mix64(c) (rng.hpp:13-20) for the hot stream loops: the
// high word h4 of the second product, before the final z ^= z >> 31, so that
// x_hi = mix64(c) >> 32 is h4 or h4 ^ 1 and x_hi >= t implies h4 >= t - 1.
// The second multiply forms only its high word. ~9 alu + ~6 fma instructions
// per position instead of ~19 alu + 8 fma for the full 64-bit mix64; measured
// 1.37 vs 1.01 Tpositions/s on a B200 (tools/microbench/hash_pipes.cu).
__device__ __forceinline__ uint32_t mix64_pre(uint64_t c, uint32_t& l3) {
  const uint32_t lo = static_cast<uint32_t>(c), hi = static_cast<uint32_t>(c >> 32);
  const uint32_t l1 = lo ^ __funnelshift_r(lo, hi, 30);
  const uint32_t h1 = hi ^ (hi >> 30);
  const uint64_t w = static_cast<uint64_t>(l1) * 0x1ce4e5b9u;
  const uint32_t h2 = static_cast<uint32_t>(w >> 32) + l1 * 0xbf58476du + h1 * 0x1ce4e5b9u;
  const uint32_t l2 = static_cast<uint32_t>(w);
  l3 = l2 ^ __funnelshift_r(l2, h2, 27);
  const uint32_t h3 = h2 ^ (h2 >> 27);
  return __umulhi(l3, 0x133111ebu) + l3 * 0x94d049bbu + h3 * 0x133111ebu;
}
// the full draw from the prefilter state (h4, l3): == mix64(c) >> 11
__device__ __forceinline__ uint64_t mix64_finish_key(uint32_t h4, uint32_t l3) {
  const uint64_t z = (static_cast<uint64_t>(h4) << 32) | (l3 * 0x133111ebu);
  return (z ^ (z >> 31)) >> 11;
}
// High-word bound of unit keys u >= lo: u = (x >> 11) 2^-53 >= lo needs
// x >> 11 >= ceil(lo 2^53), hence x_hi >= ceil(lo 2^53) >> 21.
__device__ __forceinline__ uint32_t lo_hi_word(double lo) {
  if (!(lo > 0.0)) return 0u;
  if (lo >= 1.0) return 0xffffffffu;
  return static_cast<uint32_t>(static_cast<uint64_t>(ceil(lo * 0x1.0p53)) >> 21);
}
// prefilter bound for x_hi >= t
__device__ __forceinline__ uint32_t pre_bound(uint32_t t) { return t ? t - 1u : 0u; }


// Key policy of a launch (template dispatch on wmode).
template <int WM>
struct PolOf;
template <>
struct PolOf<0> {
  using P = rsv::PolUnit;
  __device__ static P make(const SampleArgs&) { return P{}; }
};
template <>
struct PolOf<1> {
  using P = rsv::PolGammaAll;
  __device__ static P make(const SampleArgs& a) { return P{a.inv_gamma, a.tie}; }
};
template <>
struct PolOf<2> {
  using P = rsv::PolMixed<rsv::BitmapW>;
  __device__ static P make(const SampleArgs& a) { return P{rsv::BitmapW{a.bits, a.inv_gamma}, true, a.gamma, 0.0}; }
};

__device__ __forceinline__ bool is_gamma(const SampleArgs& a, uint32_t v) {
  return a.wmode == 1 || (a.wmode == 2 && ((__ldg(a.bits + (v >> 5)) >> (v & 31)) & 1u));
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
template <int WM>
__device__ __forceinline__ void row_by_warp(const SampleArgs& a, const uint32_t* nb, uint64_t deg, uint64_t key,
                                            uint32_t k, int lane) {
  const uint32_t m = a.f;
  uint32_t my_id;
  if (a.kind == A3G_SAMPLER_UNIFORM) {
    my_id = rsv::uniform_row_warp(nb, deg, m, key, lane);
  } else {
    auto pol = PolOf<WM>::make(a);
    my_id = rsv::weighted_row_warp(nb, deg, m, key, lane, pol);
  }
  const uint64_t row0 = static_cast<uint64_t>(k) * m;
  if (lane < static_cast<int>(m)) {
    a.S[row0 + lane] = my_id;
    mark_first(a.first, my_id, a.tag, static_cast<uint32_t>(row0 + lane));
  }
  if (lane == 0) a.cnt[k] = m;
}

// Records of a segment's local replay: every local insertion (id, key bits).
template <typename K>
struct SegEmit {
  uint32_t* rid;
  uint64_t* rkey;
  uint32_t* cnt;  // warp-uniform counter
  uint32_t cap;
  int lane;
  __device__ __forceinline__ void operator()(uint32_t, K key, int src, uint64_t pos) const {
    const uint32_t c = *cnt;
    if (lane == src && c < cap) {
      rid[c] = static_cast<uint32_t>(pos);
      rkey[c] = *reinterpret_cast<const uint64_t*>(&key);
    }
    *cnt = c + 1;
  }
};
template <typename K>
struct FillEmit {  // fills: lane i writes record i
  uint32_t* rid;
  uint64_t* rkey;
  __device__ __forceinline__ void operator()(uint32_t, K key, int lane, uint64_t pos) const {
    rid[lane] = static_cast<uint32_t>(pos);
    rkey[lane] = *reinterpret_cast<const uint64_t*>(&key);
  }
};

template <typename K>
__device__ __forceinline__ K key_from_bits(uint64_t b) {
  return *reinterpret_cast<const K*>(&b);
}

// Classification of a layer's frontier rows, warp per 32 rows (lane = row):
//   deg == 0           no edges, no draws (sampler.cpp:116)
//   deg <= m           fill only: output = neighbour list (sampler.cpp:30-33)
//   m > 32 < deg       thread-serial exact replay (rare wide fanouts)
//   m < deg <= seg     one stream item (whole row)
//   deg > seg          hub: ceil(deg/seg) segment items + a merge entry
// Items are appended with one warp-aggregated atomic.
template <int WM>
__global__ void __launch_bounds__(256) k_classify(SampleArgs a) {
  const int lane = threadIdx.x & 31;
  const uint32_t nrows = *a.nrows;
  const uint32_t m = a.f;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r0 = gw * 32; r0 < nrows; r0 += nw * 32) {
    const uint32_t k = r0 + lane;
    const bool valid = k < nrows;
    uint32_t dst = 0;
    uint64_t beg = 0, deg = 0;
    if (valid) {
      dst = __ldg(a.front + k);
      beg = __ldg(a.ro + dst);
      deg = __ldg(a.ro + dst + 1) - beg;
    }
    const uint64_t row0 = static_cast<uint64_t>(k) * m;
    // ---- fill-only rows, copied cooperatively
    unsigned cm = __ballot_sync(kFull, valid && deg <= m);
    while (cm) {
      const int src = __ffs(cm) - 1;
      cm &= cm - 1;
      const uint64_t sb = __shfl_sync(kFull, beg, src);
      const uint32_t sd = static_cast<uint32_t>(__shfl_sync(kFull, deg, src));
      const uint64_t sr0 = static_cast<uint64_t>(r0 + src) * m;
      for (uint32_t t = lane; t < sd; t += 32) {
        const uint32_t v = __ldg(a.col + sb + t);
        a.S[sr0 + t] = v;
        mark_first(a.first, v, a.tag, static_cast<uint32_t>(sr0 + t));
      }
    }
    if (valid && deg <= m) a.cnt[k] = static_cast<uint32_t>(deg);
    uint32_t n_items = 0, h = kInv, s0 = 0, nseg = 0;
    if (valid && deg > m) {
      if (m > 32) {  // wide fanout: exact serial replay by this thread
        serial_row(a, a.col + beg, deg, hash2(a.seed, hash2(a.layer, dst)), a.S + row0, a.scratch + row0);
        for (uint32_t t = 0; t < m; ++t) mark_first(a.first, a.S[row0 + t], a.tag, static_cast<uint32_t>(row0 + t));
        a.cnt[k] = m;
      } else if (deg > a.seg) {
        nseg = static_cast<uint32_t>((deg + a.seg - 1) / a.seg);
        h = atomicAdd(a.hub_count, 1u);
        s0 = atomicAdd(a.seg_count, nseg);
        const bool ok = h < a.hub.hub_cap && s0 + static_cast<uint64_t>(nseg) <= a.hub.seg_cap;
        if (h < a.hub.hub_cap) {
          a.hub.row[h] = k;
          a.hub.seg0[h] = s0;
          a.hub.nseg[h] = ok ? nseg : 0u;  // 0: streamed as one whole-row item instead
        }
        if (ok) {
          // per size class work lists of the two merge kernels
          if (nseg > kMergeFilterWarpsC)
            a.hub.big[atomicAdd(a.big_count, 1u)] = h;
          else
            a.hub.small[atomicAdd(a.small_count, 1u)] = h;
          for (uint32_t i = 0; i < nseg; ++i) a.hub.seg_hub[s0 + i] = h;
          n_items = nseg;
        } else {
          h = kInv;
          n_items = 1;
        }
      } else {
        n_items = 1;
      }
    }
    // draws of the batch: one per neighbour of every frontier row (sampler.cpp:22-27, the
    // reference draws fill keys too; the device hashes only rows past their fill)
    unsigned long long hp = valid ? deg : 0ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) hp += __shfl_xor_sync(kFull, hp, off);
    if (lane == 0 && hp) atomicAdd(a.positions, hp);
    // ---- warp-aggregated append of the items
    uint32_t incl = n_items;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, off);
      if (lane >= off) incl += y;
    }
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    uint32_t base = 0;
    if (lane == 0 && total) base = atomicAdd(a.item_count, total);
    base = __shfl_sync(kFull, base, 0);
    uint32_t o = base + incl - n_items;
    if (h != kInv) {
      for (uint32_t i = 0; i < nseg; ++i, ++o) {
        const uint32_t sb = i * a.seg;
        const uint32_t se = static_cast<uint32_t>(deg < sb + static_cast<uint64_t>(a.seg) ? deg : sb + a.seg);
        if (o < a.hub.item_cap) a.hub.items[o] = make_uint4(k, sb, se, s0 + i);
      }
    } else if (n_items == 1) {
      if (o < a.hub.item_cap) a.hub.items[o] = make_uint4(k, 0, static_cast<uint32_t>(deg), kInv);
    }
  }
}

// Length classes of the layer's items (class k: lengths in [2^(k+5), 2^(k+6)),
// 0 below 64, 7 from 4096): per-class index lists built with warp-aggregated
// atomics. The lane-group stream kernels claim items longest class first, so
// a warp's groups carry items within 2x of each other's length.
constexpr int kClasses = kLenClasses;

__device__ __forceinline__ uint32_t len_class(uint32_t len) {
  const int l2 = 31 - __clz(max(len, 1u));
  if constexpr (kClasses == 8) {
    return static_cast<uint32_t>(min(max(l2 - 5, 0), kClasses - 1));
  } else {
    // quarter octaves from 32: class 4 (l2 - 5) + the two bits below the leading one
    const int q = l2 >= 2 ? static_cast<int>((len >> (l2 - 2)) & 3u) : 0;
    return static_cast<uint32_t>(min(max(4 * (l2 - 5) + q, 0), kClasses - 1));
  }
}

__global__ void k_item_class(const uint4* items, const uint32_t* item_count, uint32_t cap, uint32_t* lists,
                             uint32_t* cls_count) {
  const uint32_t n = min(*item_count, cap);
  const int lane = threadIdx.x & 31;
  for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x) {
    const uint32_t i = i0 + threadIdx.x;
    const bool ok = i < n;
    const unsigned act = __ballot_sync(kFull, ok);
    if (!ok) continue;
    const uint4 it = items[i];
    const uint32_t c = len_class(it.z - it.y);
    const unsigned peers = __match_any_sync(act, c);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(cls_count + c, __popc(peers));
    base = __shfl_sync(peers, base, leader);
    lists[static_cast<uint64_t>(c) * cap + base + __popc(peers & ((1u << lane) - 1u))] = i;
  }
}

// Item of claim index ii: classes walked from the longest down.
__device__ __forceinline__ uint32_t item_of(const uint32_t* lists, const uint32_t* cls_count, uint32_t cap,
                                            uint32_t ii) {
  for (int c = kClasses - 1; c > 0; --c) {
    const uint32_t n = cls_count[c];
    if (ii < n) return lists[static_cast<uint64_t>(c) * cap + ii];
    ii -= n;
  }
  return lists[ii];
}

// Items in the length classes >= c0 (they come first in claim order).
__device__ __forceinline__ uint32_t items_from_class(const uint32_t* cls_count, int c0) {
  uint32_t n = 0;
  for (int c = kClasses - 1; c >= c0; --c) n += cls_count[c];
  return n;
}

// ----------------------------------------------------------- stream (group) -
// Integer-key items (PolUnit / PolGammaAll weights, Algorithm R) processed by
// lane groups of G = next_pow2(m) lanes: a warp carries 32/G items at once,
// each group owning one item's reservoir (slot = lane in group). A key
// depends only on (row key, position), so the hot loop hashes positions
// without reading the adjacency: lane g hashes positions b + u*G + g for
// u < 32/G (independent mix64 chains), and one vote tells whether any group
// holds a key above its minimum (x > (thr << 11 | 0x7ff) <=> x >> 11 > thr).
// Candidates are then replayed in position order in every group at once --
// per step one insertion per group, with a G-lane butterfly argmin (first
// minimum, as std::min_element) -- the exact sequential slot history of
// sampler.cpp:24-40. Items are length-sorted so a warp's groups carry equal
// work; records of hub segments store row positions (the merge translates).
// (key, slot) minimum over the G lanes of a group, first index on K-ties.
template <int G, typename P, bool DBL = false>
__device__ __forceinline__ void grp_argmin(const P& pol, uint64_t my, uint32_t gl, uint64_t& thr, uint32_t& mp) {
  // fast path: butterfly on a packed 32-bit (27-bit key bucket, 5-bit slot) --
  // one 32-bit shuffle + min per step. Buckets are key * 2^27 in u-space
  // (53-bit integer keys >> 26; fp64 keys in [0,1] scaled by 2^27, exact and
  // monotone; the empty-slot sentinels clamp to the top bucket), so
  // bucket order is key order except within a bucket; every K-tie window
  // (<= 64 (gamma + 1) integer units) spans at most two adjacent buckets. The
  // packed minimum is therefore exact unless another slot sits in the
  // minimum's bucket or the next one -- then the exact 64-bit K-order decides
  // (first slot on K-ties, as std::min_element).
  uint32_t my27;
  if (DBL) {
    const double d = __longlong_as_double(static_cast<long long>(my));
    my27 = d >= 1.0 ? 0x7ffffffu : static_cast<uint32_t>(d * 0x1.0p27);
  } else {
    my27 = (my >> 26) < 0x7ffffffull ? static_cast<uint32_t>(my >> 26) : 0x7ffffffu;
  }
  uint32_t pk = (my27 << 5) | gl;
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) pk = min(pk, __shfl_xor_sync(kFull, pk, off, G));
  const uint32_t m27 = pk >> 5;
  uint32_t i = pk & 31u;
  uint64_t k = __shfl_sync(kFull, my, static_cast<int>(i), G);
  if (__any_sync(kFull, gl != i && my27 - m27 <= 1u)) {
    // exact pass: first slot whose K equals the minimum's K
    uint64_t kk = my;
    uint32_t ii = gl;
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
      const uint64_t ok = __shfl_xor_sync(kFull, kk, off, G);
      const uint32_t oi = __shfl_xor_sync(kFull, ii, off, G);
      if (pol.gt(kk, ok) || (!pol.gt(ok, kk) && oi < ii)) {
        kk = ok;
        ii = oi;
      }
    }
    k = kk;
    i = ii;
  }
  thr = k;
  mp = i;
}

template <int WM, int G>
__global__ void __launch_bounds__(256) k_stream_grp(SampleArgs a, const uint32_t* lists, const uint32_t* cls_count) {
  using P = typename PolOf<WM>::P;
  constexpr int NG = 32 / G;
  constexpr uint64_t kStepG = static_cast<uint64_t>(G) * kPhi;
  const int lane = threadIdx.x & 31;
  const uint32_t gl = lane % G, grp = lane / G;
  const unsigned gmask = G == 32 ? kFull : (((1u << G) - 1u) << (grp * G));
  uint32_t nitems = min(*a.item_count, a.hub.item_cap);
  if (a.split_cls >= 0) nitems = min(nitems, items_from_class(cls_count, a.split_cls));
  const uint32_t m = a.f;
  const P pol = PolOf<WM>::make(a);
  const uint32_t wstride = gridDim.x * (blockDim.x >> 5) * NG;
  for (uint32_t base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NG; base < nitems; base += wstride) {
    const uint32_t ii = base + grp;
    const bool live = ii < nitems;
    uint4 im = make_uint4(0, 0, 0, kInv);
    uint32_t dst = 0;
    uint64_t beg = 0;
    if (live) {
      im = a.hub.items[item_of(lists, cls_count, a.hub.item_cap, ii)];
      dst = __ldg(a.front + im.x);
      beg = __ldg(a.ro + dst);
    }
    const uint32_t* nb = a.col + beg;
    const uint64_t key = hash2(a.seed, hash2(a.layer, dst));
    const bool seg = im.w != kInv;
    const uint64_t row0 = static_cast<uint64_t>(im.x) * m;
    const uint32_t p0 = im.y, p1 = im.z;
    if (a.kind == A3G_SAMPLER_UNIFORM) {  // Algorithm R (sampler.cpp:44-58)
      uint32_t my_pos = seg ? kInv : gl;
      const uint32_t j0 = p0 > m ? p0 : m;
      // all groups iterate to the warp's longest item
      uint32_t len = live && p1 > j0 ? p1 - j0 : 0u;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) len = max(len, __shfl_xor_sync(kFull, len, off));
      for (uint32_t b = 0; b < len; b += G) {
        const uint32_t j = j0 + b + gl;
        uint32_t r = kInv;
        if (live && j < p1) r = static_cast<uint32_t>(__umul64hi(draw(key, j - m + 1), static_cast<uint64_t>(j) + 1));
        unsigned mask = __ballot_sync(kFull, r < m) & gmask;
        while (__any_sync(kFull, mask != 0)) {
          const int src = mask ? __ffs(mask) - 1 : lane;
          const uint32_t slot = __shfl_sync(kFull, r, src);
          if (mask && gl == slot) my_pos = j0 + b + (src % G);
          if (mask) mask &= mask - 1;
        }
      }
      if (live) {
        if (seg) {
          a.hub.slot_last[static_cast<uint64_t>(im.w) * 32 + gl] = gl < m ? my_pos : kInv;
          if (G < 32)
            for (uint32_t s2 = G + gl; s2 < 32; s2 += G) a.hub.slot_last[static_cast<uint64_t>(im.w) * 32 + s2] = kInv;
        } else if (gl < m) {
          const uint32_t id = __ldg(nb + my_pos);
          a.S[row0 + gl] = id;
          mark_first(a.first, id, a.tag, static_cast<uint32_t>(row0 + gl));
          if (gl == 0) a.cnt[im.x] = m;
        }
      }
      continue;
    }
    // ---- weighted reservoir, integer keys: fill
    const uint32_t nf = live ? min(m, p1 - p0) : 0u;
    uint64_t my_key = ~0ull;
    uint32_t my_pos = 0;
    uint32_t* rid = a.hub.rec_id + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    uint64_t* rkey = a.hub.rec_key + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    if (gl < nf) {
      my_key = draw(key, static_cast<uint64_t>(p0) + gl + 1) >> 11;
      my_pos = p0 + gl;
      if (seg) {
        rid[gl] = my_pos;
        rkey[gl] = my_key;
      }
    }
    uint64_t thr;
    uint32_t mp;
    grp_argmin<G>(pol, my_key, gl, thr, mp);
    uint32_t rcnt = nf;
    // ---- replay positions [p0 + nf, p1): lane g hashes b + u*G + g, u < 32/G;
    // candidates are replayed block by block (u), one insertion per group per
    // step (r01 measurements: cheaper than one 32-bit group mask over all u)
    constexpr int U = 32 / G;
    const uint32_t jb = p0 + nf;
    uint32_t len = live && p1 > jb ? p1 - jb : 0u;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) len = max(len, __shfl_xor_sync(kFull, len, off));
    // filter on the high key word: x > thr << 11 | 0x7ff needs x_hi >= thr >> 21
    // (a superset; the rare equal-high-word false positives fail the exact
    // test below, which finishes the full draw for the candidates only)
    uint32_t thi = pre_bound(static_cast<uint32_t>(thr >> 21));
    uint64_t ctr = key + (static_cast<uint64_t>(jb) + gl + 1) * kPhi;
    for (uint32_t b = 0; b < len; b += 32, ctr += 32 * kPhi) {
      const uint32_t q = jb + b + gl;
      const uint32_t rem = live && q < p1 ? p1 - q : 0u;
      bool c[U];
      uint32_t h4[U], l3[U];
      bool anyc = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        h4[u] = mix64_pre(ctr + u * kStepG, l3[u]);  // unconditional: no branch
        c[u] = (static_cast<uint32_t>(u * G) < rem) & (h4[u] >= thi);
        anyc |= c[u];
      }
      if (!__any_sync(kFull, anyc)) continue;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!__any_sync(kFull, c[u])) continue;
        const uint64_t kk = c[u] ? mix64_finish_key(h4[u], l3[u]) : 0ull;
        const bool cu = c[u] && kk > thr;
        unsigned mask = __ballot_sync(kFull, cu) & gmask;
        while (__any_sync(kFull, mask != 0)) {
          const int src = mask ? __ffs(mask) - 1 : lane;
          const uint64_t kv = __shfl_sync(kFull, kk, src);
          const bool ins = mask != 0 && pol.gt(kv, thr);
          const uint32_t pos = jb + b + u * G + (static_cast<uint32_t>(src) % G);
          if (ins && gl == mp) {
            my_key = kv;
            my_pos = pos;
          }
          if (ins && seg && lane == src) {
            if (rcnt < kRecCap) {
              rid[rcnt] = pos;
              rkey[rcnt] = kv;
            }
          }
          if (ins) ++rcnt;
          uint64_t nthr;
          uint32_t nmp;
          grp_argmin<G>(pol, my_key, gl, nthr, nmp);
          if (ins) {
            thr = nthr;
            mp = nmp;
          }
          if (mask) mask &= ~((2u << src) - 1u);
          mask &= __ballot_sync(kFull, cu && kk > thr) & gmask;
        }
      }
      thi = pre_bound(static_cast<uint32_t>(thr >> 21));
    }
    if (!live) continue;
    if (seg) {
      if (gl == 0) {
        a.hub.rec_cnt[im.w] = rcnt;
        a.hub.tau[im.w] = thr;
        a.hub.tau_ok[im.w] = (p1 - p0 >= m) ? 1u : 0u;
      }
    } else if (gl < m) {
      const uint32_t id = __ldg(nb + my_pos);
      a.S[row0 + gl] = id;
      mark_first(a.first, id, a.tag, static_cast<uint32_t>(row0 + gl));
      if (gl == 0) a.cnt[im.x] = m;
    }
  }
}

// Lane-per-item stream for wide layers (integer-key policies, m <= MB): each
// lane owns one item with its reservoir in registers (MB fully unrolled
// slots), hashes positions in chunks of 32 into a candidate bitmask with the
// prefilter, then replays its candidates exactly in position order -- all
// lanes in lockstep, one candidate per lane per step. Against the lane-group
// kernel this spends one lane (not G) per item on hashing and serves 32 items
// (not 32/G) per replay step; it needs many items to fill the machine, so the
// host selects it by the layer's frontier bound.
// K of an integer key under PolGammaAll (out of line: rare near-tie path)
__device__ __noinline__ double key_pow(uint64_t x, double inv_g) { return pow(rsv::u_of(x), inv_g); }

template <int MB, typename P>
__device__ __forceinline__ void lane_argmin(const P& pol, const uint64_t (&rk)[MB], uint32_t m, uint64_t& thr,
                                            uint32_t& mp) {
  uint64_t mn = rk[0];
  uint32_t mi = 0;
#pragma unroll
  for (int i = 1; i < MB; ++i)
    if (rk[i] < mn) {  // strict: first slot on equal integers
      mn = rk[i];
      mi = i;
    }
  if constexpr (P::kNearTies) {  // another slot within the tie window may hold an equal K
    bool near = false;
#pragma unroll
    for (int i = 0; i < MB; ++i) near |= static_cast<uint32_t>(i) != mi && rk[i] != ~0ull && rk[i] - mn <= pol.tie;
    if (near) {  // exact K-order, first slot on K-ties (std::min_element)
      double bk = key_pow(rk[0], pol.inv_g);
      mn = rk[0];
      mi = 0;
#pragma unroll
      for (int i = 1; i < MB; ++i)
        if (rk[i] != ~0ull) {
          const double ki = key_pow(rk[i], pol.inv_g);
          if (ki < bk) {
            bk = ki;
            mn = rk[i];
            mi = i;
          }
        }
    }
  }
  thr = mn;
  mp = mi;
}

#ifndef A3G_LANE_FUSED
#define A3G_LANE_FUSED 1
#endif
// A3G_LANE_FUSED=1 variant: the slot update fused with the argmin on the
// 32-bit key words hk = k >> 21; exact unless another slot's word is within
// `win` of the minimum's (then lane_argmin decides).
template <int MB, typename P>
__device__ __forceinline__ void lane_insert(const P& pol, uint64_t (&rk)[MB], uint32_t (&hk)[MB],
                                            uint32_t (&rp)[MB], uint32_t m, uint32_t mp_in, uint64_t kx,
                                            uint32_t pos, uint32_t win, uint64_t& thr, uint32_t& mp) {
  const uint32_t hx = static_cast<uint32_t>(kx >> 21);
  uint32_t mnh = 0xffffffffu, mi = 0;
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    if (static_cast<uint32_t>(i) == mp_in) {
      rk[i] = kx;
      hk[i] = hx;
      rp[i] = pos;
    }
    if (hk[i] < mnh) {
      mnh = hk[i];
      mi = i;
    }
  }
  bool near = false;
#pragma unroll
  for (int i = 0; i < MB; ++i) near |= static_cast<uint32_t>(i) != mi && hk[i] - mnh <= win;
  if (near) {
    lane_argmin<MB>(pol, rk, m, thr, mp);
  } else {
    mp = mi;
    uint64_t t = rk[0];
#pragma unroll
    for (int i = 1; i < MB; ++i)
      if (static_cast<uint32_t>(i) == mi) t = rk[i];
    thr = t;
  }
}

template <int WM, int MB>
__global__ void __launch_bounds__(256) k_stream_lane(SampleArgs a, const uint32_t* lists, const uint32_t* cls_count) {
  using P = typename PolOf<WM>::P;
  const int lane = threadIdx.x & 31;
  const uint32_t nitems = min(*a.item_count, a.hub.item_cap);
  const uint32_t m = a.f;
  const P pol = PolOf<WM>::make(a);
  // grid sized to the layer's item bound: one batch of 32 items per warp
  // (short-lived CTAs let the high-priority compute stream's kernels in)
  const uint32_t wstride = gridDim.x * (blockDim.x >> 5) * 32;
  const uint32_t ibase = a.split_cls >= 0 ? items_from_class(cls_count, a.split_cls) : 0u;
  for (uint32_t base = ibase + (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < nitems;
       base += wstride) {
    const uint32_t ii = base + lane;
    const bool live = ii < nitems;
    uint4 im = make_uint4(0, 0, 0, kInv);
    uint32_t dst = 0;
    uint64_t beg = 0;
    if (live) {
      im = a.hub.items[item_of(lists, cls_count, a.hub.item_cap, ii)];
      dst = __ldg(a.front + im.x);
      beg = __ldg(a.ro + dst);
    }
    const uint64_t key = hash2(a.seed, hash2(a.layer, dst));
    const bool seg = im.w != kInv;
    const uint32_t p0 = im.y, p1 = live ? im.z : im.y;
    uint32_t* rid = a.hub.rec_id + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    uint64_t* rkey = a.hub.rec_key + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    // ---- fill (sampler.cpp:30-33)
    const uint32_t nf = min(m, p1 - p0);
    uint64_t rk[MB];
    uint32_t rp[MB];
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      rk[i] = ~0ull;
      rp[i] = 0;
      if (static_cast<uint32_t>(i) < nf) {
        rk[i] = draw(key, static_cast<uint64_t>(p0) + i + 1) >> 11;
        rp[i] = p0 + i;
        if (seg) {
          rid[i] = rp[i];
          rkey[i] = rk[i];
        }
      }
    }
    uint64_t thr;
    uint32_t mp;
    lane_argmin<MB>(pol, rk, m, thr, mp);
#if A3G_LANE_FUSED
    uint32_t hk[MB];
#pragma unroll
    for (int i = 0; i < MB; ++i) hk[i] = static_cast<uint32_t>(rk[i] >> 21);
    const uint64_t tw = pol.tie >> 21;
    const uint32_t win = static_cast<uint32_t>(tw < 0x7fffffffull ? tw : 0x7fffffffull) + 1u;
#endif
    uint32_t rcnt = nf;
    // ---- replay [p0 + nf, p1) in chunks of 32 positions
    const uint32_t jb = p0 + nf;
    const uint32_t len = p1 > jb ? p1 - jb : 0u;
    uint32_t wlen = len;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) wlen = max(wlen, __shfl_xor_sync(kFull, wlen, off));
    uint64_t ctr = key + (static_cast<uint64_t>(jb) + 1) * kPhi;  // draw index of position jb
    for (uint32_t b = 0; b < wlen; b += 32, ctr += 32 * kPhi) {
      const uint32_t thi = pre_bound(static_cast<uint32_t>(thr >> 21));
      uint32_t cm = 0;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        uint32_t l3;
        const uint32_t h4 = mix64_pre(ctr + static_cast<uint64_t>(c) * kPhi, l3);
        cm |= static_cast<uint32_t>(h4 >= thi) << c;
      }
      const uint32_t rem = len > b ? len - b : 0u;
      if (rem < 32) cm &= (1u << rem) - 1u;
      while (__any_sync(kFull, cm != 0)) {
        if (cm) {
          const int c = __ffs(cm) - 1;
          cm &= cm - 1;
          const uint64_t kx = mix64(ctr + static_cast<uint64_t>(c) * kPhi) >> 11;
          if (pol.gt(kx, thr)) {
            const uint32_t pos = jb + b + c;
            if (seg && rcnt < kRecCap) {
              rid[rcnt] = pos;
              rkey[rcnt] = kx;
            }
            ++rcnt;
#if A3G_LANE_FUSED
            lane_insert<MB>(pol, rk, hk, rp, m, mp, kx, pos, win, thr, mp);
#else
#pragma unroll
            for (int i = 0; i < MB; ++i)
              if (static_cast<uint32_t>(i) == mp) {
                rk[i] = kx;
                rp[i] = pos;
              }
            lane_argmin<MB>(pol, rk, m, thr, mp);
#endif
          }
        }
      }
    }
    if (!live) continue;
    if (seg) {
      a.hub.rec_cnt[im.w] = rcnt;
      a.hub.tau[im.w] = thr;
      a.hub.tau_ok[im.w] = (p1 - p0 >= m) ? 1u : 0u;
    } else {
      const uint32_t* nb = a.col + beg;
      const uint64_t row0 = static_cast<uint64_t>(im.x) * m;
#pragma unroll
      for (int i = 0; i < MB; ++i)
        if (static_cast<uint32_t>(i) < m) {
          const uint32_t id = __ldg(nb + rp[i]);
          a.S[row0 + i] = id;
          mark_first(a.first, id, a.tag, static_cast<uint32_t>(row0 + i));
        }
      a.cnt[im.x] = m;
    }
  }
}

// k_stream_lane with the lane reservoirs in shared memory, slot-major per
// CTA ([slot][thread]: a warp's 32 lanes touch 32 consecutive words, no bank
// conflicts). The slot update is one dynamic-index store instead of a select
// over all MB register slots, and the argmin scans the 32-bit key words with a
// running second minimum, so the near-tie test needs no second pass. Same
// candidates, same replay order, same results (default for fanouts <= 10;
// A3G_LANE_SMEM=0 selects the register reservoirs for A/B). Measured: C2 step
// -4%, C3 -6%, C5 -3% (profiles/r02_sampler_experiments.md).
template <int MB>
struct LaneSmem {
  uint64_t rk[MB][256];
  uint32_t hk[MB][256];
  uint32_t rp[MB][256];
};

template <int MB, typename P>
__device__ __forceinline__ void lane_argmin_s(const P& pol, const LaneSmem<MB>& R, int t, uint32_t m, uint64_t& thr,
                                              uint32_t& mp) {
  uint64_t rk[MB];
#pragma unroll
  for (int i = 0; i < MB; ++i) rk[i] = R.rk[i][t];
  lane_argmin<MB>(pol, rk, m, thr, mp);
}

// Packed slot word: the top 28 bits of the key's 32-bit word (HS: 21 for
// 53-bit integer keys, 32 for the bits of positive fp64 keys) over the slot
// index, so one unsigned min yields the minimum's bucket and its first slot.
template <int HS>
__device__ __forceinline__ uint32_t slot_word(uint64_t k, uint32_t i) {
  return (static_cast<uint32_t>(k >> HS) & ~15u) | i;
}

// win: buckets (units of 2^(HS+4)) within which another slot may hold an
// equal or smaller key in exact order -- then the exact argmin decides.
template <int MB, int HS = 21, typename P>
__device__ __forceinline__ void lane_insert_s(const P& pol, LaneSmem<MB>& R, int t, uint32_t m, uint32_t mp_in,
                                              uint64_t kx, uint32_t pos, uint32_t win, uint64_t& thr, uint32_t& mp) {
  static_assert(MB <= 16, "slot index in 4 bits");
  R.rk[mp_in][t] = kx;
  R.hk[mp_in][t] = slot_word<HS>(kx, mp_in);
  R.rp[mp_in][t] = pos;
  uint32_t mn = 0xffffffffu, mn2 = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const uint32_t w = R.hk[i][t];
    mn2 = min(mn2, max(mn, w));
    mn = min(mn, w);
  }
  if ((mn2 >> 4) - (mn >> 4) <= win) {  // another slot within the window: exact order decides
    lane_argmin_s<MB>(pol, R, t, m, thr, mp);
  } else {
    mp = mn & 15u;
    thr = R.rk[mp][t];
  }
}

template <int WM, int MB>
__global__ void __launch_bounds__(256) k_stream_lane_s(SampleArgs a, const uint32_t* lists, const uint32_t* cls_count) {
  using P = typename PolOf<WM>::P;
  __shared__ LaneSmem<MB> R;
  const int lane = threadIdx.x & 31, t = threadIdx.x;
  const uint32_t nitems = min(*a.item_count, a.hub.item_cap);
  const uint32_t m = a.f;
  const P pol = PolOf<WM>::make(a);
  const uint32_t wstride = gridDim.x * (blockDim.x >> 5) * 32;
  const uint32_t ibase = a.split_cls >= 0 ? items_from_class(cls_count, a.split_cls) : 0u;
  const uint64_t tw = pol.tie >> 25;  // the tie window in slot-word buckets
  const uint32_t win = static_cast<uint32_t>(tw < 0x7ffffffull ? tw : 0x7ffffffull) + 1u;
  for (uint32_t base = ibase + (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < nitems;
       base += wstride) {
    const uint32_t ii = base + lane;
    const bool live = ii < nitems;
    uint4 im = make_uint4(0, 0, 0, kInv);
    uint32_t dst = 0;
    uint64_t beg = 0;
    if (live) {
      im = a.hub.items[item_of(lists, cls_count, a.hub.item_cap, ii)];
      dst = __ldg(a.front + im.x);
      beg = __ldg(a.ro + dst);
    }
    const uint64_t key = hash2(a.seed, hash2(a.layer, dst));
    const bool seg = im.w != kInv;
    const uint32_t p0 = im.y, p1 = live ? im.z : im.y;
    uint32_t* rid = a.hub.rec_id + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    uint64_t* rkey = a.hub.rec_key + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    // ---- fill (sampler.cpp:30-33)
    const uint32_t nf = min(m, p1 - p0);
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      uint64_t k = ~0ull;
      uint32_t p = 0;
      if (static_cast<uint32_t>(i) < nf) {
        k = draw(key, static_cast<uint64_t>(p0) + i + 1) >> 11;
        p = p0 + i;
        if (seg) {
          rid[i] = p;
          rkey[i] = k;
        }
      }
      R.rk[i][t] = k;
      R.hk[i][t] = slot_word<21>(k, i);
      R.rp[i][t] = p;
    }
    uint64_t thr;
    uint32_t mp;
    lane_argmin_s<MB>(pol, R, t, m, thr, mp);
    uint32_t rcnt = nf;
    // ---- replay [p0 + nf, p1) in chunks of 32 positions
    const uint32_t jb = p0 + nf;
    const uint32_t len = p1 > jb ? p1 - jb : 0u;
    uint32_t wlen = len;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) wlen = max(wlen, __shfl_xor_sync(kFull, wlen, off));
    uint64_t ctr = key + (static_cast<uint64_t>(jb) + 1) * kPhi;
    for (uint32_t b = 0; b < wlen; b += 32, ctr += 32 * kPhi) {
      const uint32_t thi = pre_bound(static_cast<uint32_t>(thr >> 21));
      uint32_t cm = 0;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        uint32_t l3;
        const uint32_t h4 = mix64_pre(ctr + static_cast<uint64_t>(c) * kPhi, l3);
        cm |= static_cast<uint32_t>(h4 >= thi) << c;
      }
      const uint32_t rem = len > b ? len - b : 0u;
      if (rem < 32) cm &= (1u << rem) - 1u;
      while (__any_sync(kFull, cm != 0)) {
        if (cm) {
          const int c = __ffs(cm) - 1;
          cm &= cm - 1;
          const uint64_t kx = mix64(ctr + static_cast<uint64_t>(c) * kPhi) >> 11;
          if (pol.gt(kx, thr)) {
            const uint32_t pos = jb + b + c;
            if (seg && rcnt < kRecCap) {
              rid[rcnt] = pos;
              rkey[rcnt] = kx;
            }
            ++rcnt;
            lane_insert_s<MB>(pol, R, t, m, mp, kx, pos, win, thr, mp);
          }
        }
      }
    }
    if (!live) continue;
    if (seg) {
      a.hub.rec_cnt[im.w] = rcnt;
      a.hub.tau[im.w] = thr;
      a.hub.tau_ok[im.w] = (p1 - p0 >= m) ? 1u : 0u;
    } else {
      const uint32_t* nb = a.col + beg;
      const uint64_t row0 = static_cast<uint64_t>(im.x) * m;
#pragma unroll
      for (int i = 0; i < MB; ++i)
        if (static_cast<uint32_t>(i) < m) {
          const uint32_t id = __ldg(nb + R.rp[i][t]);
          a.S[row0 + i] = id;
          mark_first(a.first, id, a.tag, static_cast<uint32_t>(row0 + i));
        }
      a.cnt[im.x] = m;
    }
  }
}

// Lower filter bound lo <= thr^gamma of cached candidates (a cached key
// pow(u, 1/gamma) can beat thr only if u >= lo). Integer gamma <= 64: binary
// powering (<= 12 correctly rounded products, relative error < 1.4e-15) with a
// 1e-9 margin -- u < lo then gives pow(u, 1/gamma) < thr (1 - 1e-10 / gamma)
// even with pow's 2-ulp error; cheap enough to refresh after every insertion.
// Otherwise rsv::gamma_lo (pow with a 1e-6 margin).
__device__ __forceinline__ double lane_gamma_lo(double thr, double gamma, bool gint) {
  if (!gint) return rsv::gamma_lo(thr, gamma);
  if (!(thr < 1.0)) return thr >= 1.0 ? 1.0 : 0.0;  // +inf (unfilled) / NaN guards
  uint32_t e = static_cast<uint32_t>(gamma);
  double p = 1.0, x = thr;
  while (e) {
    if (e & 1u) p *= x;
    x *= x;
    e >>= 1;
  }
  return p * (1.0 - 1e-9);
}

// Lane-per-item stream for bitmap weights (partial cache, gamma > 1), m <= MB:
// as k_stream_lane with fp64 keys (their IEEE bits order like the values, so
// the register argmin compares bit patterns). Each 32-position chunk reads the
// chunk's 32 per-edge cached bits (a3g_cache::d_ebits, two words) instead of
// 32 adjacency entries + 32 bitmap words; the prefilter bound per position is
// lo = thr^gamma (1 - 1e-6) for cached targets (k = u^(1/gamma) can beat thr
// only if u >= lo, reservoir.cuh PolMixed) and thr for the others (k = u).
// Both bounds are taken at the chunk start: they only grow, so stale bounds
// only add candidates, each tested exactly in position order.
template <int MB>
__global__ void __launch_bounds__(256) k_stream_lane_mixed(SampleArgs a, const uint32_t* lists,
                                                           const uint32_t* cls_count) {
  const int lane = threadIdx.x & 31;
  const uint32_t nitems = min(*a.item_count, a.hub.item_cap);
  const uint32_t m = a.f;
  const double ig = a.inv_gamma, gamma = a.gamma;
  const bool gint = gamma == floor(gamma) && gamma <= 64.0;  // lane_gamma_lo by multiplications
  const uint32_t* eb = a.ebits;
  const rsv::PolUnit ipol{};
  // grid sized to the layer's item bound: one batch of 32 items per warp
  // (short-lived CTAs let the high-priority compute stream's kernels in)
  const uint32_t wstride = gridDim.x * (blockDim.x >> 5) * 32;
  const uint32_t ibase = a.split_cls >= 0 ? items_from_class(cls_count, a.split_cls) : 0u;
  for (uint32_t base = ibase + (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < nitems;
       base += wstride) {
    const uint32_t ii = base + lane;
    const bool live = ii < nitems;
    uint4 im = make_uint4(0, 0, 0, kInv);
    uint32_t dst = 0;
    uint64_t beg = 0;
    if (live) {
      im = a.hub.items[item_of(lists, cls_count, a.hub.item_cap, ii)];
      dst = __ldg(a.front + im.x);
      beg = __ldg(a.ro + dst);
    }
    const uint64_t key = hash2(a.seed, hash2(a.layer, dst));
    const bool seg = im.w != kInv;
    const uint32_t p0 = im.y, p1 = live ? im.z : im.y;
    uint32_t* rid = a.hub.rec_id + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    uint64_t* rkey = a.hub.rec_key + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    auto ebit = [&](uint64_t e) { return (__ldg(eb + (e >> 5)) >> (e & 31)) & 1u; };
    // ---- fill (sampler.cpp:30-33)
    const uint32_t nf = min(m, p1 - p0);
    uint64_t rk[MB];
    uint32_t rp[MB];
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      rk[i] = static_cast<uint64_t>(__double_as_longlong(INFINITY));
      rp[i] = 0;
      if (static_cast<uint32_t>(i) < nf) {
        const uint32_t j = p0 + i;
        const double u = unit_of(draw(key, static_cast<uint64_t>(j) + 1));
        const double k = ebit(beg + j) ? pow(u, ig) : u;
        rk[i] = static_cast<uint64_t>(__double_as_longlong(k));
        rp[i] = j;
        if (seg) {
          rid[i] = j;
          rkey[i] = rk[i];
        }
      }
    }
    uint64_t thrb;
    uint32_t mp;
    lane_argmin<MB>(ipol, rk, m, thrb, mp);
    uint32_t rcnt = nf;
    const uint32_t jb = p0 + nf;
    const uint32_t len = p1 > jb ? p1 - jb : 0u;
    uint32_t wlen = len;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) wlen = max(wlen, __shfl_xor_sync(kFull, wlen, off));
    uint64_t ctr = key + (static_cast<uint64_t>(jb) + 1) * kPhi;
    for (uint32_t b = 0; b < wlen; b += 32, ctr += 32 * kPhi) {
      const double thr = __longlong_as_double(static_cast<long long>(thrb));
      double lo = lane_gamma_lo(thr, gamma, gint);
      const uint32_t b_thr = pre_bound(lo_hi_word(thr)), b_lo = pre_bound(lo_hi_word(lo));
      const uint32_t rem = len > b ? len - b : 0u;
      uint32_t cb = 0;
      if (rem) {
        const uint64_t e0 = beg + jb + b;
        cb = __funnelshift_r(__ldg(eb + (e0 >> 5)), __ldg(eb + (e0 >> 5) + 1), static_cast<uint32_t>(e0 & 31));
      }
      uint32_t cm = 0;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        uint32_t l3;
        const uint32_t h4 = mix64_pre(ctr + static_cast<uint64_t>(c) * kPhi, l3);
        cm |= static_cast<uint32_t>(h4 >= (((cb >> c) & 1u) ? b_lo : b_thr)) << c;
      }
      if (rem < 32) cm &= (1u << rem) - 1u;
      while (__any_sync(kFull, cm != 0)) {
        if (cm) {
          const int c = __ffs(cm) - 1;
          cm &= cm - 1;
          const double t = __longlong_as_double(static_cast<long long>(thrb));
          const double uu = unit_of(mix64(ctr + static_cast<uint64_t>(c) * kPhi));
          double k = uu;
          bool ins;
          if ((cb >> c) & 1u) {
            ins = uu >= lo;  // lo follows every insertion (cheap for integer gamma)
            if (ins) {
              k = pow(uu, ig);
              ins = k > t;
            }
          } else {
            ins = uu > t;
          }
          if (ins) {
            const uint32_t pos = jb + b + c;
            const uint64_t kb = static_cast<uint64_t>(__double_as_longlong(k));
#pragma unroll
            for (int i = 0; i < MB; ++i)
              if (static_cast<uint32_t>(i) == mp) {
                rk[i] = kb;
                rp[i] = pos;
              }
            if (seg && rcnt < kRecCap) {
              rid[rcnt] = pos;
              rkey[rcnt] = kb;
            }
            ++rcnt;
            lane_argmin<MB>(ipol, rk, m, thrb, mp);
            if (gint) lo = lane_gamma_lo(__longlong_as_double(static_cast<long long>(thrb)), gamma, true);
          }
        }
      }
    }
    if (!live) continue;
    if (seg) {
      a.hub.rec_cnt[im.w] = rcnt;
      a.hub.tau[im.w] = thrb;
      a.hub.tau_ok[im.w] = (p1 - p0 >= m) ? 1u : 0u;
    } else {
      const uint32_t* nb = a.col + beg;
      const uint64_t row0 = static_cast<uint64_t>(im.x) * m;
#pragma unroll
      for (int i = 0; i < MB; ++i)
        if (static_cast<uint32_t>(i) < m) {
          const uint32_t id = __ldg(nb + rp[i]);
          a.S[row0 + i] = id;
          mark_first(a.first, id, a.tag, static_cast<uint32_t>(row0 + i));
        }
      a.cnt[im.x] = m;
    }
  }
}

// k_stream_lane_mixed with the lane reservoirs in shared memory (as
// k_stream_lane_s; A/B: A3G_LANE_SMEM).
template <int MB>
// four resident CTAs per SM (64 registers): C5 step -2%, C3 unchanged; the
// same bound on k_stream_lane_s spills and measured 5% slower at C2
__global__ void __launch_bounds__(256, 4) k_stream_lane_mixed_s(SampleArgs a, const uint32_t* lists,
                                                           const uint32_t* cls_count) {
  __shared__ LaneSmem<MB> R;
  const int lane = threadIdx.x & 31, tid = threadIdx.x;
  const uint32_t nitems = min(*a.item_count, a.hub.item_cap);
  const uint32_t m = a.f;
  const double ig = a.inv_gamma, gamma = a.gamma;
  const bool gint = gamma == floor(gamma) && gamma <= 64.0;  // lane_gamma_lo by multiplications
  const uint32_t* eb = a.ebits;
  const rsv::PolUnit ipol{};
  // grid sized to the layer's item bound: one batch of 32 items per warp
  // (short-lived CTAs let the high-priority compute stream's kernels in)
  const uint32_t wstride = gridDim.x * (blockDim.x >> 5) * 32;
  const uint32_t ibase = a.split_cls >= 0 ? items_from_class(cls_count, a.split_cls) : 0u;
  for (uint32_t base = ibase + (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < nitems;
       base += wstride) {
    const uint32_t ii = base + lane;
    const bool live = ii < nitems;
    uint4 im = make_uint4(0, 0, 0, kInv);
    uint32_t dst = 0;
    uint64_t beg = 0;
    if (live) {
      im = a.hub.items[item_of(lists, cls_count, a.hub.item_cap, ii)];
      dst = __ldg(a.front + im.x);
      beg = __ldg(a.ro + dst);
    }
    const uint64_t key = hash2(a.seed, hash2(a.layer, dst));
    const bool seg = im.w != kInv;
    const uint32_t p0 = im.y, p1 = live ? im.z : im.y;
    uint32_t* rid = a.hub.rec_id + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    uint64_t* rkey = a.hub.rec_key + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    auto ebit = [&](uint64_t e) { return (__ldg(eb + (e >> 5)) >> (e & 31)) & 1u; };
    // ---- fill (sampler.cpp:30-33)
    const uint32_t nf = min(m, p1 - p0);
#pragma unroll
    for (int i = 0; i < MB; ++i) {
      uint64_t kb = static_cast<uint64_t>(__double_as_longlong(INFINITY));
      uint32_t p = 0;
      if (static_cast<uint32_t>(i) < nf) {
        const uint32_t j = p0 + i;
        const double u = unit_of(draw(key, static_cast<uint64_t>(j) + 1));
        const double k = ebit(beg + j) ? pow(u, ig) : u;
        kb = static_cast<uint64_t>(__double_as_longlong(k));
        p = j;
        if (seg) {
          rid[i] = j;
          rkey[i] = kb;
        }
      }
      R.rk[i][tid] = kb;
      R.hk[i][tid] = slot_word<32>(kb, i);
      R.rp[i][tid] = p;
    }
    uint64_t thrb;
    uint32_t mp;
    lane_argmin_s<MB>(ipol, R, tid, m, thrb, mp);
    uint32_t rcnt = nf;
    const uint32_t jb = p0 + nf;
    const uint32_t len = p1 > jb ? p1 - jb : 0u;
    uint32_t wlen = len;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) wlen = max(wlen, __shfl_xor_sync(kFull, wlen, off));
    uint64_t ctr = key + (static_cast<uint64_t>(jb) + 1) * kPhi;
    for (uint32_t b = 0; b < wlen; b += 32, ctr += 32 * kPhi) {
      const double thr = __longlong_as_double(static_cast<long long>(thrb));
      double lo = lane_gamma_lo(thr, gamma, gint);
      const uint32_t b_thr = pre_bound(lo_hi_word(thr)), b_lo = pre_bound(lo_hi_word(lo));
      const uint32_t rem = len > b ? len - b : 0u;
      uint32_t cb = 0;
      if (rem) {
        const uint64_t e0 = beg + jb + b;
        cb = __funnelshift_r(__ldg(eb + (e0 >> 5)), __ldg(eb + (e0 >> 5) + 1), static_cast<uint32_t>(e0 & 31));
      }
      uint32_t cm = 0;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        uint32_t l3;
        const uint32_t h4 = mix64_pre(ctr + static_cast<uint64_t>(c) * kPhi, l3);
        cm |= static_cast<uint32_t>(h4 >= (((cb >> c) & 1u) ? b_lo : b_thr)) << c;
      }
      if (rem < 32) cm &= (1u << rem) - 1u;
      while (__any_sync(kFull, cm != 0)) {
        if (cm) {
          const int c = __ffs(cm) - 1;
          cm &= cm - 1;
          const double t = __longlong_as_double(static_cast<long long>(thrb));
          const double uu = unit_of(mix64(ctr + static_cast<uint64_t>(c) * kPhi));
          double k = uu;
          bool ins;
          if ((cb >> c) & 1u) {
            ins = uu >= lo;  // lo follows every insertion (cheap for integer gamma)
            if (ins) {
              k = pow(uu, ig);
              ins = k > t;
            }
          } else {
            ins = uu > t;
          }
          if (ins) {
            const uint32_t pos = jb + b + c;
            const uint64_t kb = static_cast<uint64_t>(__double_as_longlong(k));
            if (seg && rcnt < kRecCap) {
              rid[rcnt] = pos;
              rkey[rcnt] = kb;
            }
            ++rcnt;
            // high words order positive doubles; equal high words: exact argmin
            lane_insert_s<MB, 32>(ipol, R, tid, m, mp, kb, pos, 0u, thrb, mp);
            if (gint) lo = lane_gamma_lo(__longlong_as_double(static_cast<long long>(thrb)), gamma, true);
          }
        }
      }
    }
    if (!live) continue;
    if (seg) {
      a.hub.rec_cnt[im.w] = rcnt;
      a.hub.tau[im.w] = thrb;
      a.hub.tau_ok[im.w] = (p1 - p0 >= m) ? 1u : 0u;
    } else {
      const uint32_t* nb = a.col + beg;
      const uint64_t row0 = static_cast<uint64_t>(im.x) * m;
#pragma unroll
      for (int i = 0; i < MB; ++i)
        if (static_cast<uint32_t>(i) < m) {
          const uint32_t id = __ldg(nb + R.rp[i][tid]);
          a.S[row0 + i] = id;
          mark_first(a.first, id, a.tag, static_cast<uint32_t>(row0 + i));
        }
      a.cnt[im.x] = m;
    }
  }
}

// Per-edge cached bits: warp per 32 consecutive edges (coalesced adjacency
// reads), one ballot per word.
__global__ void k_edge_bits(const uint32_t* col, uint64_t m, const uint32_t* bits, uint32_t* ebits) {
  const uint64_t nw = (m + 31) / 32;
  const int lane = threadIdx.x & 31;
  for (uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; w < nw;
       w += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
    const uint64_t e = w * 32 + lane;
    bool c = false;
    if (e < m) {
      const uint32_t v = __ldg(col + e);
      c = (__ldg(bits + (v >> 5)) >> (v & 31)) & 1u;
    }
    const unsigned word = __ballot_sync(kFull, c);
    if (lane == 0) ebits[w] = word;
  }
}

// Bitmap-weighted items (partial cache, gamma > 1: w = gamma if cached else
// 1, assign_weights sampler.cpp:60-68) by lane groups, as k_stream_grp but
// with fp64 keys: each position needs its neighbour id (the cached bit), and a
// cached neighbour's key pow(u, 1/gamma) is evaluated only when
// u >= thr^gamma (1 - 1e-6) -- below that no <= 2-ulp pow can beat the
// minimum (reservoir.cuh PolMixed). Keys are >= 0, so their IEEE bits order
// like the values: the argmin is the packed top-32-bit butterfly with an
// exact 64-bit fallback on (near-)equal top bits.
template <int G>
__global__ void __launch_bounds__(256) k_stream_grp_mixed(SampleArgs a, const uint32_t* lists,
                                                          const uint32_t* cls_count) {
  constexpr int NG = 32 / G;
  constexpr int U = 32 / G;
  constexpr uint64_t kStepG = static_cast<uint64_t>(G) * kPhi;
  const int lane = threadIdx.x & 31;
  const uint32_t gl = lane % G, grp = lane / G;
  const unsigned gmask = G == 32 ? kFull : (((1u << G) - 1u) << (grp * G));
  uint32_t nitems = min(*a.item_count, a.hub.item_cap);
  if (a.split_cls >= 0) nitems = min(nitems, items_from_class(cls_count, a.split_cls));
  const uint32_t m = a.f;
  const double ig = a.inv_gamma, gamma = a.gamma;
  const uint32_t* bits = a.bits;
  auto cached = [&](uint32_t v) { return (__ldg(bits + (v >> 5)) >> (v & 31)) & 1u; };
  const rsv::PolUnit ipol{};  // bit-pattern argmin (keys >= 0)
  const uint32_t wstride = gridDim.x * (blockDim.x >> 5) * NG;
  for (uint32_t base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * NG; base < nitems; base += wstride) {
    const uint32_t ii = base + grp;
    const bool live = ii < nitems;
    uint4 im = make_uint4(0, 0, 0, kInv);
    uint32_t dst = 0;
    uint64_t beg = 0;
    if (live) {
      im = a.hub.items[item_of(lists, cls_count, a.hub.item_cap, ii)];
      dst = __ldg(a.front + im.x);
      beg = __ldg(a.ro + dst);
    }
    const uint32_t* nb = a.col + beg;
    const uint64_t key = hash2(a.seed, hash2(a.layer, dst));
    const bool seg = im.w != kInv;
    const uint64_t row0 = static_cast<uint64_t>(im.x) * m;
    const uint32_t p0 = im.y, p1 = im.z;
    const uint32_t nf = live ? min(m, p1 - p0) : 0u;
    uint64_t my_key = __double_as_longlong(INFINITY);  // key bits
    uint32_t my_pos = 0;
    uint32_t* rid = a.hub.rec_id + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    uint64_t* rkey = a.hub.rec_key + static_cast<uint64_t>(seg ? im.w : 0) * kRecCap;
    if (gl < nf) {
      const uint32_t j = p0 + gl;
      const double u = unit_of(draw(key, static_cast<uint64_t>(j) + 1));
      const double k = cached(__ldg(nb + j)) ? pow(u, ig) : u;
      my_key = __double_as_longlong(k);
      my_pos = j;
      if (seg) {
        rid[gl] = j;
        rkey[gl] = my_key;
      }
    }
    uint64_t thrb;
    uint32_t mp;
    grp_argmin<G, rsv::PolUnit, true>(ipol, my_key, gl, thrb, mp);
    double thr = __longlong_as_double(thrb);
    double lo = rsv::gamma_lo(thr, gamma);
    uint32_t rcnt = nf;
    const uint32_t jb = p0 + nf;
    uint32_t len = live && p1 > jb ? p1 - jb : 0u;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) len = max(len, __shfl_xor_sync(kFull, len, off));
    uint64_t ctr = key + (static_cast<uint64_t>(jb) + gl + 1) * kPhi;
    for (uint32_t b = 0; b < len; b += 32, ctr += 32 * kPhi) {
      double kk[U];
      bool c[U];
      bool anyc = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t j = jb + b + u * G + gl;
        const bool valid = j < p1;
        const uint32_t v = valid ? __ldg(nb + j) : 0u;
        const double uu = unit_of(mix64(ctr + u * kStepG));
        const bool cw = valid && cached(v);
        kk[u] = uu;
        c[u] = valid && (cw ? uu >= lo : uu > thr);
        if (c[u] && cw) {
          kk[u] = pow(uu, ig);
          c[u] = kk[u] > thr;
        }
        anyc |= c[u];
      }
      if (!__any_sync(kFull, anyc)) continue;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        unsigned mask = __ballot_sync(kFull, c[u] && kk[u] > thr) & gmask;
        while (__any_sync(kFull, mask != 0)) {
          const int src = mask ? __ffs(mask) - 1 : lane;
          const double kv = __shfl_sync(kFull, kk[u], src);
          const bool ins = mask != 0 && kv > thr;
          const uint32_t pos = jb + b + u * G + (static_cast<uint32_t>(src) % G);
          if (ins && gl == mp) {
            my_key = __double_as_longlong(kv);
            my_pos = pos;
          }
          if (ins && seg && lane == src) {
            if (rcnt < kRecCap) {
              rid[rcnt] = pos;
              rkey[rcnt] = __double_as_longlong(kv);
            }
          }
          if (ins) ++rcnt;
          uint64_t nthr;
          uint32_t nmp;
          grp_argmin<G, rsv::PolUnit, true>(ipol, my_key, gl, nthr, nmp);
          if (ins) {
            thr = __longlong_as_double(nthr);
            mp = nmp;
          }
          if (mask) mask &= ~((2u << src) - 1u);
          mask &= __ballot_sync(kFull, c[u] && kk[u] > thr) & gmask;
        }
      }
      lo = rsv::gamma_lo(thr, gamma);
    }
    if (!live) continue;
    if (seg) {
      if (gl == 0) {
        a.hub.rec_cnt[im.w] = rcnt;
        a.hub.tau[im.w] = __double_as_longlong(thr);
        a.hub.tau_ok[im.w] = (p1 - p0 >= m) ? 1u : 0u;
      }
    } else if (gl < m) {
      const uint32_t id = __ldg(nb + my_pos);
      a.S[row0 + gl] = id;
      mark_first(a.first, id, a.tag, static_cast<uint32_t>(row0 + gl));
      if (gl == 0) a.cnt[im.x] = m;
    }
  }
}

// Warp per hub with few segments (<= kMergeFilterWarps): replay the records in
// segment order, dropping those that cannot beat max_{s'<s} tau_{s'}.
template <int WM>
__device__ void merge_small_hub(const SampleArgs& a, uint32_t h, int lane);

constexpr int kMergeFilterWarps = kMergeFilterWarpsC;
constexpr int kMergeThreads = (kMergeFilterWarps + 1) * 32;
constexpr size_t kMergeSmemWin = 2ull * kMergeFilterWarps * kRecCap * (8 + 4);

// Big hubs (more than kMergeFilterWarps segments), block per hub, without a
// serial window chain: (A) L_s = max tau over segments < s and the record
// prefix over segments (warp scans), (B) every thread filters records of the
// flattened (segment, record) list against L_s -- a global insertion in
// segment s must beat the running minimum, which is >= L_s -- into a keep
// bitmap (independent loads, no warp collectives), then ranks the kept ones
// by popcounts and writes them in (segment, record) order to shared memory,
// (C) warp 0 replays the few survivors exactly. Falls back to the windowed
// k_hub_merge path (same block) when a hub has more segments or survivors
// than the shared-memory plan holds.
constexpr int kM2Warps = kMergeFilterWarps + 1;  // the k_hub_merge block
constexpr int kM2Threads = kM2Warps * 32;
constexpr uint32_t kM2MaxSegs = 1024;
constexpr uint32_t kM2MaxSurv = 3072;
constexpr uint32_t kM2Words = kRecCap / 32;  // keep-bitmap words per segment
constexpr size_t kM2Smem = kM2MaxSegs * (8 + 4 + 4 + 4 + 4 * kM2Words) + kM2MaxSurv * (8 + 4);

template <int WM>
__device__ bool hub_merge_parallel(const SampleArgs& a, uint32_t h, uint8_t* smem) {
  using P = typename PolOf<WM>::P;
  using K = typename P::K;
  K* s_L = reinterpret_cast<K*>(smem);                                   // [segs] prefix max tau
  uint32_t* s_lok = reinterpret_cast<uint32_t*>(smem + kM2MaxSegs * 8);  // [segs]
  uint32_t* s_pre = s_lok + kM2MaxSegs;                                  // [segs] record prefix
  uint32_t* s_off = s_pre + kM2MaxSegs;                                  // [segs] survivor prefix
  uint32_t* s_bits = s_off + kM2MaxSegs;                                 // [segs][kM2Words]
  K* s_key = reinterpret_cast<K*>(s_bits + kM2MaxSegs * kM2Words);        // [kM2MaxSurv]
  uint32_t* s_pos = reinterpret_cast<uint32_t*>(s_key + kM2MaxSurv);      // [kM2MaxSurv]
  __shared__ uint32_t s_nrec, s_total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t ns = a.hub.nseg[h], s0 = a.hub.seg0[h], k = a.hub.row[h];
  const uint32_t m = a.f;
  if (ns > kM2MaxSegs) return false;
  P pol = PolOf<WM>::make(a);
  for (uint32_t i = threadIdx.x; i < ns * kM2Words; i += blockDim.x) s_bits[i] = 0;
  if (warp == 0) {
    // (A) exclusive prefix max of tau (segments with tau_ok) + record prefix
    K run{};
    int rok = 0;
    uint32_t rrun = 0;
    for (uint32_t c0 = 0; c0 < ns; c0 += 32) {
      const uint32_t s = c0 + lane;
      int ok = 0;
      K tv{};
      uint32_t rc = 0;
      if (s < ns) {
        ok = a.hub.tau_ok[s0 + s];
        tv = key_from_bits<K>(a.hub.tau[s0 + s]);
        rc = a.hub.rec_cnt[s0 + s];
        if (s == 0) rc = rc > m ? rc - m : 0u;  // segment 0's fill records seed the reservoir
      }
      K iv = tv;
      int iok = ok;
      uint32_t inc = rc;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const K ov = __shfl_up_sync(kFull, iv, off);
        const int oo = __shfl_up_sync(kFull, iok, off);
        const uint32_t oc = __shfl_up_sync(kFull, inc, off);
        if (lane >= off) {
          if (oo && (!iok || ov > iv)) {
            iv = ov;
            iok = 1;
          }
          inc += oc;
        }
      }
      K ev = __shfl_up_sync(kFull, iv, 1);
      int eok = __shfl_up_sync(kFull, iok, 1);
      if (lane == 0) eok = 0;
      if (rok && (!eok || run > ev)) {
        ev = run;
        eok = 1;
      }
      if (s < ns) {
        s_L[s] = ev;
        s_lok[s] = eok;
        s_pre[s] = rrun + inc - rc;
      }
      const K lv = __shfl_sync(kFull, iv, 31);
      const int lo = __shfl_sync(kFull, iok, 31);
      if (lo && (!rok || lv > run)) {
        run = lv;
        rok = 1;
      }
      rrun += __shfl_sync(kFull, inc, 31);
    }
    if (lane == 0) s_nrec = rrun;
  }
  __syncthreads();
  const uint32_t nrec = s_nrec;
  // segment of flattened record r: last s with s_pre[s] <= r
  auto seg_of = [&](uint32_t r) {
    uint32_t lo = 0, hi = ns;  // s_pre[lo] <= r < s_pre[hi]
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_pre[mid] <= r) lo = mid; else hi = mid;
    }
    return lo;
  };
  // (B1) keep bitmap; 4 records per thread per round with their loads issued
  // together (the round trips, not the work, bound this phase)
  constexpr int kB1 = 4;
  for (uint32_t r0 = threadIdx.x; r0 < nrec; r0 += kB1 * blockDim.x) {
    uint32_t sg[kB1], ix[kB1];
    uint64_t kb[kB1];
#pragma unroll
    for (int q = 0; q < kB1; ++q) {
      const uint32_t r = r0 + q * blockDim.x;
      sg[q] = r < nrec ? seg_of(r) : 0u;
      ix[q] = r < nrec ? r - s_pre[sg[q]] + (sg[q] == 0 ? m : 0u) : 0u;
      kb[q] = r < nrec ? a.hub.rec_key[static_cast<uint64_t>(s0 + sg[q]) * kRecCap + ix[q]] : 0ull;
    }
#pragma unroll
    for (int q = 0; q < kB1; ++q) {
      if (r0 + q * blockDim.x >= nrec) break;
      const uint32_t sq = sg[q], iq = ix[q];
      if (!s_lok[sq] || pol.keep(key_from_bits<K>(kb[q]), s_L[sq]))
        atomicOr(&s_bits[sq * kM2Words + (iq >> 5)], 1u << (iq & 31));
    }
  }
  __syncthreads();
  if (warp == 0) {  // survivors per segment -> exclusive offsets
    uint32_t run = 0;
    for (uint32_t c0 = 0; c0 < ns; c0 += 32) {
      const uint32_t s = c0 + lane;
      uint32_t v = 0;
      if (s < ns)
        for (uint32_t w = 0; w < kM2Words; ++w) v += __popc(s_bits[s * kM2Words + w]);
      uint32_t inc = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, off);
        if (lane >= off) inc += y;
      }
      if (s < ns) s_off[s] = run + inc - v;
      run += __shfl_sync(kFull, inc, 31);
    }
    if (lane == 0) s_total = run;
  }
  __syncthreads();
  if (s_total > kM2MaxSurv) return false;  // uniform: read after the barrier
  // (B2) kept records to their (segment, record)-ordered rank
  for (uint32_t r = threadIdx.x; r < nrec; r += blockDim.x) {
    const uint32_t s = seg_of(r);
    const uint32_t i = r - s_pre[s] + (s == 0 ? m : 0u);
    const uint32_t* bw = s_bits + s * kM2Words;
    if (!((bw[i >> 5] >> (i & 31)) & 1u)) continue;
    uint32_t rank = s_off[s] + __popc(bw[i >> 5] & ((1u << (i & 31)) - 1u));
    for (uint32_t w = 0; w < (i >> 5); ++w) rank += __popc(bw[w]);
    const uint64_t rb = static_cast<uint64_t>(s0 + s) * kRecCap + i;
    s_key[rank] = key_from_bits<K>(a.hub.rec_key[rb]);
    s_pos[rank] = a.hub.rec_id[rb];
  }
  __syncthreads();
  // (C) exact replay of the survivors by warp 0
  if (warp == 0) {
    const uint32_t dst = a.front[k];
    const uint64_t beg = a.ro[dst];
    const uint32_t* nb = a.col + beg;
    const uint64_t rb0 = static_cast<uint64_t>(s0) * kRecCap;
    rsv::WState<K> st;
    st.my_key = lane < static_cast<int>(m) ? key_from_bits<K>(a.hub.rec_key[rb0 + lane]) : pol.inf();
    st.my_id = lane < static_cast<int>(m) ? a.hub.rec_id[rb0 + lane] : 0u;
    pol.argmin(st.thr, st.mp, st.my_key, lane);
    const uint32_t n = s_total;
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
      const uint32_t i = i0 + lane;
      const bool valid = i < n;
      const K kk = valid ? s_key[i] : K{};
      const uint32_t v = valid ? s_pos[i] : 0u;
      unsigned mask = __ballot_sync(kFull, valid && pol.cheap_gt(kk, st.thr));
      while (mask) {
        const int src = __ffs(mask) - 1;
        const K kv = __shfl_sync(kFull, kk, src);
        const uint32_t iv = __shfl_sync(kFull, v, src);
        if (pol.gt(kv, st.thr)) {
          if (lane == st.mp) {
            st.my_key = kv;
            st.my_id = iv;
          }
          pol.argmin(st.thr, st.mp, st.my_key, lane);
          mask &= __ballot_sync(kFull, valid && pol.cheap_gt(kk, st.thr));
        }
        mask &= ~((2u << src) - 1u);
      }
    }
    const uint64_t row0 = static_cast<uint64_t>(k) * m;
    if (lane < static_cast<int>(m)) {
      const uint32_t id = __ldg(nb + st.my_id);  // records hold row positions
      a.S[row0 + lane] = id;
      mark_first(a.first, id, a.tag, static_cast<uint32_t>(row0 + lane));
    }
    if (lane == 0) a.cnt[k] = m;
  }
  return true;
}

constexpr size_t kMergeSmem = kMergeSmemWin > kM2Smem ? kMergeSmemWin : kM2Smem;

// Block per hub: warp 0 replays window w-1 while warps 1..8 filter window w.
template <int WM>
__global__ void __launch_bounds__(kMergeThreads) k_hub_merge(SampleArgs a) {
  using P = typename PolOf<WM>::P;
  using K = typename P::K;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  K* s_key = reinterpret_cast<K*>(smem_raw);  // [2][8][kRecCap]
  uint32_t* s_id = reinterpret_cast<uint32_t*>(smem_raw + 2ull * kMergeFilterWarps * kRecCap * 8);
  __shared__ uint32_t s_n[2][kMergeFilterWarps];
  __shared__ K s_lrun[2];
  __shared__ int s_lok[2];
  __shared__ uint32_t s_hub[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nbig = min(*a.big_count, a.hub.hub_cap);
  const uint32_t m = a.f;
  for (uint32_t hb = blockIdx.x; hb < nbig; hb += gridDim.x) {
    const uint32_t h = a.hub.big[hb];
    if (threadIdx.x == 0) {
      s_hub[0] = a.hub.nseg[h];
      s_hub[1] = a.hub.seg0[h];
      s_hub[2] = a.hub.row[h];
      s_lok[0] = 0;
      s_lok[1] = 0;
    }
    __syncthreads();
    const uint32_t ns = s_hub[0];
    if (ns <= kMergeFilterWarps) {  // 0: streamed whole; small: merge_small_hub
      __syncthreads();
      continue;
    }
    const uint32_t s0 = s_hub[1], k = s_hub[2];
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
    int of = 0;
    for (uint32_t s = threadIdx.x; s < ns; s += kMergeThreads) of |= a.hub.rec_cnt[s0 + s] > kRecCap;
    if (__syncthreads_or(of)) {  // a segment overflowed its records: exact whole-row replay
      if (warp == 0) row_by_warp<WM>(a, nb, deg, key, k, lane);
      __syncthreads();
      continue;
    }
    const bool par = hub_merge_parallel<WM>(a, h, smem_raw);  // uniform across the block
    __syncthreads();
    if (par) continue;
    P pol = PolOf<WM>::make(a);
    rsv::WState<K> st;
    if (warp == 0) {  // global fill = records 0..m-1 of segment 0 (positions 0..m-1)
      const uint64_t rb = static_cast<uint64_t>(s0) * kRecCap;
      st.my_key = lane < static_cast<int>(m) ? key_from_bits<K>(a.hub.rec_key[rb + lane]) : pol.inf();
      st.my_id = lane < static_cast<int>(m) ? a.hub.rec_id[rb + lane] : 0u;
      pol.argmin(st.thr, st.mp, st.my_key, lane);
    }
    const uint32_t nwin = (ns + kMergeFilterWarps - 1) / kMergeFilterWarps;
    for (uint32_t it = 0; it <= nwin; ++it) {
      if (warp > 0 && it < nwin) {
        // ---- filter window `it` into buffer it%2
        const uint32_t fw = warp - 1, buf = it & 1, w0 = it * kMergeFilterWarps;
        const uint32_t s = w0 + fw;
        // L = max tau over segments < s (prefix from earlier windows + this window)
        K L = s_lrun[buf];
        int lok = s_lok[buf];
        {
          const uint32_t t = w0 + lane;
          K tv{};
          int tok = 0;
          if (lane < static_cast<int>(fw) && t < ns) {
            tok = a.hub.tau_ok[s0 + t];
            tv = key_from_bits<K>(a.hub.tau[s0 + t]);
          }
          for (int off = 16; off > 0; off >>= 1) {
            const K ov = __shfl_xor_sync(kFull, tv, off);
            const int oo = __shfl_xor_sync(kFull, tok, off);
            if (oo && (!tok || ov > tv)) {
              tv = ov;
              tok = 1;
            }
          }
          if (tok && (!lok || tv > L)) {
            L = tv;
            lok = 1;
          }
        }
        uint32_t n_keep = 0;
        if (s < ns) {
          const uint64_t rb = static_cast<uint64_t>(s0 + s) * kRecCap;
          const uint32_t rc = a.hub.rec_cnt[s0 + s];
          K* kb = s_key + (buf * kMergeFilterWarps + fw) * kRecCap;
          uint32_t* ib = s_id + (buf * kMergeFilterWarps + fw) * kRecCap;
          for (uint32_t i0 = (s == 0 ? m : 0); i0 < rc; i0 += 32) {
            const uint32_t i = i0 + lane;
            K kv{};
            uint32_t iv = 0;
            if (i < rc) {
              kv = key_from_bits<K>(a.hub.rec_key[rb + i]);
              iv = a.hub.rec_id[rb + i];
            }
            const bool keep = i < rc && (!lok || pol.keep(kv, L));
            const unsigned bm = __ballot_sync(kFull, keep);
            if (keep) {
              const uint32_t o = n_keep + __popc(bm & ((1u << lane) - 1u));
              kb[o] = kv;
              ib[o] = iv;
            }
            n_keep += __popc(bm);
          }
        }
        if (lane == 0) s_n[buf][fw] = n_keep;
        if (fw == 0) {  // running bound for the next window
          const uint32_t t = w0 + lane;
          K tv{};
          int tok = 0;
          if (lane < kMergeFilterWarps && t < ns) {
            tok = a.hub.tau_ok[s0 + t];
            tv = key_from_bits<K>(a.hub.tau[s0 + t]);
          }
          for (int off = 16; off > 0; off >>= 1) {
            const K ov = __shfl_xor_sync(kFull, tv, off);
            const int oo = __shfl_xor_sync(kFull, tok, off);
            if (oo && (!tok || ov > tv)) {
              tv = ov;
              tok = 1;
            }
          }
          K nl = s_lrun[buf];
          int nok = s_lok[buf];
          if (tok && (!nok || tv > nl)) {
            nl = tv;
            nok = 1;
          }
          if (lane == 0) {
            s_lrun[buf ^ 1] = nl;
            s_lok[buf ^ 1] = nok;
          }
        }
      }
      if (warp == 0 && it > 0) {
        // ---- replay window it-1 from buffer (it-1)%2, in segment order
        const uint32_t buf = (it - 1) & 1, w0 = (it - 1) * kMergeFilterWarps;
        for (uint32_t fw = 0; fw < kMergeFilterWarps && w0 + fw < ns; ++fw) {
          const uint32_t n = s_n[buf][fw];
          const K* kb = s_key + (buf * kMergeFilterWarps + fw) * kRecCap;
          const uint32_t* ib = s_id + (buf * kMergeFilterWarps + fw) * kRecCap;
          for (uint32_t i0 = 0; i0 < n; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool valid = i < n;
            const K kk = valid ? kb[i] : K{};
            const uint32_t v = valid ? ib[i] : 0u;
            unsigned mask = __ballot_sync(kFull, valid && pol.cheap_gt(kk, st.thr));
            while (mask) {
              const int src = __ffs(mask) - 1;
              const K kv = __shfl_sync(kFull, kk, src);
              const uint32_t iv = __shfl_sync(kFull, v, src);
              if (pol.gt(kv, st.thr)) {
                if (lane == st.mp) {
                  st.my_key = kv;
                  st.my_id = iv;
                }
                pol.argmin(st.thr, st.mp, st.my_key, lane);
                mask &= __ballot_sync(kFull, valid && pol.cheap_gt(kk, st.thr));
              }
              mask &= ~((2u << src) - 1u);
            }
          }
        }
      }
      __syncthreads();
    }
    if (warp == 0) {
      if (lane < static_cast<int>(m)) {
        const uint32_t id = __ldg(nb + st.my_id);  // records hold row positions
        a.S[row0 + lane] = id;
        mark_first(a.first, id, a.tag, static_cast<uint32_t>(row0 + lane));
      }
      if (lane == 0) a.cnt[k] = m;
    }
    __syncthreads();
  }
  // small hubs (1..kMergeFilterWarps segments): warp per hub, claimed
  // dynamically so warps of blocks without (or done with) big hubs take them
  const uint32_t nsmall = min(*a.small_count, a.hub.hub_cap);
  for (;;) {
    uint32_t hs = 0;
    if (lane == 0) hs = atomicAdd(a.work, 1u);
    hs = __shfl_sync(kFull, hs, 0);
    if (hs >= nsmall) break;
    merge_small_hub<WM>(a, a.hub.small[hs], lane);
  }
}

// Warp merge of one hub with 1..kMergeFilterWarps segments: replay the
// records in segment order, dropping those that cannot beat max_{s'<s} tau_{s'}.
template <int WM>
__device__ void merge_small_hub(const SampleArgs& a, uint32_t h, int lane) {
  using P = typename PolOf<WM>::P;
  using K = typename P::K;
  const uint32_t m = a.f;
  {
    const uint32_t ns = a.hub.nseg[h];
    if (ns == 0 || ns > kMergeFilterWarps) return;
    const uint32_t s0 = a.hub.seg0[h], k = a.hub.row[h];
    const uint32_t dst = a.front[k];
    const uint64_t beg = a.ro[dst], deg = a.ro[dst + 1] - beg;
    const uint32_t* nb = a.col + beg;
    const uint64_t key = hash2(a.seed, hash2(a.layer, dst));
    const uint64_t row0 = static_cast<uint64_t>(k) * m;
    uint32_t rc_l = 0, tok_l = 0;
    uint64_t tau_l = 0;
    if (lane < static_cast<int>(ns)) {
      rc_l = a.hub.rec_cnt[s0 + lane];
      tok_l = a.hub.tau_ok[s0 + lane];
      tau_l = a.hub.tau[s0 + lane];
    }
    uint32_t my_id;
    if (a.kind == A3G_SAMPLER_UNIFORM) {
      my_id = lane < static_cast<int>(m) ? nb[lane] : 0u;
      for (int s = static_cast<int>(ns) - 1; s >= 0; --s) {
        const uint32_t last = a.hub.slot_last[static_cast<uint64_t>(s0 + s) * 32 + lane];
        if (last != kInv) {
          my_id = nb[last];
          break;
        }
      }
    } else if (__ballot_sync(kFull, rc_l > kRecCap)) {  // records overflowed: whole-row replay
      row_by_warp<WM>(a, nb, deg, key, k, lane);
      return;
    } else {
      P pol = PolOf<WM>::make(a);
      rsv::WState<K> st;
      const uint64_t rb0 = static_cast<uint64_t>(s0) * kRecCap;
      st.my_key = lane < static_cast<int>(m) ? key_from_bits<K>(a.hub.rec_key[rb0 + lane]) : pol.inf();
      st.my_id = lane < static_cast<int>(m) ? a.hub.rec_id[rb0 + lane] : 0u;
      pol.argmin(st.thr, st.mp, st.my_key, lane);
      K L{};
      bool lok = false;
      for (uint32_t s = 0; s < ns; ++s) {
        const uint32_t rc = __shfl_sync(kFull, rc_l, s);
        const uint64_t rb = static_cast<uint64_t>(s0 + s) * kRecCap;
        for (uint32_t i0 = (s == 0 ? m : 0); i0 < rc; i0 += 32) {
          const uint32_t i = i0 + lane;
          const bool valid = i < rc;
          K kk{};
          uint32_t v = 0;
          if (valid) {
            kk = key_from_bits<K>(a.hub.rec_key[rb + i]);
            v = a.hub.rec_id[rb + i];
          }
          const bool keep = valid && (!lok || pol.keep(kk, L));
          unsigned mask = __ballot_sync(kFull, keep && pol.cheap_gt(kk, st.thr));
          while (mask) {
            const int src = __ffs(mask) - 1;
            const K kv = __shfl_sync(kFull, kk, src);
            const uint32_t iv = __shfl_sync(kFull, v, src);
            if (pol.gt(kv, st.thr)) {
              if (lane == st.mp) {
                st.my_key = kv;
                st.my_id = iv;
              }
              pol.argmin(st.thr, st.mp, st.my_key, lane);
              mask &= __ballot_sync(kFull, keep && pol.cheap_gt(kk, st.thr));
            }
            mask &= ~((2u << src) - 1u);
          }
        }
        if (__shfl_sync(kFull, tok_l, s)) {
          const K ts = key_from_bits<K>(__shfl_sync(kFull, tau_l, s));
          if (!lok || ts > L) L = ts;
          lok = true;
        }
      }
      my_id = lane < static_cast<int>(m) ? __ldg(nb + st.my_id) : 0u;  // records hold row positions
    }
    if (lane < static_cast<int>(m)) {
      a.S[row0 + lane] = my_id;
      mark_first(a.first, my_id, a.tag, static_cast<uint32_t>(row0 + lane));
    }
    if (lane == 0) a.cnt[k] = m;
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
      id = rsv::uniform_row_warp(nb, deg, m, key, lane, c0);
    } else {
      rsv::PolMixed<rsv::ListW> pol{rsv::ListW{w}, false, 1.0, 0.0};
      id = rsv::weighted_row_warp(nb, deg, m, key, lane, pol, c0);
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

// Device-resident seeds are not visible to the host validation
// (sampler.cpp:92-94 "seed out of range"): flag them in the batch counters
// (raised as ParameterError once the host syncs) and clamp them to node 0 so
// no kernel of this batch reads the CSR out of bounds.
__global__ void k_check_seeds(uint32_t* seeds, uint32_t n_seeds, uint64_t num_nodes, BatchCounters* c) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_seeds && seeds[i] >= num_nodes) {
    seeds[i] = 0;
    atomicOr(&c->bad_seeds, 1u);
  }
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

// Flags of the kFinRounds positions base + r*kFinThreads + tid, with the three
// dependent loads (slot id -> first-position word -> interner word) issued
// as three batches of independent loads instead of 3 x kFinRounds serial
// round trips (the tables are L2-resident; the kernel is latency-bound).
__device__ __forceinline__ void fin_flags_all(const FinArgs& a, uint64_t P, uint64_t base, Flags (&fl)[kFinRounds]) {
  uint32_t valid = 0;
#pragma unroll
  for (int r = 0; r < kFinRounds; ++r) {
    const uint64_t p = base + r * kFinThreads + threadIdx.x;
    fl[r] = Flags{false, false, false, 0};
    bool ok = p < P;
    if (ok && a.cnt) {
      const uint64_t row = p / a.f;
      ok = static_cast<uint32_t>(p - row * a.f) < __ldg(a.cnt + row);
    }
    if (ok) {
      valid |= 1u << r;
      fl[r].v = __ldg(a.S + p);
    }
  }
  uint64_t fw[kFinRounds];
#pragma unroll
  for (int r = 0; r < kFinRounds; ++r) fw[r] = (valid >> r) & 1u ? a.first[fl[r].v] : 0ull;
  uint64_t gw[kFinRounds];
#pragma unroll
  for (int r = 0; r < kFinRounds; ++r) {
    const uint64_t p = base + r * kFinThreads + threadIdx.x;
    const uint64_t want = (static_cast<uint64_t>(a.tag) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(p));
    fl[r].valid = (valid >> r) & 1u;
    fl[r].first = fl[r].valid && fw[r] == want;
    gw[r] = fl[r].first ? a.gidx[fl[r].v] : 0ull;
  }
#pragma unroll
  for (int r = 0; r < kFinRounds; ++r) fl[r].isnew = fl[r].first && static_cast<uint32_t>(gw[r] >> 32) != a.gtag;
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
  Flags fl[kFinRounds];
  fin_flags_all(a, P, base, fl);
#pragma unroll
  for (int r = 0; r < kFinRounds; ++r) {
    cv += __popc(__ballot_sync(kFull, fl[r].valid));
    cf += __popc(__ballot_sync(kFull, fl[r].first));
    cn += __popc(__ballot_sync(kFull, fl[r].isnew));
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
  Flags fla[kFinRounds];
  fin_flags_all(a, P, base, fla);
#pragma unroll
  for (int r = 0; r < kFinRounds; ++r) {
    const Flags& fl = fla[r];
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
__global__ void k_gather_unique(const __grid_constant__ StoreView view, uint32_t F, const uint32_t* unique,
                                const uint32_t* ucount, const uint32_t* bits, int bitmode, float* out,
                                BatchCounters* ctr) {
  const uint32_t U = *ucount;
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  uint32_t hits = 0, seen = 0;
  for (uint32_t i = gw; i < U; i += nw) {
    const uint32_t v = unique[i];
    const T* src = reinterpret_cast<const T*>(row_ptr(view, v));
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

constexpr int kGrpThreads = 256;  // CTA size of the lane-group stream kernels (64 measured slower)

// frontier bound from which a layer's items go lane-per-item (A3G_LANE_MIN_ROWS
// overrides it for tuning sweeps)
// (r01 A/B, 3 reps each: dense C2 layer 1 (15K rows of ~500 neighbours) runs
// 4% faster lane-per-item with 8192, sparse C1 layer 1 (10K rows of ~9) 7%
// slower -- most of its rows are fill-only, too few items for lane parallelism)
static uint64_t lane_min_rows(bool dense) {
  static const char* e = std::getenv("A3G_LANE_MIN_ROWS");
  if (e) return std::strtoull(e, nullptr, 10);
  return dense ? 8192ull : 32768ull;
}

// A3G_DIAG_SKIP=<stage>[,<stage>...] (diagnostics only, results are wrong):
// skip a sampler stage to see what bounds the pipelined throughput.
static bool diag_skip(const char* stage) {
  static const char* e = std::getenv("A3G_DIAG_SKIP");
  return e && std::strstr(e, stage) != nullptr;
}

// aux / ev_fork / ev_join: with A3G_SPLIT_CLS (long items to the lane-group
// kernel) and A3G_SPLIT_FORK=1, the lane-group launch forks onto the arena's
// auxiliary stream so it runs beside the lane kernel.
template <int WM>
void launch_layer_kernels(const SampleArgs& sa, uint64_t rows_bound, int sm_count, cudaStream_t st,
                          cudaStream_t aux, cudaEvent_t ev_fork, cudaEvent_t ev_join) {
  if (!diag_skip("classify")) k_classify<WM><<<sm_count * 2, 256, 0, st>>>(sa);
  A3G_LAUNCH_DONE("k_classify", st);
  if (sa.f <= 32) {
    bool fork = false;
    static std::atomic<uint64_t> attr_done{0};
    smem_attr_once(attr_done, reinterpret_cast<const void*>(k_hub_merge<WM>), kMergeSmem);
    {
      // lane groups over the length-sorted items: integer keys (or Algorithm
      // R) in k_stream_grp, bitmap weights (fp64 keys) in k_stream_grp_mixed
      const HubArena& hb = sa.hub;
      k_item_class<<<sm_count * 2, 256, 0, st>>>(hb.items, sa.item_count, hb.item_cap, hb.sort_keys[0],
                                                 sa.cls_count);
      A3G_LAUNCH_DONE("k_item_class", st);
      const uint32_t* lists = hb.sort_keys[0];
      constexpr int W = WM == 2 ? 0 : WM;
      const uint64_t item_bound = std::min<uint64_t>(rows_bound + sa.hub.seg_cap, sa.hub.item_cap);
      // lane-group kernels: one pass of 32/G items per warp, grid over the
      // item bound (short-lived CTAs, as the lane kernels)
      auto grp_grid = [&](int G) {
        // a CTA covers (kGrpThreads / 32) warps x (32 / G) items
        return static_cast<int>(std::max<uint64_t>(1, (item_bound * G + kGrpThreads - 1) / kGrpThreads));
      };
      const int lane_grid = static_cast<int>(std::max<uint64_t>(1, (item_bound + 255) / 256));
      const bool lane = sa.kind != A3G_SAMPLER_UNIFORM && sa.f <= 16 &&
                        rows_bound >= lane_min_rows(sa.seg >= 4 * kSegMin) && (WM != 2 || sa.ebits);
      // lane layers may route their longest items (length class >= split) to
      // the lane-group kernel first (A3G_SPLIT_CLS sweeps; off by default)
      static const int split = [] {
        const char* e = std::getenv("A3G_SPLIT_CLS");
        return e ? std::atoi(e) : -1;
      }();
      SampleArgs sl = sa;
      sl.split_cls = lane ? split : -1;
      static const bool fork_env = std::getenv("A3G_SPLIT_FORK") != nullptr;
      fork = lane && split >= 0 && fork_env && aux && aux != st && ev_fork && ev_join;
      cudaStream_t gst = st;
      if (fork) {
        A3G_CUDA(cudaEventRecord(ev_fork, st));
        A3G_CUDA(cudaStreamWaitEvent(aux, ev_fork, 0));
        gst = aux;
      }
      if (!lane || split >= 0) {  // lane groups: the whole layer, or its long items
        if (WM == 2 && sa.kind != A3G_SAMPLER_UNIFORM) {
          if (sa.f <= 8)
            k_stream_grp_mixed<8><<<grp_grid(8), kGrpThreads, 0, gst>>>(sl, lists, sa.cls_count);
          else if (sa.f <= 16)
            k_stream_grp_mixed<16><<<grp_grid(16), kGrpThreads, 0, gst>>>(sl, lists, sa.cls_count);
          else
            k_stream_grp_mixed<32><<<grp_grid(32), kGrpThreads, 0, gst>>>(sl, lists, sa.cls_count);
          A3G_LAUNCH_DONE("k_stream_grp_mixed", gst);
        } else {
          if (sa.f <= 8)
            k_stream_grp<W, 8><<<grp_grid(8), kGrpThreads, 0, gst>>>(sl, lists, sa.cls_count);
          else if (sa.f <= 16)
            k_stream_grp<W, 16><<<grp_grid(16), kGrpThreads, 0, gst>>>(sl, lists, sa.cls_count);
          else
            k_stream_grp<W, 32><<<grp_grid(32), kGrpThreads, 0, gst>>>(sl, lists, sa.cls_count);
          A3G_LAUNCH_DONE("k_stream_grp", gst);
        }
      }
      if (fork) A3G_CUDA(cudaEventRecord(ev_join, aux));
      if (lane) {  // register reservoirs sized to the fanout (exact sizes for the common 5 / 10)
        if (WM == 2) {
          static const bool lane_smem_m = [] {  // shared-memory reservoirs (default; =0: registers, A/B)
            const char* e = std::getenv("A3G_LANE_SMEM");
            return !(e && std::atoi(e) == 0);
          }();
          if (lane_smem_m && sa.f <= 10) {
            if (sa.f == 5)
              k_stream_lane_mixed_s<5><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
            else if (sa.f <= 8)
              k_stream_lane_mixed_s<8><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
            else
              k_stream_lane_mixed_s<10><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
          } else if (sa.f == 5)
            k_stream_lane_mixed<5><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
          else if (sa.f <= 8)
            k_stream_lane_mixed<8><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
          else if (sa.f == 10)
            k_stream_lane_mixed<10><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
          else
            k_stream_lane_mixed<16><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
          A3G_LAUNCH_DONE("k_stream_lane_mixed", st);
        } else {
          static const bool lane_smem = [] {  // shared-memory reservoirs (default; =0: registers, A/B)
            const char* e = std::getenv("A3G_LANE_SMEM");
            return !(e && std::atoi(e) == 0);
          }();
          if (lane_smem && sa.f <= 10) {
            if (sa.f == 5)
              k_stream_lane_s<W, 5><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
            else if (sa.f <= 8)
              k_stream_lane_s<W, 8><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
            else
              k_stream_lane_s<W, 10><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
          } else if (sa.f == 5)
          {
            if (!diag_skip("lane")) k_stream_lane<W, 5><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
          }
          else if (sa.f <= 8)
            k_stream_lane<W, 8><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
          else if (sa.f == 10)
          {
            if (!diag_skip("lane")) k_stream_lane<W, 10><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
          }
          else
            k_stream_lane<W, 16><<<lane_grid, 256, 0, st>>>(sl, lists, sa.cls_count);
          A3G_LAUNCH_DONE("k_stream_lane", st);
        }
      }
    }
    static const int merge_ctas_q = [] {  // hub-merge CTAs per 4 SMs (A3G_MERGE_CTAS4 sweeps)
      const char* e = std::getenv("A3G_MERGE_CTAS4");
      return e ? std::max(1, std::atoi(e)) : 2;  // r01 sweep: 2 (74 CTAs) beat 8 and 4 in the pipeline
    }();
    if (fork) A3G_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
    if (!diag_skip("merge"))
      k_hub_merge<WM><<<std::max(1, sm_count * merge_ctas_q / 4), kMergeThreads, kMergeSmem, st>>>(sa);
    A3G_LAUNCH_DONE("k_hub_merge", st);
  }
}

}  // namespace

// ------------------------------------------------------------ host side ----
void build_edge_bits(const uint32_t* col, uint64_t m, const uint32_t* bits, uint32_t* ebits, int sm_count,
                     cudaStream_t st) {
  k_edge_bits<<<sm_count * 8, 256, 0, st>>>(col, m, bits, ebits);
  A3G_LAUNCH_DONE("k_edge_bits", st);
}

void launch_sample(SamplerState& s, uint32_t n_seeds, double gamma, int kind, uint64_t rng_seed,
                   cudaStream_t st) {
  a3g_graph* g = s.g;
  a3g_cache* c = s.c;
  BatchCounters* ctr = s.d_ctr;
  k_init_counters<<<1, 64, 0, st>>>(ctr, n_seeds);
  A3G_LAUNCH_DONE("k_init_counters", st);
  if (s.check_seeds) {
    k_check_seeds<<<(n_seeds + 255) / 256, 256, 0, st>>>(s.d_seeds, n_seeds, g->n, ctr);
    A3G_LAUNCH_DONE("k_check_seeds", st);
  }
  if (s.cap_inner) A3G_CUDA(cudaMemsetAsync(s.d_inv1, 0xff, s.cap_inner * sizeof(int32_t), st));
  ++s.gtag;
  // ---- seeds phase (sampler.cpp:100-105)
  const uint32_t tag0 = ++s.tag;
  k_mark_list<<<(n_seeds + 255) / 256, 256, 0, st>>>(s.d_seeds, n_seeds, s.d_first, tag0);
  A3G_LAUNCH_DONE("k_mark_list", st);
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
    A3G_LAUNCH_DONE("seed finalize", st);
  }
  // ---- layers (sampler.cpp:107-135)
  int wmode = 0;
  if (kind == A3G_SAMPLER_WEIGHTED && gamma != 1.0) {
    if (c->all_cached)
      wmode = 1;
    else if (!c->none_cached)
      wmode = 2;
  }
  for (uint32_t l = 0; l < s.L; ++l) {
    LayerArena& la = s.layer[l];
    const uint32_t tag = ++s.tag;
    SampleArgs sa{};
    sa.ro = g->d_ro;
    sa.col = g->d_col;
    sa.bits = c->d_bits;
    sa.ebits = c->d_ebits;
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
    sa.big_count = &ctr->hub_big[l];
    sa.cls_count = ctr->icls[l];
    sa.small_count = &ctr->hub_small[l];
    sa.item_count = &ctr->items[l];
    sa.item_work = &ctr->iwork[l];
    sa.positions = &ctr->positions;
    sa.seed = rng_seed;
    sa.gamma = gamma;
    sa.inv_gamma = 1.0 / gamma;
    sa.tie = 64ull * (static_cast<uint64_t>(std::ceil(std::min(gamma, 1e12))) + 1);
    sa.f = la.f;
    sa.layer = l;
    sa.seg = s.seg;
    sa.split_cls = -1;
    sa.tag = tag;
    sa.kind = kind;
    sa.wmode = wmode;
    if (wmode == 1)
      launch_layer_kernels<1>(sa, la.cap_rows, s.sm_count, st, s.stream, s.ev_fork, s.ev_join);
    else if (wmode == 2)
      launch_layer_kernels<2>(sa, la.cap_rows, s.sm_count, st, s.stream, s.ev_fork, s.ev_join);
    else
      launch_layer_kernels<0>(sa, la.cap_rows, s.sm_count, st, s.stream, s.ev_fork, s.ev_join);
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
    if (!diag_skip("fin")) {
      k_fin_count<<<nb, kFinThreads, 0, st>>>(fa);
      k_fin_emit<<<nb, kFinThreads, 0, st>>>(fa);
    }
    A3G_LAUNCH_DONE("layer finalize", st);
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
    A3G_LAUNCH_DONE("k_resolve", st);
  }
}

// cache.cpp:48-68 lookup over an id list: the device of every id (-1 =
// miss; any-device presence is a hit), and the accounting counts
// cnt = [hits, misses, per-device hits...]. With one device the cached
// bitmap decides (device 0); with several, the device map.
__global__ void k_cache_lookup(const uint32_t* ids, uint64_t n, const uint32_t* bits, const int32_t* dmap,
                               int32_t* dev_out, unsigned long long* cnt, uint32_t num_devices) {
  __shared__ unsigned long long s_cnt[2 + kMaxCacheDevices];
  for (uint32_t i = threadIdx.x; i < 2 + num_devices; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t v = ids[i];
    int32_t d;
    if (dmap)
      d = __ldg(dmap + v);
    else
      d = ((__ldg(bits + (v >> 5)) >> (v & 31)) & 1u) ? 0 : -1;
    if (dev_out) dev_out[i] = d;
    if (d < 0) {
      atomicAdd(&s_cnt[1], 1ull);
    } else {
      atomicAdd(&s_cnt[0], 1ull);
      if (static_cast<uint32_t>(d) < num_devices) atomicAdd(&s_cnt[2 + d], 1ull);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 2 + num_devices; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(cnt + i, s_cnt[i]);
}

void launch_cache_lookup(const a3g_cache* c, const uint32_t* d_ids, uint64_t n, int32_t* d_dev,
                         unsigned long long* d_cnt, int sm_count, cudaStream_t st) {
  const uint32_t nd = c->num_devices < kMaxCacheDevices ? c->num_devices : kMaxCacheDevices;
  const int grid = static_cast<int>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(sm_count) * 4));
  k_cache_lookup<<<grid > 0 ? grid : 1, 256, 0, st>>>(d_ids, n, c->d_bits, c->num_devices > 1 ? c->d_map : nullptr,
                                                       d_dev, d_cnt, nd);
  A3G_LAUNCH_DONE("k_cache_lookup", st);
}

void launch_gather_unique(SamplerState& s, float* out, cudaStream_t st) {
  a3g_graph* g = s.g;
  a3g_cache* c = s.c;
  const int bitmode = c->all_cached ? 1 : (c->none_cached ? 0 : 2);
  const uint32_t* uc = &s.d_ctr->ucount[s.L];
  if (g->feat_dtype == A3G_FEAT_BF16)
    k_gather_unique<uint16_t><<<s.sm_count * 4, 256, 0, st>>>(g->view, g->F, s.d_unique, uc, c->d_bits,
                                                               bitmode, out, s.d_ctr);
  else
    k_gather_unique<float><<<s.sm_count * 4, 256, 0, st>>>(g->view, g->F, s.d_unique, uc, c->d_bits, bitmode,
                                                            out, s.d_ctr);
  A3G_LAUNCH_DONE("k_gather_unique", st);
}

void launch_reservoir_list(const uint32_t* d_nb, const double* d_w, uint64_t deg, uint32_t m,
                           uint64_t key, uint64_t c0, int kind, uint32_t* d_out, double* d_keys,
                           cudaStream_t st) {
  k_reservoir_list<<<1, 32, 0, st>>>(d_nb, d_w, deg, m, key, c0, kind, d_out, d_keys);
  A3G_LAUNCH_DONE("k_reservoir_list", st);
}

}  // namespace a3g

