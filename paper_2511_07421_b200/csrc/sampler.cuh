// sampler.cuh -- k-hop sampler arena (device twin of sampling::SampleBatch,
// sampler.hpp:30-46) and its launch entry points.
#pragma once

#include "a3g_internal.cuh"

namespace a3g {

// Per-layer CSR block, padded: row k (frontier node k) owns slots
// [k*f, k*f + cnt[k]). The reference's edge list of layer l is the row-major
// walk over valid slots (sampler.cpp:125-127).
struct LayerArena {
  uint32_t f = 0;           // fanout
  uint64_t cap_rows = 0;    // frontier capacity
  uint32_t* front = nullptr;      // frontier node ids            [cap_rows]
  uint32_t* front_idx = nullptr;  // unique index of frontier node [cap_rows]
  uint32_t* cnt = nullptr;        // sampled count per row          [cap_rows]
  uint32_t* S = nullptr;          // sampled node ids               [cap_rows*f]
  uint32_t* sidx = nullptr;       // unique index of sampled node   [cap_rows*f]
  double* scratch = nullptr;      // reservoir keys for f > 32 rows [cap_rows*f]
};

// Hub splitting (rows with deg > seg): per-segment local records.
constexpr uint32_t kSegMin = 2048;  // hub segment unit (SamplerState::seg: 4096, or 8192 on dense graphs)
constexpr uint32_t kRecCap = 256;   // record capacity per segment (expected m(1+ln(seg/m)) <= 190 for m <= 32)

struct HubArena {
  uint32_t hub_cap = 0, seg_cap = 0;
  uint32_t* row = nullptr;       // [hub_cap] frontier row of hub h
  uint32_t* seg0 = nullptr;      // [hub_cap] first segment
  uint32_t* nseg = nullptr;      // [hub_cap] #segments (0: handled in-row)
  uint32_t* big = nullptr;       // [hub_cap] hubs with > 8 segments
  uint32_t* small = nullptr;     // [hub_cap] hubs with 1..8 segments
  uint32_t* seg_hub = nullptr;   // [seg_cap] owning hub
  uint32_t* rec_cnt = nullptr;   // [seg_cap]
  uint64_t* tau = nullptr;       // [seg_cap] m-th largest key of the segment (policy key bits)
  uint32_t* tau_ok = nullptr;    // [seg_cap] 0: segment shorter than m (no bound)
  uint32_t* rec_id = nullptr;    // [seg_cap * kRecCap]
  uint64_t* rec_key = nullptr;   // [seg_cap * kRecCap] policy key bits
  uint32_t* slot_last = nullptr; // [seg_cap * 32] uniform kind: last position per slot
  uint32_t item_cap = 0;
  uint4* items = nullptr;        // [item_cap] stream work: (row, begin, end, segment | kInv)
  uint32_t* sort_keys[2] = {nullptr, nullptr};  // [0]: per-length-class item lists (8 x item_cap)
};

struct SamplerState {
  HubArena hub;
  a3g_graph* g = nullptr;
  a3g_cache* c = nullptr;
  uint32_t max_seeds = 0;
  uint32_t L = 0;
  std::vector<uint32_t> fanouts;
  LayerArena layer[kMaxLayers];
  uint64_t cap_unique = 0;
  uint64_t cap_inner = 0;
  uint32_t* d_seeds = nullptr;     // [max_seeds]
  uint32_t* d_front0 = nullptr;    // unique seeds (frontier 0)
  uint32_t* d_unique = nullptr;    // [cap_unique]
  int32_t* d_inv1 = nullptr;       // unique idx (< n_inner) -> row in layer-1 frontier, -1 if none
  uint64_t* d_first = nullptr;     // [n] tagged first position (tag<<32 | ~pos)
  uint64_t* d_gidx = nullptr;      // [n] tagged global index   (gtag<<32 | idx)
  uint4* d_blk = nullptr;          // block partials of the finalize scans
  uint64_t blk_cap = 0;
  BatchCounters* d_ctr = nullptr;
  BatchCounters* h_ctr = nullptr;  // pinned mirror
  uint32_t* h_seeds = nullptr;     // pinned staging of host seeds
  uint32_t tag = 0;                // first-position tag (per phase)
  uint32_t gtag = 0;               // interner tag (per batch)
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;  // fork of a layer's lane-group launch onto `stream`
  // last batch parameters
  uint32_t last_n_seeds = 0;
  bool check_seeds = false;  // seeds came from device memory: range-check them on the device
  bool has_batch = false;
  int sm_count = 148;
  int device = 0;  // the graph's device (kept so destroy never dereferences the graph)
  // Hub segment length. Rows longer than this are split and merged; shorter
  // ones are one item. Longer segments mean fewer merges but longer serial
  // items: 4096 pays on dense graphs (mean degree >= 128, e.g. C2: 0.80 vs
  // 0.88 ms/step), 2048 on sparse ones (C3: 1.24 vs 1.36 ms/step), r01 sweep.
  uint32_t seg = kSegMin;
};

// Launch the whole k-hop sample for seeds already in s.d_seeds (n_seeds on host).
void launch_sample(SamplerState& s, uint32_t n_seeds, double gamma, int kind, uint64_t rng_seed,
                   cudaStream_t st);
// Single explicit neighbour list (test hook for a3g_*_reservoir).
void launch_reservoir_list(const uint32_t* d_nb, const double* d_w, uint64_t deg, uint32_t m,
                           uint64_t key, uint64_t c0, int kind, uint32_t* d_out, double* d_keys,
                           cudaStream_t st);
// cache.cpp:48-68 lookup of n device ids: per-id device (d_dev, may be null)
// and d_cnt[0..2+num_devices) += [hits, misses, per-device hits].
void launch_cache_lookup(const a3g_cache* c, const uint32_t* d_ids, uint64_t n, int32_t* d_dev,
                         unsigned long long* d_cnt, int sm_count, cudaStream_t st);
// Gather unique rows to `out` (device f32, F contiguous) and count hits/misses.
void launch_gather_unique(SamplerState& s, float* out, cudaStream_t st);
// per-edge cached bits of a partial cache: ebits[e / 32] bit e % 32 = bits[col[e]]
void build_edge_bits(const uint32_t* col, uint64_t m, const uint32_t* bits, uint32_t* ebits, int sm_count,
                     cudaStream_t st);

}  // namespace a3g

struct a3g_sampler {
  a3g::SamplerState st;
};
