// a3g_internal.cuh -- shared device/host definitions of the B200 hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/a3g.h"

namespace a3g {

// ------------------------------------------------------------ errors -------
struct Error : std::runtime_error {
  a3g_status status;
  Error(a3g_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] inline void raise(a3g_status s, const std::string& m) { throw Error(s, m); }
inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    raise(e == cudaErrorMemoryAllocation ? A3G_ERR_OOM : A3G_ERR_CUDA,
          std::string(what) + ": " + cudaGetErrorString(e));
  }
}
// Thread-local message behind a3g_last_error() (api.cu).
void set_error(const std::string& msg);

// Runs fn, mapping exceptions onto a3g_status (the C-ABI never throws).
template <typename Fn>
a3g_status guard(Fn&& fn) {
  try {
    fn();
    return A3G_OK;
  } catch (const Error& e) {
    set_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return A3G_ERR_OOM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return A3G_ERR_CUDA;
  }
}

#define A3G_CUDA(x) ::a3g::cuda_check((x), #x)
#define A3G_LAUNCH_CHECK(name) ::a3g::cuda_check(cudaGetLastError(), name)

// Launch timeline (diagnostics, A3G_TIMELINE=1): an event after every kernel
// of the traced steps on its stream; a3g_train_steps prints the end times.
void tl_mark(const char* name, cudaStream_t st);
#define A3G_LAUNCH_DONE(name, st)                        \
  do {                                                   \
    ::a3g::cuda_check(cudaGetLastError(), name);         \
    ::a3g::tl_mark(name, st);                            \
  } while (0)

// cudaFuncSetAttribute is per device (context), and the handles may be driven
// from several host threads: `done` holds one bit per device that already
// has the attribute (one std::atomic per kernel instantiation at the call site).
inline void smem_attr_once(std::atomic<uint64_t>& done, const void* fn, size_t bytes) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)),
             "cudaFuncSetAttribute");
  done.fetch_or(bit, std::memory_order_release);
}

// ------------------------------------------------------------ RNG ----------
// include/a3gnn/rng.hpp:13-55, bit-exact on the device.
constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}
__host__ __device__ __forceinline__ uint64_t hash2(uint64_t a, uint64_t b) {
  return mix64(a ^ mix64(b + kPhi));
}
__host__ __device__ __forceinline__ uint64_t hash3(uint64_t a, uint64_t b, uint64_t c) {
  return hash2(hash2(a, b), c);
}
// i-th draw (1-based) of stream `key` (rng.hpp:43-46)
__host__ __device__ __forceinline__ uint64_t draw(uint64_t key, uint64_t i) {
  return mix64(key + i * kPhi);
}
// next_unit (rng.hpp:49): 53-bit uniform in [0,1)
__host__ __device__ __forceinline__ double unit_of(uint64_t x) {
  return (double)(x >> 11) * 0x1.0p-53;
}

// ------------------------------------------------------------ limits -------
constexpr int kMaxLayers = 8;
constexpr uint32_t kInv = 0xffffffffu;
// Length classes of the stream items (sampler.cu k_item_class): quarter-octave
// classes keep the items a warp's lanes share within 1.25x of each other's
// length (A3G_LEN_CLASSES=8: the r01 octave classes)
#ifndef A3G_LEN_CLASSES
#define A3G_LEN_CLASSES 32
#endif
constexpr int kLenClasses = A3G_LEN_CLASSES;
constexpr uint32_t kMaxCacheDevices = 64;  // per-device hit counters of the lookup

// Device-resident per-batch counters (one struct per sampler arena).
struct BatchCounters {
  uint32_t nfront[kMaxLayers + 1];  // frontier size of layer l (nfront[0] = unique seeds)
  uint32_t ucount[kMaxLayers + 1];  // |unique| after phase p (p=0 seeds, p=l+1 after layer l)
  uint32_t edges[kMaxLayers];       // E_l
  uint32_t work[kMaxLayers];        // dynamic row counters of the sampling kernels
  uint32_t hubs[kMaxLayers];        // hub rows registered per layer
  uint32_t segs[kMaxLayers];        // hub segments reserved per layer
  uint32_t items[kMaxLayers];       // stream items appended per layer
  uint32_t iwork[kMaxLayers];       // stream items claimed per layer
  uint32_t hub_big[kMaxLayers];     // hubs with > 8 segments (block merge)
  uint32_t hub_small[kMaxLayers];   // hubs with 1..8 segments (warp merge)
  uint32_t icls[kMaxLayers][kLenClasses];  // stream items per length class (k_item_class)
  uint32_t n_seeds;                 // seeds given (incl. duplicates)
  uint32_t hits, misses;            // retrieve_features accounting
  uint32_t pad;
  uint32_t bad_seeds;               // device-resident seeds >= n seen (k_check_seeds; raised after sync)
  uint32_t pad2;
  unsigned long long positions;     // neighbour positions drawn (sum of frontier degrees, all layers)
};

// ------------------------------------------------------------ feature store -
// Where feature row v lives. loc[v] = (tier << 28) | slot:
// tier r < 15 = HBM shard of device r (local, or an NVLink peer pointer),
// tier 15 = mapped pinned host memory (zero-copy over PCIe). loc == nullptr:
// identity layout, row v at base[0] + v * row_bytes.
constexpr uint32_t kLocShift = 28;
constexpr uint32_t kLocSlotMask = (1u << kLocShift) - 1u;
constexpr uint32_t kTierHost = 15;
constexpr int kMaxTiers = 16;

struct StoreView {
  const uint8_t* base[kMaxTiers];
  const uint32_t* loc;
  uint32_t row_bytes;
};

#ifdef __CUDACC__
// Kernels take StoreView inside a __grid_constant__ parameter so base[tier]
// is an indexed constant-bank load, not a local-memory copy.
__device__ __forceinline__ const uint8_t* row_ptr(const StoreView& s, uint32_t v) {
  if (!s.loc) return s.base[0] + static_cast<uint64_t>(v) * s.row_bytes;
  const uint32_t l = __ldg(s.loc + v);
  return s.base[l >> kLocShift] + static_cast<uint64_t>(l & kLocSlotMask) * s.row_bytes;
}
#endif

}  // namespace a3g

struct a3g_store;

// ---------------------------------------------------------- handles --------
struct a3g_graph {
  int device = 0;
  uint64_t n = 0, m = 0;
  uint32_t F = 0;
  uint32_t pitch = 0;  // feature row pitch in elements (multiple of 8)
  int feat_dtype = A3G_FEAT_F32;
  uint64_t* d_ro = nullptr;
  uint32_t* d_col = nullptr;
  void* d_feat = nullptr;  // n x pitch (f32 or bf16), zero padded
  uint32_t* d_labels = nullptr;
  std::vector<uint64_t> h_ro;       // host copy (validation, degrees)
  std::vector<uint32_t> h_labels;   // host copy
  bool has_features = false;
  uint64_t synth_patched = 0;       // a3g_graph_synthesize_features: elements recomputed on the host
  a3g::StoreView view{};            // how kernels reach feature rows (default: d_feat, identity)
  a3g_store* store = nullptr;       // attached tiered store (a3g_store_create), else null
};

struct a3g_cache {
  a3g_graph* g = nullptr;
  std::vector<int32_t> device_map;
  uint32_t num_devices = 1;
  uint64_t total_cached = 0;
  uint32_t* d_bits = nullptr;  // n bits: cached on any device
  uint32_t* d_ebits = nullptr; // m bits (+1 pad word): cached bit of every CSR edge's target
                               // (partial caches only; the lane-per-item mixed stream)
  int32_t* d_map = nullptr;    // device_map on the device (num_devices > 1 only: per-device lookup)
  std::vector<uint32_t> hot_order;  // cached nodes in placement (hotness) order, a3g_cache_build only
  bool all_cached = false, none_cached = true;
};

struct a3g_comm;
