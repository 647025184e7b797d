// store.cu -- tiered feature store: the B200 placement of the reference's
// static cache (proj/src/cache.cpp:12-46, device_map) -- DESIGN.md §5.
//
//   A3G_STORE_HBM      every row in local HBM (per-GPU replication).
//   A3G_STORE_CACHE    rows with device_map[v] != -1 in local HBM (compact
//                      slots), the misses in mapped pinned host memory that the
//                      gather reads zero-copy over PCIe.
//   A3G_STORE_SHARDED  rank r holds the rows with device_map[v] == r; the
//                      others' shards are NVLink peer loads through peer
//                      pointers (same-process UVA or cudaIpc handles); misses
//                      in mapped pinned host memory.
//
// The kernels see one StoreView (a3g_internal.cuh): loc[v] = (tier<<28)|slot.
// Slots of a shard are the ascending-id order of its rows, so every rank
// derives every other rank's slots from the shared device_map alone.
#include <cstring>
#include <vector>

#include "a3g_internal.cuh"

struct a3g_store {
  a3g_graph* g = nullptr;
  int policy = A3G_STORE_HBM;
  int rank = 0, nranks = 1;
  void* d_local = nullptr;  // this rank's rows (HBM)
  uint64_t n_local = 0;
  void* h_host = nullptr;   // missed rows (pinned, mapped)
  uint64_t n_host = 0;
  uint64_t n_remote = 0;    // rows living on other ranks
  uint32_t* d_loc = nullptr;
  bool peer_ipc[a3g::kMaxTiers] = {};
  a3g::StoreView saved{};   // graph view before attach
  void* saved_feat = nullptr;
  bool saved_has = false;
};

namespace a3g {
namespace {

void encode_rows(const float* features, uint32_t F, uint32_t row_bytes, int dtype, const uint32_t* ids,
                 uint64_t count, uint8_t* dst) {
  for (uint64_t i = 0; i < count; ++i) {
    const float* src = features + static_cast<uint64_t>(ids[i]) * F;
    uint8_t* d = dst + i * row_bytes;
    std::memset(d, 0, row_bytes);
    if (dtype == A3G_FEAT_F32) {
      std::memcpy(d, src, F * 4ull);
    } else {  // round-to-nearest-even bf16, as a3g_graph_create
      uint16_t* o = reinterpret_cast<uint16_t*>(d);
      for (uint32_t c = 0; c < F; ++c) {
        uint32_t x;
        std::memcpy(&x, src + c, 4);
        o[c] = static_cast<uint16_t>((x + 0x7fffu + ((x >> 16) & 1u)) >> 16);
      }
    }
  }
}

// Upload rows `ids` (in order) to a fresh device buffer through a pinned slab.
void* upload_rows(const float* features, uint32_t F, uint32_t row_bytes, int dtype, const std::vector<uint32_t>& ids) {
  void* d = nullptr;
  A3G_CUDA(cudaMalloc(&d, std::max<size_t>(1, ids.size() * static_cast<size_t>(row_bytes))));
  const uint64_t slab = std::max<uint64_t>(1, (64ull << 20) / row_bytes);
  std::vector<uint8_t> stage(std::min<uint64_t>(slab, ids.size() + 1) * row_bytes);
  for (uint64_t i0 = 0; i0 < ids.size(); i0 += slab) {
    const uint64_t cnt = std::min<uint64_t>(slab, ids.size() - i0);
    encode_rows(features, F, row_bytes, dtype, ids.data() + i0, cnt, stage.data());
    A3G_CUDA(cudaMemcpy(static_cast<uint8_t*>(d) + i0 * row_bytes, stage.data(), cnt * row_bytes,
                        cudaMemcpyHostToDevice));
  }
  return d;
}

// Rows `ids` of the graph's own device table (a synthesized papers-scale
// table has no host copy): one warp per row, 16-byte chunks.
__global__ void k_copy_rows(const uint8_t* __restrict__ src, uint32_t rb, const uint32_t* __restrict__ ids,
                            uint64_t count, uint8_t* __restrict__ dst) {
  const uint64_t w = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31, q16 = rb / 16;
  for (uint64_t i = w; i < count; i += nw) {
    const uint4* s = reinterpret_cast<const uint4*>(src + static_cast<uint64_t>(ids[i]) * rb);
    uint4* d = reinterpret_cast<uint4*>(dst + i * rb);
    for (uint32_t q = lane; q < q16; q += 32) d[q] = s[q];
  }
}

// Copies rows `ids` (in order) of g's device table to dst (device, or mapped
// pinned host through device slabs).
void copy_device_rows(const a3g_graph* g, const std::vector<uint32_t>& ids, uint8_t* dst, bool dst_host) {
  const uint32_t rb = g->view.row_bytes;
  const uint64_t slab = std::max<uint64_t>(1, (256ull << 20) / rb);
  uint32_t* d_ids = nullptr;
  uint8_t* d_stage = nullptr;
  A3G_CUDA(cudaMalloc(&d_ids, std::min<uint64_t>(slab, std::max<size_t>(ids.size(), 1)) * 4));
  if (dst_host) A3G_CUDA(cudaMalloc(&d_stage, std::min<uint64_t>(slab, std::max<size_t>(ids.size(), 1)) * rb));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
  for (uint64_t i0 = 0; i0 < ids.size(); i0 += slab) {
    const uint64_t cnt = std::min<uint64_t>(slab, ids.size() - i0);
    A3G_CUDA(cudaMemcpy(d_ids, ids.data() + i0, cnt * 4, cudaMemcpyHostToDevice));
    uint8_t* out = dst_host ? d_stage : dst + i0 * rb;
    k_copy_rows<<<sms * 8, 256>>>(static_cast<const uint8_t*>(g->d_feat), rb, d_ids, cnt, out);
    A3G_LAUNCH_CHECK("k_copy_rows");
    if (dst_host) A3G_CUDA(cudaMemcpy(dst + i0 * rb, d_stage, cnt * rb, cudaMemcpyDeviceToHost));
  }
  A3G_CUDA(cudaDeviceSynchronize());
  cudaFree(d_ids);
  if (d_stage) cudaFree(d_stage);
}

void refresh_view(a3g_store* s) {
  StoreView& v = s->g->view;
  v.base[s->rank] = static_cast<const uint8_t*>(s->d_local);
  v.base[kTierHost] = nullptr;
  if (s->h_host) {
    void* dp = nullptr;
    A3G_CUDA(cudaHostGetDevicePointer(&dp, s->h_host, 0));
    v.base[kTierHost] = static_cast<const uint8_t*>(dp);
  }
  v.loc = s->policy == A3G_STORE_HBM ? nullptr : s->d_loc;
}

}  // namespace
}  // namespace a3g

using namespace a3g;

extern "C" {

a3g_status a3g_store_create(a3g_graph* g, const float* features, const int32_t* device_map, int policy,
                            int rank, int nranks, a3g_store** out) {
  return guard([&] {
    if (!g) raise(A3G_ERR_PARAMETER, "store: graph is required");
    // features == NULL: the rows come from the graph's own device table
    // (a3g_graph_synthesize_features / a3g_graph_create with features)
    if (!features && (!g->d_feat || !g->has_features || g->store))
      raise(A3G_ERR_PARAMETER, "store: host features, or a graph holding its own device table, are required");
    if (policy < A3G_STORE_HBM || policy > A3G_STORE_SHARDED) raise(A3G_ERR_PARAMETER, "store: unknown policy");
    if (nranks < 1 || nranks >= static_cast<int>(kTierHost) || rank < 0 || rank >= nranks)
      raise(A3G_ERR_PARAMETER, "store: rank/nranks out of range (at most 15 devices)");
    if (policy != A3G_STORE_HBM && !device_map) raise(A3G_ERR_PARAMETER, "store: device_map required");
    if (g->store) raise(A3G_ERR_PARAMETER, "store: graph already has a store attached");
    if (g->n > kLocSlotMask) raise(A3G_ERR_PARAMETER, "store: more than 2^28 nodes");
    A3G_CUDA(cudaSetDevice(g->device));
    auto* s = new a3g_store;
    s->g = g;
    s->policy = policy;
    s->rank = policy == A3G_STORE_SHARDED ? rank : 0;
    s->nranks = policy == A3G_STORE_SHARDED ? nranks : 1;
    const uint64_t n = g->n;
    const uint32_t rb = g->view.row_bytes;
    try {
      std::vector<uint32_t> local, host;
      std::vector<uint32_t> loc(policy == A3G_STORE_HBM ? 0 : n);
      std::vector<uint64_t> per_rank(kMaxTiers, 0);
      if (policy == A3G_STORE_HBM) {
        local.resize(n);
        for (uint64_t v = 0; v < n; ++v) local[v] = static_cast<uint32_t>(v);
      } else {
        for (uint64_t v = 0; v < n; ++v) {
          const int32_t d = device_map[v];
          int tier;
          if (d < 0) {
            tier = kTierHost;
          } else if (policy == A3G_STORE_CACHE) {
            tier = 0;
          } else {
            if (d >= nranks) raise(A3G_ERR_PARAMETER, "store: device_map names a device >= nranks");
            tier = d;
          }
          const uint64_t slot = per_rank[tier]++;
          loc[v] = (static_cast<uint32_t>(tier) << kLocShift) | static_cast<uint32_t>(slot);
          if (tier == kTierHost)
            host.push_back(static_cast<uint32_t>(v));
          else if (tier == s->rank)
            local.push_back(static_cast<uint32_t>(v));
          else
            ++s->n_remote;
        }
      }
      s->n_local = local.size();
      if (features) {
        s->d_local = upload_rows(features, g->F, rb, g->feat_dtype, local);
      } else {
        A3G_CUDA(cudaMalloc(&s->d_local, std::max<size_t>(1, local.size() * static_cast<size_t>(rb))));
        copy_device_rows(g, local, static_cast<uint8_t*>(s->d_local), false);
      }
      if (!host.empty()) {
        s->n_host = host.size();
        A3G_CUDA(cudaHostAlloc(&s->h_host, host.size() * static_cast<size_t>(rb),
                               cudaHostAllocMapped | cudaHostAllocPortable));
        if (features)
          encode_rows(features, g->F, rb, g->feat_dtype, host.data(), host.size(),
                      static_cast<uint8_t*>(s->h_host));
        else
          copy_device_rows(g, host, static_cast<uint8_t*>(s->h_host), true);
      }
      if (!loc.empty()) {
        A3G_CUDA(cudaMalloc(&s->d_loc, n * 4));
        A3G_CUDA(cudaMemcpy(s->d_loc, loc.data(), n * 4, cudaMemcpyHostToDevice));
      }
    } catch (...) {
      if (s->d_local) cudaFree(s->d_local);
      if (s->h_host) cudaFreeHost(s->h_host);
      if (s->d_loc) cudaFree(s->d_loc);
      delete s;
      throw;
    }
    s->saved = g->view;
    s->saved_has = g->has_features;
    g->view = StoreView{};
    g->view.row_bytes = rb;
    g->store = s;
    g->has_features = true;
    refresh_view(s);
    *out = s;
  });
}

a3g_status a3g_store_info(const a3g_store* s, uint64_t* local_rows, uint64_t* host_rows, uint64_t* remote_rows) {
  return guard([&] {
    if (local_rows) *local_rows = s->n_local;
    if (host_rows) *host_rows = s->n_host;
    if (remote_rows) *remote_rows = s->n_remote;
  });
}

a3g_status a3g_store_local_ptr(a3g_store* s, void** dev_ptr) {
  return guard([&] { *dev_ptr = s->d_local; });
}

a3g_status a3g_store_set_peer(a3g_store* s, int rank, void* dev_ptr) {
  return guard([&] {
    if (s->policy != A3G_STORE_SHARDED) raise(A3G_ERR_PARAMETER, "store: peers need A3G_STORE_SHARDED");
    if (rank < 0 || rank >= s->nranks || rank == s->rank) raise(A3G_ERR_PARAMETER, "store: bad peer rank");
    cudaPointerAttributes at{};
    A3G_CUDA(cudaPointerGetAttributes(&at, dev_ptr));
    if (at.type == cudaMemoryTypeDevice && at.device != s->g->device) {
      const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "cudaDeviceEnablePeerAccess");
      cudaGetLastError();
    }
    s->g->view.base[rank] = static_cast<const uint8_t*>(dev_ptr);
  });
}

a3g_status a3g_store_ipc_handle(a3g_store* s, uint8_t handle[64]) {
  return guard([&] {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
    cudaIpcMemHandle_t h;
    A3G_CUDA(cudaSetDevice(s->g->device));
    A3G_CUDA(cudaIpcGetMemHandle(&h, s->d_local));
    std::memcpy(handle, &h, 64);
  });
}

a3g_status a3g_store_open_peer(a3g_store* s, int rank, const uint8_t handle[64]) {
  return guard([&] {
    if (s->policy != A3G_STORE_SHARDED) raise(A3G_ERR_PARAMETER, "store: peers need A3G_STORE_SHARDED");
    if (rank < 0 || rank >= s->nranks || rank == s->rank) raise(A3G_ERR_PARAMETER, "store: bad peer rank");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void* p = nullptr;
    A3G_CUDA(cudaSetDevice(s->g->device));
    A3G_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    s->peer_ipc[rank] = true;
    s->g->view.base[rank] = static_cast<const uint8_t*>(p);
  });
}

void a3g_store_destroy(a3g_store* s) {
  if (!s) return;
  a3g_graph* g = s->g;
  cudaSetDevice(g->device);
  cudaDeviceSynchronize();
  for (int r = 0; r < kMaxTiers; ++r)
    if (s->peer_ipc[r] && g->view.base[r]) cudaIpcCloseMemHandle(const_cast<uint8_t*>(g->view.base[r]));
  if (g->store == s) {
    g->view = s->saved;
    g->has_features = s->saved_has;
    g->store = nullptr;
  }
  if (s->d_local) cudaFree(s->d_local);
  if (s->h_host) cudaFreeHost(s->h_host);
  if (s->d_loc) cudaFree(s->d_loc);
  delete s;
}

}  // extern "C"
