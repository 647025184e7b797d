// comm.cpp -- NCCL glue for the data-parallel gradient sum.
//
// Replaces the in-process arithmetic mean sync_gradients (proj/src/trainer.cpp:213-229)
// with an allreduce(sum) of n_k-weighted gradients over NVLink. NCCL is
// resolved with dlopen at communicator creation so the library loads on
// hosts without NCCL (and reuses the libnccl.so.2 already mapped by torch).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "a3g_internal.cuh"

struct a3g_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
  // host transport (a3g_comm_create_host): the packed buffer goes through a
  // pinned host copy to the caller's allreduce
  a3g_allreduce_fn host_fn = nullptr;
  void* host_user = nullptr;
  float* h_buf = nullptr;
  size_t h_cap = 0;
};

namespace a3g {
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*err)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(api.h, "ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(api.h, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(api.h, "ncclAllReduce"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(api.h, "ncclCommDestroy"));
    api.err = reinterpret_cast<decltype(api.err)>(dlsym(api.h, "ncclGetErrorString"));
  });
  if (!api.h || !api.get_unique_id || !api.init_rank || !api.all_reduce)
    raise(A3G_ERR_NCCL, "NCCL (libnccl.so.2) not available");
  return api;
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    raise(A3G_ERR_NCCL, std::string(what) + ": " + (nccl().err ? nccl().err(r) : "nccl error"));
}
}  // namespace

void comm_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

a3g_comm* comm_create(const uint8_t id_bytes[128], int nranks, int rank, int device) {
  ncclUniqueId id;
  std::memcpy(id.internal, id_bytes, 128);
  A3G_CUDA(cudaSetDevice(device));
  auto* c = new a3g_comm;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  try {
    nccl_check(nccl().init_rank(&c->comm, nranks, id, rank), "ncclCommInitRank");
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

a3g_comm* comm_create_host(int nranks, int rank, a3g_allreduce_fn fn, void* user) {
  if (!fn) raise(A3G_ERR_PARAMETER, "comm: allreduce callback is null");
  if (nranks < 1 || rank < 0 || rank >= nranks) raise(A3G_ERR_PARAMETER, "comm: bad rank / nranks");
  auto* c = new a3g_comm;
  c->nranks = nranks;
  c->rank = rank;
  c->host_fn = fn;
  c->host_user = user;
  return c;
}

void comm_destroy(a3g_comm* c) {
  if (!c) return;
  if (c->comm && nccl().destroy) nccl().destroy(c->comm);
  if (c->h_buf) cudaFreeHost(c->h_buf);
  delete c;
}

void comm_allreduce_sum(a3g_comm* comm, float* buf, size_t count, cudaStream_t st) {
  if (comm->host_fn) {
    // the gradients of this step are complete once the stream reaches here
    if (count > comm->h_cap) {
      if (comm->h_buf) cudaFreeHost(comm->h_buf);
      comm->h_buf = nullptr;
      A3G_CUDA(cudaMallocHost(&comm->h_buf, count * sizeof(float)));
      comm->h_cap = count;
    }
    A3G_CUDA(cudaMemcpyAsync(comm->h_buf, buf, count * sizeof(float), cudaMemcpyDeviceToHost, st));
    A3G_CUDA(cudaStreamSynchronize(st));
    if (comm->host_fn(comm->h_buf, count, comm->host_user) != 0)
      raise(A3G_ERR_NCCL, "comm: host allreduce callback failed");
    A3G_CUDA(cudaMemcpyAsync(buf, comm->h_buf, count * sizeof(float), cudaMemcpyHostToDevice, st));
    A3G_CUDA(cudaStreamSynchronize(st));  // h_buf is reused by the next step
    return;
  }
  nccl_check(nccl().all_reduce(buf, buf, count, ncclFloat32, ncclSum, comm->comm, st), "ncclAllReduce");
}

}  // namespace a3g
