// synth.cu -- device synthesis of the power-law generator's features for
// papers-scale graphs (BASELINE config 5: 111M nodes x 128-d bf16 = 28 GB,
// whose f32 host table would not fit the host). The formula is the
// reference's fill_features_and_masks (proj/src/generators.cpp:12-24): element
// (v, d) is the Box-Muller Gaussian of draws 2(v*F+d)+1, +2 of the noise
// substream, plus 1.0f at d == label % F. The topology, labels and masks come
// from the host generator at feat_dim 1 (they never depend on F).
// fp64 log/sqrt/cos of the device library can differ from glibc by an ulp,
// which changes the f32 (then bf16) value of ~1e-9 of the elements; parity at
// this scale is sampling-only.
#include <cstring>

#include "a3g_internal.cuh"

namespace a3g {
namespace {

template <typename T>
__device__ __forceinline__ T enc(float x);
template <>
__device__ __forceinline__ float enc<float>(float x) {
  return x;
}
template <>
__device__ __forceinline__ uint16_t enc<uint16_t>(float x) {
  const uint32_t u = __float_as_uint(x);
  return static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);  // RNE, as a3g_graph_create
}

template <typename T>
__global__ void k_synth_features(uint64_t noise_key, uint64_t n, uint32_t F, uint32_t pitch, const uint32_t* labels,
                                  T* out) {
  const uint64_t total = n * pitch;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t v = i / pitch;
    const uint32_t d = static_cast<uint32_t>(i - v * pitch);
    float x = 0.f;
    if (d < F) {
      const uint64_t c = 2 * (v * F + d);
      double u1 = unit_of(draw(noise_key, c + 1));
      const double u2 = unit_of(draw(noise_key, c + 2));
      if (u1 <= 0.0) u1 = 0x1.0p-53;
      x = static_cast<float>(sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925 * u2));
      if (d == labels[v] % F) x += 1.0f;
    }
    out[i] = enc<T>(x);
  }
}

}  // namespace
}  // namespace a3g

using namespace a3g;

extern "C" a3g_status a3g_graph_synthesize_features(a3g_graph* g, uint32_t feat_dim, int feat_dtype, uint64_t seed) {
  return guard([&] {
    if (g->has_features || g->store) raise(A3G_ERR_PARAMETER, "synthesize_features: graph already has features");
    if (feat_dim < 1) raise(A3G_ERR_PARAMETER, "synthesize_features: feat_dim must be >= 1");
    A3G_CUDA(cudaSetDevice(g->device));
    g->F = feat_dim;
    g->pitch = (feat_dim + 7) / 8 * 8;
    g->feat_dtype = feat_dtype;
    const size_t esz = feat_dtype == A3G_FEAT_BF16 ? 2 : 4;
    const size_t row_bytes = static_cast<size_t>(g->pitch) * esz;
    void* d = nullptr;
    A3G_CUDA(cudaMalloc(&d, std::max<size_t>(1, g->n * row_bytes)));
    // generator streams (host_graph.cpp / generators.cpp): rng = (seed, 0x97a3), noise = substream 0xfea7
    const uint64_t rng_key = hash2(seed, 0x97a3);
    const uint64_t noise_key = hash2(rng_key, 0xfea7ull ^ 0xd6e8feb86659fd93ull);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device);
    if (feat_dtype == A3G_FEAT_BF16)
      k_synth_features<uint16_t><<<sms * 8, 256>>>(noise_key, g->n, feat_dim, g->pitch, g->d_labels,
                                                   static_cast<uint16_t*>(d));
    else
      k_synth_features<float><<<sms * 8, 256>>>(noise_key, g->n, feat_dim, g->pitch, g->d_labels,
                                                static_cast<float*>(d));
    A3G_LAUNCH_CHECK("k_synth_features");
    A3G_CUDA(cudaDeviceSynchronize());
    g->d_feat = d;
    g->view = StoreView{};
    g->view.base[0] = static_cast<const uint8_t*>(d);
    g->view.loc = nullptr;
    g->view.row_bytes = static_cast<uint32_t>(row_bytes);
    g->has_features = true;
  });
}
