// gemm_tc.cu -- the dense update of the mean-GCN on the 5th-generation tensor
// cores (tcgen05.mma, accumulators in TMEM), trainer.cpp:110-113 and :203-204:
//
//   k_h1_tc   h1 = ReLU(agg_inner . W1)           M = inner rows, N = H, K = F
//   k_dw1_tc  dW1 = agg_inner^T . (dh1 * [h1>0])  M = F,          N = H, K = inner rows
//
// Precision: fp32 operands are split three ways, x = x0 + x1 + x2 with
// x0 = bf16(x), x1 = bf16(x - x0), x2 = bf16(x - x0 - x1) (|x - sum| <= 2^-25|x|),
// and D accumulates the six products of total order <= 2 (x0y0, x0y1, x1y0,
// x0y2, x2y0, x1y1; kind::f16 MMAs, fp32 accumulation in TMEM): ~2^-24
// relative per product, i.e. fp32-class results from the bf16 tensor pipe.
// (A two-way split, ~2^-17, flips the ReLU mask of near-zero h1 entries ~100x
// more often than fp32 does and breaks the 1e-3 gradient bar.)
//
// Structure (one CTA = 4 warps, 128-lane TMEM accumulator, cta_group::1):
// all 128 threads stage an fp32 block into shared memory as three bf16 terms in the
// canonical no-swizzle core-matrix layout (8 rows x 16 bytes per core matrix),
// fence the generic->async proxy, and one thread issues the MMAs; the MMAs'
// completion (tcgen05.commit -> mbarrier) releases the stage, so staging of
// block k+1 overlaps the MMAs of block k (2 stages). The epilogue reads TMEM
// with tcgen05.ld (warp w owns lanes 32w..32w+31).
#include <cuda_bf16.h>

#include <algorithm>

#include "ptx.cuh"
#include "trainer.cuh"

namespace a3g {
namespace {

constexpr int kTcThreads = 256;  // 8 warps: conversion throughput; warps 0-3 own the TMEM lanes
constexpr int kPerThr = 2048 / kTcThreads;  // float4 of a 128 x 64 (or 64 x 128) block per thread
constexpr uint32_t kCore = 128;  // bytes per core matrix (8 rows x 16 B)

// ---------------------------------------------------------------- PTX ------
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(ptx::smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] . B[smem]^T, kind::f16 (bf16 in, fp32 accumulate)
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on `bar` when every MMA issued so far by this thread has completed
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   ptx::smem_u32(bar))
               : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns of this warp's TMEM sub-partition
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor, no swizzle (layout type 0), version 1.
// lbo / sbo: byte strides between core matrices along the leading (K for
// K-major, K for MN-major as well -- see DESIGN.md §3) and strided dimension.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
// Instruction descriptor kind::f16: D fp32, A/B bf16, M = 128, N = n.
__device__ __forceinline__ uint32_t idesc_bf16(uint32_t n, bool a_mn_major, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn_major ? 1u << 15 : 0u) | (b_mn_major ? 1u << 16 : 0u) |
         ((n >> 3) << 17) | ((128u >> 4) << 24);
}

constexpr int kParts = 3;  // bf16 terms per fp32 operand

// MMA N (and TMEM columns) for hidden width H: 16, 32, 64, 128 or 256
__host__ __device__ __forceinline__ uint32_t hn_of(uint32_t H) {
  return H <= 16 ? 16u : H <= 32 ? 32u : H <= 64 ? 64u : H <= 128 ? 128u : 256u;
}
__host__ __device__ __forceinline__ uint32_t tmem_cols_of(uint32_t HN) { return HN < 32 ? 32u : HN; }

__device__ __forceinline__ void split3(float x, __nv_bfloat16 (&p)[kParts]) {
  p[0] = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(p[0]);
  p[1] = __float2bfloat16_rn(r1);
  p[2] = __float2bfloat16_rn(r1 - __bfloat162float(p[1]));
}

// Store 4 consecutive-column values of (row, col..col+3) as the three bf16
// terms (part i at base + i*part_bytes) into the core-matrix tiles: core
// (rg, cg) at rg*rs + cg*cs bytes, row r%8 at 16 B, column c%8 at 2 B.
__device__ __forceinline__ void put4(uint8_t* base, uint32_t part_bytes, uint32_t row, uint32_t col, uint32_t rs,
                                     uint32_t cs, float4 v) {
  const uint32_t off = (row >> 3) * rs + (col >> 3) * cs + (row & 7) * 16 + (col & 7) * 2;
  __nv_bfloat16 t[4][kParts];
  split3(v.x, t[0]);
  split3(v.y, t[1]);
  split3(v.z, t[2]);
  split3(v.w, t[3]);
#pragma unroll
  for (int i = 0; i < kParts; ++i) {
    __nv_bfloat16 q[4] = {t[0][i], t[1][i], t[2][i], t[3][i]};
    *reinterpret_cast<uint2*>(base + i * part_bytes + off) = *reinterpret_cast<const uint2*>(q);
  }
}

// Issue one K step: the six products of total order <= 2, (A part, B part) =
// (0,0) (0,1) (1,0) (0,2) (2,0) (1,1).

__device__ __forceinline__ void mma_step6(uint32_t tmem, const uint32_t (&a_addr)[kParts],
                                          const uint32_t (&b_addr)[kParts], uint32_t a_lbo, uint32_t a_sbo,
                                          uint32_t b_lbo, uint32_t b_sbo, uint32_t idesc, bool first) {
#pragma unroll
  for (int t = 0; t < 6; ++t) {
    const int ia = t == 0 || t == 1 || t == 3 ? 0 : (t == 5 ? 1 : (t == 2 ? 1 : 2));
    const int ib = t == 0 || t == 2 || t == 4 ? 0 : (t == 5 ? 1 : (t == 1 ? 1 : 2));
    mma_bf16(tmem, smem_desc(a_addr[ia], a_lbo, a_sbo), smem_desc(b_addr[ib], b_lbo, b_sbo), idesc,
             (first && t == 0) ? 0u : 1u);
  }
}

struct TcArgs {
  const float* agg;      // agg_inner, rows x pitch (fp32)
  uint32_t pitch, F, H, HN;
  const uint32_t* n_inner;
  const float* w1;       // F x H
  const float* dh1;      // rows x H
  float* h1;             // rows x H (k_h1_tc out; k_dw1_tc in: the ReLU mask)
  float* part;           // k_dw1_tc: nsplit x F x H partial dW1
  uint32_t k_pad;        // k_h1_tc: F rounded up to 64
  uint32_t rows_per_split;
  uint32_t kb_per_split; // k_h1_tc: K blocks per split (gridDim.y splits)
  float* hpart;          // k_h1_tc with > 1 split: [split][rows][H] pre-ReLU partials
  uint32_t part_rows;    // row capacity of hpart
};

// cp.async (LDGSTS) 16 B global -> shared; src_size 0 zero-fills (the source
// is not read). The f32 blocks of agg_inner land in a staging buffer with no
// register cost, one block ahead of the conversion + MMAs.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ptx::smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr uint32_t kStgBytes = 128 * 64 * 4;   // f32 staging block (32 KB)
constexpr uint32_t kPartBytes = 128 * 64 * 2;  // one bf16 term of a 128 x 64 block

// ------------------------------------------------------------- forward -----
// CTA = 128 inner rows (M). Per K block of 64 features: cp.async of the f32
// agg block (kb+1 in flight while kb converts), conversion to three bf16
// terms (A: K-major, 8-row groups at 128 B, 8-col groups at 2 KB) and of the
// W1^T block (B: K-major, N = HN), then 4 K-steps x 6 MMAs by one thread.
// smem: stg[2] | A terms[3] | B terms[3] (HN x 64).
__global__ void __launch_bounds__(kTcThreads) k_h1_tc(const __grid_constant__ TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  const uint32_t n = *a.n_inner;
  const uint32_t r0 = blockIdx.x * 128;
  if (r0 >= n) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* stg = reinterpret_cast<float*>(smem);
  uint8_t* apart = smem + 2 * kStgBytes;
  uint8_t* bpart = apart + kParts * kPartBytes;
  const uint32_t b_part = a.HN * 64 * 2;
  const uint32_t b_cs = (a.HN / 8) * kCore;  // B: core (n/8, k/8) at (k/8)*b_cs + (n/8)*128
  if (warp == 0) tmem_alloc(&tmem_slot, tmem_cols_of(a.HN));
  if (tid == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  auto issue = [&](uint32_t kb) {
    float* dst = stg + (kb & 1) * (kStgBytes / 4);
#pragma unroll
    for (int j = 0; j < kPerThr; ++j) {
      const uint32_t i = tid + j * kTcThreads, rr = i >> 4, c = (i & 15) * 4;
      const uint32_t row = r0 + rr, col = kb * 64 + c;
      const bool ok = row < n && col < a.pitch;
      cp_async16(dst + rr * 64 + c, ok ? a.agg + static_cast<uint64_t>(row) * a.pitch + col : a.agg, ok);
    }
    cp_async_commit();
  };
  // split-K: this CTA's K blocks [kb0, kb0 + nkb); local index t drives the
  // double buffer and the mbarrier phases
  const uint32_t kb0 = blockIdx.y * a.kb_per_split;
  const uint32_t nkb = min(a.k_pad / 64 - kb0, a.kb_per_split);
  issue(kb0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t idesc = idesc_bf16(a.HN, false, false);
  for (uint32_t t = 0; t < nkb; ++t) {
    const uint32_t kb = kb0 + t;
    if (t + 1 < nkb) {
      issue(kb + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();                                // block t staged by every thread
    if (t >= 1) ptx::mbar_wait(&bar, (t - 1) & 1);  // MMAs of t-1 done reading the terms
    const float* src = stg + (kb & 1) * (kStgBytes / 4);
#pragma unroll 4
    for (int j = 0; j < kPerThr; ++j) {
      const uint32_t i = tid + j * kTcThreads, rr = i >> 4, c = (i & 15) * 4;
      put4(apart, kPartBytes, rr, c, kCore, 16 * kCore, *reinterpret_cast<const float4*>(src + rr * 64 + c));
    }
    for (uint32_t i = tid; i < a.HN * 16; i += kTcThreads) {  // W1^T block (L1/L2-resident W1)
      const uint32_t nn = i >> 4, c = (i & 15) * 4, k = kb * 64 + c;
      float t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) t[j] = (nn < a.H && k + j < a.F) ? __ldg(a.w1 + (k + j) * a.H + nn) : 0.f;
      put4(bpart, b_part, nn, c, kCore, b_cs, make_float4(t[0], t[1], t[2], t[3]));
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (uint32_t s = 0; s < 4; ++s) {
        uint32_t aa[kParts], bb[kParts];
#pragma unroll
        for (int i = 0; i < kParts; ++i) {
          aa[i] = ptx::smem_u32(apart + i * kPartBytes) + s * 2 * 16 * kCore;
          bb[i] = ptx::smem_u32(bpart + i * b_part) + s * 2 * b_cs;
        }
        mma_step6(tmem, aa, bb, 16 * kCore, kCore, b_cs, kCore, idesc, (t | s) == 0);
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  ptx::mbar_wait(&bar, (nkb - 1) & 1);
  tc_fence_after();
  const bool split = gridDim.y > 1;
  float* out = split ? a.hpart + (static_cast<uint64_t>(blockIdx.y) * a.part_rows) * a.H : a.h1;
  // epilogue: TMEM -> shared tile [128][HN + 1] (warp w owns rows 32w..) ->
  // coalesced row-major stores of the 128 x H block (the MMAs are done: the
  // staging buffers are free)
  float* tile = reinterpret_cast<float*>(smem);
  const uint32_t ts = a.HN + 1;
  for (uint32_t c0 = 0; warp < 4 && c0 < a.HN; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) tile[(warp * 32 + lane) * ts + c0 + j] = split ? v[j] : fmaxf(v[j], 0.f);
  }
  __syncthreads();
  const uint32_t rows = min(128u, n - r0);
  for (uint32_t i = tid; i < rows * a.H; i += kTcThreads) {
    const uint32_t rr = i / a.H, c = i - rr * a.H;
    out[static_cast<uint64_t>(r0 + rr) * a.H + c] = tile[rr * ts + c];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, tmem_cols_of(a.HN));
}

// ------------------------------------------------------------ backward -----
// CTA (feature tile blockIdx.x, row split blockIdx.y): per K block of 64 rows,
// cp.async of the f32 agg block (64 rows x 128 features) and of the matching
// dh1 / h1 rows; conversion to A = agg^T terms (MN-major: feature groups at
// 128 B, row groups at 2 KB) and B = G = dh1 * [h1 > 0] terms (MN-major,
// N = HN); 4 K-steps x 6 MMAs accumulate over the split's rows in TMEM.
// smem: stgA[2] | stgG[2] (dh1 | h1, 64 x H each) | A terms[3] | G terms[3].
__global__ void __launch_bounds__(kTcThreads) k_dw1_tc(const __grid_constant__ TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  const uint32_t n = *a.n_inner;
  const uint32_t f0 = blockIdx.x * 128;
  const uint32_t rb = blockIdx.y * a.rows_per_split;
  const uint32_t re = min(n, rb + a.rows_per_split);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* out = a.part + static_cast<uint64_t>(blockIdx.y) * a.F * a.H;
  if (rb >= re) {  // empty split: zero partial
    for (uint32_t i = tid; i < 128 * a.H; i += kTcThreads) {
      const uint32_t f = f0 + i / a.H;
      if (f < a.F) out[static_cast<uint64_t>(f) * a.H + i % a.H] = 0.f;
    }
    return;
  }
  const uint32_t H = a.H;
  float* stg = reinterpret_cast<float*>(smem);
  uint8_t* apart = smem + 2 * kStgBytes;
  uint8_t* gpart = apart + kParts * kPartBytes;
  const uint32_t g_part = 64 * a.HN * 2;
  const uint32_t g_rs = (a.HN / 8) * kCore;  // G core (row/8, h/8) at (row/8)*g_rs + (h/8)*128
  if (warp == 0) tmem_alloc(&tmem_slot, tmem_cols_of(a.HN));
  if (tid == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  auto issue = [&](uint32_t kb) {
    const uint32_t kr0 = rb + kb * 64;
    float* dst = stg + (kb & 1) * (kStgBytes / 4);
#pragma unroll
    for (int j = 0; j < kPerThr; ++j) {
      const uint32_t i = tid + j * kTcThreads, rr = i >> 5, c = (i & 31) * 4;
      const uint32_t row = kr0 + rr, f = f0 + c;
      const bool ok = row < re && f < a.pitch;
      cp_async16(dst + rr * 128 + c, ok ? a.agg + static_cast<uint64_t>(row) * a.pitch + f : a.agg, ok);
    }
    cp_async_commit();
  };
  issue(0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t idesc = idesc_bf16(a.HN, true, true);
  const uint32_t nkb = (re - rb + 63) / 64;
  for (uint32_t kb = 0; kb < nkb; ++kb) {
    if (kb + 1 < nkb) {
      issue(kb + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (kb >= 1) ptx::mbar_wait(&bar, (kb - 1) & 1);
    const float* src = stg + (kb & 1) * (kStgBytes / 4);
#pragma unroll 4
    for (int j = 0; j < kPerThr; ++j) {
      const uint32_t i = tid + j * kTcThreads, rr = i >> 5, c = (i & 31) * 4;
      put4(apart, kPartBytes, rr, c, 16 * kCore, kCore, *reinterpret_cast<const float4*>(src + rr * 128 + c));
    }
    // G = dh1 * [h1 > 0] (trainer.cpp:200) of rows kr0.., read straight from
    // global (row-major, H floats per row: consecutive threads, consecutive h)
    const uint32_t kr0 = rb + kb * 64;
    for (uint32_t i = tid; i < 64 * (a.HN / 4); i += kTcThreads) {
      const uint32_t rr = i / (a.HN / 4), c = (i % (a.HN / 4)) * 4;
      const uint32_t row = kr0 + rr;
      float t[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t h = c + j;
        const uint64_t o = static_cast<uint64_t>(row) * H + h;
        t[j] = (row < re && h < H && __ldg(a.h1 + o) > 0.f) ? __ldg(a.dh1 + o) : 0.f;
      }
      put4(gpart, g_part, rr, c, g_rs, kCore, make_float4(t[0], t[1], t[2], t[3]));
    }
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (uint32_t s = 0; s < 4; ++s) {
        // K step s = rows 16s..16s+15 = row groups 2s, 2s+1
        uint32_t aa[kParts], bb[kParts];
#pragma unroll
        for (int i = 0; i < kParts; ++i) {
          aa[i] = ptx::smem_u32(apart + i * kPartBytes) + s * 2 * 16 * kCore;
          bb[i] = ptx::smem_u32(gpart + i * g_part) + s * 2 * g_rs;
        }
        // MN-major: LBO = stride between K (row) groups, SBO = between M/N groups
        mma_step6(tmem, aa, bb, 16 * kCore, kCore, g_rs, kCore, idesc, (kb | s) == 0);
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  ptx::mbar_wait(&bar, (nkb - 1) & 1);
  tc_fence_after();
  // epilogue through a shared tile, as k_h1_tc: coalesced stores of the
  // 128-feature x H partial
  float* tile = reinterpret_cast<float*>(smem);
  const uint32_t ts = a.HN + 1;
  for (uint32_t c0 = 0; warp < 4 && c0 < a.HN; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) tile[(warp * 32 + lane) * ts + c0 + j] = v[j];
  }
  __syncthreads();
  const uint32_t nf = min(128u, a.F - f0);
  for (uint32_t i = tid; i < nf * H; i += kTcThreads) {
    const uint32_t ff = i / H, c = i - ff * H;
    out[static_cast<uint64_t>(f0 + ff) * H + c] = tile[ff * ts + c];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, tmem_cols_of(a.HN));
}

// h1 = ReLU(sum of the split-K partials), in split order (deterministic).
__global__ void k_h1_reduce(const float* hpart, uint32_t nsplit, uint32_t part_rows, const uint32_t* n_inner,
                            uint32_t H, float* h1) {
  const uint64_t total = static_cast<uint64_t>(*n_inner) * H;
  const uint64_t stride = static_cast<uint64_t>(part_rows) * H;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    float v = 0.f;
    for (uint32_t k = 0; k < nsplit; ++k) v += hpart[k * stride + i];
    h1[i] = fmaxf(v, 0.f);
  }
}

}  // namespace

size_t tc_h1_smem(uint32_t /*F*/, uint32_t H) {
  const uint32_t HN = hn_of(H);
  const size_t main = 2ull * kStgBytes + kParts * kPartBytes + static_cast<size_t>(kParts) * HN * 64 * 2;
  return std::max<size_t>(main, static_cast<size_t>(128) * (HN + 1) * 4);  // epilogue tile
}
size_t tc_dw1_smem(uint32_t H) {
  const uint32_t HN = hn_of(H);
  const size_t main = 2ull * kStgBytes + kParts * kPartBytes + static_cast<size_t>(kParts) * 64 * HN * 2;
  return std::max<size_t>(main, static_cast<size_t>(128) * (HN + 1) * 4);
}

void launch_h1_tc(TrainerState& t, const float* agg, const uint32_t* n_inner, float* h1, cudaStream_t st) {
  TcArgs a{};
  a.agg = agg;
  a.pitch = t.pitch;
  a.F = t.F;
  a.H = t.H;
  a.HN = hn_of(t.H);
  a.n_inner = n_inner;
  a.w1 = t.d_w1;
  a.h1 = h1;
  a.k_pad = (t.F + 63) / 64 * 64;
  // split K so the grid covers ~4 CTAs per SM (the row tiles alone are < 1 wave)
  const uint32_t tiles = static_cast<uint32_t>((t.cap_inner + 127) / 128);
  const uint32_t nkb = a.k_pad / 64;
  uint32_t ksplit = tiles >= static_cast<uint32_t>(t.sm_count)
                        ? 1u
                        : std::min<uint32_t>(std::min<uint32_t>(nkb, t.h1_split_cap),
                                             std::max<uint32_t>(1, (4u * t.sm_count + tiles - 1) / tiles));
  a.kb_per_split = (nkb + ksplit - 1) / ksplit;
  ksplit = (nkb + a.kb_per_split - 1) / a.kb_per_split;
  a.hpart = t.d_hpart;
  a.part_rows = static_cast<uint32_t>(t.cap_inner);
  const size_t smem = tc_h1_smem(t.F, t.H);
  A3G_CUDA(cudaFuncSetAttribute(k_h1_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  k_h1_tc<<<dim3(tiles, ksplit), kTcThreads, smem, st>>>(a);
  A3G_LAUNCH_DONE("k_h1_tc", st);
  t.h1_split_used = ksplit > 1;
  if (ksplit > 1) {
    k_h1_reduce<<<t.sm_count * 2, 256, 0, st>>>(t.d_hpart, ksplit, a.part_rows, n_inner, t.H, h1);
    A3G_LAUNCH_DONE("k_h1_reduce", st);
  }
}

void launch_dw1_tc(const TrainerState& t, const float* agg, const uint32_t* n_inner, const float* h1,
                   const float* dh1, float* part, uint32_t nsplit, cudaStream_t st) {
  TcArgs a{};
  a.agg = agg;
  a.pitch = t.pitch;
  a.F = t.F;
  a.H = t.H;
  a.HN = hn_of(t.H);
  a.n_inner = n_inner;
  a.h1 = const_cast<float*>(h1);
  a.dh1 = dh1;
  a.part = part;
  a.rows_per_split = static_cast<uint32_t>((t.cap_inner + nsplit - 1) / nsplit);
  a.rows_per_split = (a.rows_per_split + 63) / 64 * 64;
  const size_t smem = tc_dw1_smem(t.H);
  A3G_CUDA(cudaFuncSetAttribute(k_dw1_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const dim3 grid((t.F + 127) / 128, nsplit);
  k_dw1_tc<<<grid, kTcThreads, smem, st>>>(a);
  A3G_LAUNCH_DONE("k_dw1_tc", st);
}

}  // namespace a3g
