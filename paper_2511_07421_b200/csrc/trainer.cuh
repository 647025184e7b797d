// trainer.cuh -- device state of the 2-layer mean-GCN step (trainer.hpp:24-60).
#pragma once

#include "sampler.cuh"

namespace a3g {

struct TrainerState {
  a3g_graph* g = nullptr;
  a3g_cache* c = nullptr;
  // Sampler arenas of the stream pipeline: with n sampling streams, step i
  // samples into arena i % (n + 1) on stream i % n -- n batches are sampled
  // concurrently (the sampler's many small latency-bound kernels interleave)
  // while compute consumes in order; an arena is reused only after its step's
  // compute. Arenas beyond the first are allocated on first use.
  // default depth by batch size: small batches (<= 2048 seeds) are sampled by
  // short, latency-bound kernel chains and fill the GPU better with 12 in
  // flight (C2 step -5% against 8 with 32 hardware queues); large batches keep
  // 8 (C3 neutral, C5 +4% at 12)
  static constexpr int kSampStreams = 12;
  static constexpr int kArenas = kSampStreams + 1;
  static constexpr int kDefaultStreams = 8;
  static constexpr int kDefaultStreamsSmall = 12;
  static constexpr uint32_t kSmallBatch = 2048;
  a3g_sampler* smp[kArenas] = {};
  uint32_t F = 0, H = 0, C = 0, pitch = 0, L = 0, max_seeds = 0;
  double lr = 0.2;
  uint64_t cap_inner = 0;
  float* d_w1 = nullptr;   // F x H
  float* d_w2 = nullptr;   // H x C
  float* d_gw = nullptr;   // [F*H | H*C | n_k | loss*n_k]  (packed for the allreduce)
  float* d_agg_inner = nullptr;  // cap_inner x pitch
  float* d_h1 = nullptr;         // cap_inner x H (post-ReLU)
  float* d_dh1 = nullptr;        // cap_inner x H
  float* d_agg_outer = nullptr;  // max_seeds x H
  float* d_logits = nullptr;     // max_seeds x C
  float* d_dlogits = nullptr;    // max_seeds x C
  float* d_loss_s = nullptr;     // max_seeds
  float* d_dagg = nullptr;       // max_seeds x H: per-edge dh1 contribution of each seed
  unsigned long long* d_dh1_fx = nullptr;  // cap_inner x H fixed-point dh1 accumulator (kept zero between steps)
  uint32_t* d_amax = nullptr;    // max |dagg| bits of the step
  float* d_part = nullptr;       // nparts x F x H
  uint32_t nparts = 0;
  double* d_losses = nullptr;    // per-step losses of train_steps
  unsigned long long* d_stats = nullptr;  // per-step A3G_STEP_STATS rows of train_steps
  uint64_t stats_cap = 0, last_steps = 0;
  uint64_t losses_cap = 0;
  unsigned long long* d_agg_bytes = nullptr;  // algorithmic bytes moved by k_agg1 (accumulated)
  uint32_t* d_seed_buf = nullptr;  // device copy of all batches' seeds (train_steps)
  uint64_t seed_buf_cap = 0;
  uint32_t* h_seed_stage = nullptr;  // pinned staging
  uint64_t h_seed_cap = 0;
  double* h_losses = nullptr;        // pinned
  cudaStream_t s_comp = nullptr, s_samp = nullptr;  // s_samp: sampling stream 0
  cudaStream_t s_sx[kSampStreams] = {};              // sampling streams (s_sx[0] == s_samp)
  int pipe_streams = kDefaultStreams;  // a3g_trainer_set_pipeline: 0 = sequential (one stream), 1..kSampStreams
  std::vector<uint32_t> fanouts;       // for the lazily allocated arenas
  bool tc_gemms = false;               // A3G_TC_GEMMS=1: h1 and dW1 on tcgen05 (default: h1 fused
                                       // into k_agg1, dW1 on the CUDA cores, both HBM-bound)
  uint32_t dw1_splits = 1;             // row splits of k_dw1_fma (kDw1Rows rows each)
  bool h1_fused = false;               // last step used the fused epilogue
  cudaEvent_t ev_sampled[kArenas] = {}, ev_consumed[kArenas] = {};
  cudaEvent_t ev_seeds = nullptr;                     // host seeds copied (sampling streams wait on it)
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
  std::vector<cudaEvent_t> ev_agg;  // pairs around k_agg1 launches (timing; events from ev_pool)
  std::vector<cudaEvent_t> ev_pool;  // timing events, created once and reused across calls
  size_t ev_used = 0;
  std::vector<cudaEvent_t> ev_h1, ev_dw1;  // pairs around the tcgen05 h1 / dW1 GEMMs (timing)
  double last_h1_ms = 0, last_dw1_ms = 0;
  uint64_t last_gemm_launches = 0;
  bool last_seeds_on_device = false;  // the last train_steps call range-checked device seeds
  bool timing = true;
  double last_total_ms = 0, last_agg_ms = 0, last_agg_bytes = 0;
  uint64_t last_agg_launches = 0;
  a3g_comm* comm = nullptr;
  int sm_count = 148;
  uint32_t tc_splits = 1;   // row splits of the dW1 tcgen05 GEMM (partials in d_part)
  float* d_hpart = nullptr; // split-K partials of the h1 GEMM [h1_split_cap][cap_inner][H]
  uint32_t h1_split_cap = 1;
  bool h1_split_used = false;  // the last step's h1 GEMM ran split-K (+ k_h1_reduce)
  float* d_gather = nullptr;   // a3g_trainer_profile_step: the unique rows of a retrieve_features stage
  bool tier_acct = false;                    // a3g_trainer_set_tier_accounting
  uint32_t* d_tier_seen = nullptr;           // n-bit "row already counted" map (cleared per step)
  unsigned long long* d_tier_rows = nullptr; // [kMaxTiers] distinct rows gathered per tier
  uint64_t gather_cap = 0;
};

// A timing event from the trainer's pool (reset by a3g_train_steps_v).
inline cudaEvent_t pool_event(TrainerState& t) {
  if (t.ev_used == t.ev_pool.size()) {
    cudaEvent_t e = nullptr;
    A3G_CUDA(cudaEventCreate(&e));
    t.ev_pool.push_back(e);
  }
  return t.ev_pool[t.ev_used++];
}

// Compute part of one step on s_comp for the batch in arena `smp`
// (gather+aggregate -> forward -> backward -> [allreduce] -> sgd).
// d_stats: this step's A3G_STEP_STATS row (zeroed by the caller) or null.
void launch_step_stats(TrainerState& t, a3g_sampler* smp, unsigned long long* d_stats, cudaStream_t st);
void launch_train_compute(TrainerState& t, a3g_sampler* smp, double lr, double* d_loss_slot,
                          unsigned long long* d_stats, cudaStream_t st, bool record_timing);
// tcgen05 dense update (gemm_tc.cu)
size_t tc_h1_smem(uint32_t F, uint32_t H);
size_t tc_dw1_smem(uint32_t H);
void launch_h1_tc(TrainerState& t, const float* agg, const uint32_t* n_inner, float* h1, cudaStream_t st);
void launch_dw1_tc(const TrainerState& t, const float* agg, const uint32_t* n_inner, const float* h1,
                   const float* dh1, float* part, uint32_t nsplit, cudaStream_t st);
// evaluate_full_graph (trainer.cpp:241-303) with the current device weights.
double evaluate_full_graph(TrainerState& t, const uint8_t* test_mask);

}  // namespace a3g

struct a3g_trainer {
  a3g::TrainerState st;
};
