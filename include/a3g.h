/*
 * a3g.h -- C-ABI of the B200-native A3GNN data-parallel mini-batch hot path.
 *
 * Plain pointers and sizes only; every call returns an a3g_status and, on
 * failure, a thread-local message via a3g_last_error(). The status codes map
 * 1:1 onto the reference's exception types (proj/include/a3gnn/common.hpp:14-40)
 * so the C++ drop-in (include/a3gnn_b200.hpp) can rethrow the same exception.
 *
 * The reference is a C++ library with no FFI of its own; each entry point below
 * cites the reference declaration it replaces (proj/include/a3gnn/...). The
 * reference-side binding a maintainer would add is in INTEGRATION.md.
 *
 * Threading: handles are owned by the creating thread; calls on distinct
 * samplers/trainers (distinct arenas and streams) may run concurrently, which
 * mirrors the reference's concurrent producers (pipeline_exec.cpp:235-256).
 * Streams are passed explicitly as `void*` (a cudaStream_t; NULL = the
 * handle's own stream).
 */
#ifndef A3G_H_
#define A3G_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum a3g_status {
  A3G_OK = 0,
  A3G_ERR_PARAMETER = 1, /* a3gnn::ParameterError (common.hpp:14) */
  A3G_ERR_LOOKUP = 2,    /* a3gnn::LookupError    (common.hpp:20) */
  A3G_ERR_CONFIG = 3,    /* a3gnn::ConfigError    (common.hpp:26) */
  A3G_ERR_IO = 4,        /* a3gnn::IoError        (common.hpp:37) */
  A3G_ERR_CUDA = 5,
  A3G_ERR_NCCL = 6,
  A3G_ERR_OOM = 7
} a3g_status;

enum { A3G_SAMPLER_WEIGHTED = 0, A3G_SAMPLER_UNIFORM = 1 }; /* sampler.hpp:18-21 */
enum { A3G_FEAT_F32 = 0, A3G_FEAT_BF16 = 1 };
/* Feature placement of the reference's static cache (cache.cpp:12-46). */
enum { A3G_STORE_HBM = 0, A3G_STORE_CACHE = 1, A3G_STORE_SHARDED = 2 };
/* Per-step statistics rows of a3g_trainer_step_stats. */
enum {
  A3G_STAT_UNIQUE = 0, /* |unique_nodes| */
  A3G_STAT_EDGES = 1,  /* total sampled edges */
  A3G_STAT_INNER = 2,  /* inner rows (seeds + layer-0 sources, trainer.cpp:76-89) */
  A3G_STAT_SEEDS = 3,  /* unique seeds */
  A3G_STAT_HITS = 4,   /* cache hits over unique_nodes (cache.cpp:48-68) */
  A3G_STAT_MISSES = 5,
  A3G_STAT_BAD_SEEDS = 6, /* device-resident seeds >= num_nodes (the call raised ParameterError) */
  A3G_STAT_POSITIONS = 7, /* neighbour positions drawn: sum of frontier degrees (the sampler work) */
  A3G_STEP_STATS = 8
};

typedef struct a3g_host_graph {
  /* graph.hpp:14-36 layout, host memory owned by the library */
  uint64_t num_nodes;
  uint64_t num_edges;
  uint32_t feat_dim;
  uint64_t* row_offsets; /* n+1 */
  uint32_t* col_indices; /* m, ascending per row (graph.cpp:66) */
  float* features;       /* n x feat_dim, row-major */
  uint32_t* labels;      /* n */
  uint8_t* train_mask;   /* n */
  uint8_t* test_mask;    /* n */
} a3g_host_graph;

typedef struct a3g_graph a3g_graph;     /* device-resident CSR + feature store */
typedef struct a3g_cache a3g_cache;     /* static hotness cache state */
typedef struct a3g_sampler a3g_sampler; /* k-hop sampler arena (one batch in flight) */
typedef struct a3g_trainer a3g_trainer; /* model, grads, streams, pipeline */
typedef struct a3g_comm a3g_comm;       /* NCCL communicator (data-parallel sync) */
typedef struct a3g_store a3g_store;     /* tiered feature store (HBM / NVLink peers / pinned host) */

const char* a3g_last_error(void);
const char* a3g_version(void);

/* ---------------------------------------------------------------- host --- */
/* generators.cpp:79-149 generate_power_law, bit-identical, multithreaded. */
a3g_status a3g_host_graph_power_law(uint64_t num_nodes, uint32_t min_degree, double exponent,
                                    uint32_t feat_dim, uint64_t seed, int threads,
                                    a3g_host_graph** out);
/* graph_io.cpp:40-87 A3G1 load/save (graph_io.hpp:3-7 format). */
a3g_status a3g_host_graph_load(const char* path, a3g_host_graph** out);
a3g_status a3g_host_graph_save(const a3g_host_graph* g, const char* path);
/* graph.cpp:59-84 from_edges (sorts (src,dst)); features zero. */
a3g_status a3g_host_graph_from_edges(uint64_t num_nodes, const uint32_t* src, const uint32_t* dst,
                                     uint64_t num_edges, uint32_t feat_dim, a3g_host_graph** out);
void a3g_host_graph_free(a3g_host_graph* g);

/* trainer.cpp:345-348 */
uint64_t a3g_sampling_seed(uint64_t base, uint32_t epoch, uint32_t step, uint32_t worker);
/* trainer.cpp:330-343: shuffled order of train_nodes; batch i = order[i*B, (i+1)*B). */
void a3g_plan_epoch_order(const uint32_t* train_nodes, uint64_t n, uint32_t epoch, uint64_t seed,
                          uint32_t* order_out);

/* --------------------------------------------------------------- graph --- */
/* Uploads CSR (+ optional features/labels) to `device`. features may be NULL
 * (topology-only sampling). feat_dtype A3G_FEAT_BF16 rounds the f32 input to
 * bf16 rows in HBM. Rows are pitched to 32 bytes. Replaces the shared,
 * immutable graph::Graph (graph.hpp:3-4). */
a3g_status a3g_graph_create(int device, uint64_t num_nodes, uint64_t num_edges, uint32_t feat_dim,
                            const uint64_t* row_offsets, const uint32_t* col_indices,
                            const float* features, int feat_dtype, const uint32_t* labels,
                            a3g_graph** out);
void a3g_graph_destroy(a3g_graph* g);
/* Papers-scale inputs (BASELINE config 5): fill the device feature table of a
 * graph created without features, with the power-law generator's features
 * (generators.cpp:12-24: Gaussian noise of substream 0xfea7 + one-hot label)
 * synthesized on the device at feat_dim, stored as feat_dtype. The topology,
 * labels and masks come from a3g_host_graph_power_law at feat_dim 1. */
a3g_status a3g_graph_synthesize_features(a3g_graph* g, uint32_t feat_dim, int feat_dtype, uint64_t seed);
/* Elements of the last synthesis that sat within 2^-44 relative of a float
 * rounding boundary and were recomputed with the host's glibc (synth.cu). */
uint64_t a3g_graph_synth_patched(const a3g_graph* g);

/* --------------------------------------------------------------- store --- */
/* Places the feature rows of `g` by `policy` (A3G_STORE_*) from host f32
 * features (n x feat_dim, encoded to the graph's feat_dtype) -- or, with
 * features == NULL, from the graph's own device table (the synthesized
 * papers-scale table, which has no host copy) -- and attaches the store to
 * the graph: every gather of the path then reads through it.
 * device_map: the cache placement (i32[n], -1 = miss, cache.hpp:31); ignored
 * for A3G_STORE_HBM. rank/nranks: this GPU's shard for A3G_STORE_SHARDED. */
a3g_status a3g_store_create(a3g_graph* g, const float* features, const int32_t* device_map, int policy,
                            int rank, int nranks, a3g_store** out);
a3g_status a3g_store_info(const a3g_store* s, uint64_t* local_rows, uint64_t* host_rows,
                          uint64_t* remote_rows);
/* Peer shards: same-process device pointers (a3g_store_local_ptr of the peer's
 * store; peer access is enabled), or cudaIpc handles across processes. */
a3g_status a3g_store_local_ptr(a3g_store* s, void** dev_ptr);
a3g_status a3g_store_set_peer(a3g_store* s, int rank, void* dev_ptr);
a3g_status a3g_store_ipc_handle(a3g_store* s, uint8_t handle[64]);
a3g_status a3g_store_open_peer(a3g_store* s, int rank, const uint8_t handle[64]);
void a3g_store_destroy(a3g_store* s); /* detaches; the graph keeps its own rows (if any) */

/* --------------------------------------------------------------- cache --- */
/* cache.cpp:12-46 build_static_cache: (out-degree desc, id asc), round-robin
 * over num_devices, floor(volume_bytes / (F*4)) nodes per device.
 * device_map_out (i32[n], -1 = miss) may be NULL. */
a3g_status a3g_cache_build(a3g_graph* g, uint64_t volume_bytes, uint32_t num_devices,
                           int32_t* device_map_out, a3g_cache** out);
/* A CacheState given explicitly (test fixtures: test_sampler.cpp:15-25). */
a3g_status a3g_cache_from_map(a3g_graph* g, const int32_t* device_map, uint32_t num_devices,
                              a3g_cache** out);
uint64_t a3g_cache_total_cached(const a3g_cache* c);
/* The cached nodes in placement order (cache.cpp:24-44: out-degree desc, id
 * asc; node i went to device i % num_devices): u32[total_cached]. Only for
 * caches made by a3g_cache_build. Feeds CacheState::cached_per_device. */
a3g_status a3g_cache_hot_order(const a3g_cache* c, uint32_t* out);
/* cache.cpp:48-68 lookup on the device: the device of every id (device_out,
 * i32[n], -1 = miss; NULL skips) and the accounting counts (hits, misses,
 * per_device_hits u64[num_devices]; any may be NULL). Any-device presence is
 * a hit. ParameterError on ids >= num_nodes. */
a3g_status a3g_cache_lookup(a3g_cache* c, const uint32_t* ids, uint64_t n, int32_t* device_out, uint64_t* hits,
                            uint64_t* misses, uint64_t* per_device_hits);
void a3g_cache_destroy(a3g_cache* c);

/* ------------------------------------------------------------- sampler --- */
/* Arena for batches of <= max_seeds seeds with the given fanouts (outermost
 * first, sampler.hpp:24). */
a3g_status a3g_sampler_create(a3g_graph* g, a3g_cache* c, uint32_t max_seeds,
                              const uint32_t* fanouts, uint32_t num_layers, a3g_sampler** out);
void a3g_sampler_destroy(a3g_sampler* s);

/* sampler.hpp:62-63 sample_khop, device-resident result. seeds are host
 * memory (copied inside) unless seeds_on_device. kind: A3G_SAMPLER_*.
 * Validation order/semantics as sampler.cpp:91-94,110 and assign_weights :62. */
a3g_status a3g_sample_khop(a3g_sampler* s, const uint32_t* seeds, uint32_t n_seeds,
                           int seeds_on_device, double bias_rate, int kind, uint64_t rng_seed,
                           void* stream);

/* Sizes of the last batch (synchronises the sampler stream).
 * layer_edges: u64[num_layers]. */
a3g_status a3g_batch_sizes(a3g_sampler* s, uint64_t* num_unique, uint64_t* num_seed_unique,
                           uint64_t* num_duplicates_removed, uint64_t* layer_edges);
/* Copies the last batch into host buffers sized by a3g_batch_sizes:
 * SampleBatch (sampler.hpp:30-46) as unique_nodes and per-layer
 * (dst_idx, src_idx) pairs in the reference's edge order. NULL skips. */
a3g_status a3g_batch_copy(a3g_sampler* s, uint32_t* unique_nodes, uint32_t* const* layer_dst,
                          uint32_t* const* layer_src);

/* cache.hpp:78-80 retrieve_features for the last batch: gathers the
 * unique_nodes' f32 rows into `out` (host, or device if out_on_device),
 * counts cache hits/misses (cache.cpp:48-68) and returns B (cache.cpp:84). */
a3g_status a3g_retrieve_features(a3g_sampler* s, float* out, int out_on_device, uint64_t* hits,
                                 uint64_t* misses, uint64_t* batch_bytes, void* stream);

/* cache.cpp:48-68 lookup + kernels_scalar.cpp:95-101 gather_rows for an
 * explicit id list (host ids, host f32 out n x F; hits/misses counted). */
a3g_status a3g_gather_rows(a3g_graph* g, a3g_cache* c, const uint32_t* ids, uint64_t n, float* out,
                           uint64_t* hits, uint64_t* misses);

/* sampler.cpp:9-42 / 44-58 on one explicit neighbour list, on the device
 * (test hook; weights arbitrary > 0). Draws start at counter ctr0+1 of
 * stream key `key` (rng.hpp:43-46). Returns the reservoir in slot order. */
a3g_status a3g_weighted_reservoir(const uint32_t* nbrs, const double* weights, uint64_t n,
                                  uint32_t m, uint64_t key, uint64_t ctr0, uint32_t* out,
                                  uint64_t* count);
a3g_status a3g_uniform_reservoir(const uint32_t* nbrs, uint64_t n, uint32_t m, uint64_t key,
                                 uint64_t ctr0, uint32_t* out, uint64_t* count);

/* ------------------------------------------------------------- trainer --- */
/* trainer.cpp:12-28 init_model (Glorot-uniform from RngStream(seed, 0x6a10)). */
a3g_status a3g_init_model(uint32_t feat_dim, uint32_t hidden_dim, uint32_t num_classes, uint64_t seed,
                          double* w1, double* w2);

/* 2-layer mean-GCN (trainer.hpp:24-60) in fp32 on the device. Weights are
 * initialised as init_model (trainer.cpp:12-28) from model_seed. */
a3g_status a3g_trainer_create(a3g_graph* g, a3g_cache* c, uint32_t max_seeds,
                              const uint32_t* fanouts, uint32_t num_layers, uint32_t hidden_dim,
                              uint32_t num_classes, double learning_rate, uint64_t model_seed,
                              a3g_trainer** out);
void a3g_trainer_destroy(a3g_trainer* t);
/* Set/get weights (row-major W1 FxH, W2 HxC) as f64 host arrays. */
a3g_status a3g_trainer_set_weights(a3g_trainer* t, const double* w1, const double* w2);
a3g_status a3g_trainer_get_weights(a3g_trainer* t, double* w1, double* w2);
/* Pipeline shape of a3g_train_steps[_v] (pipeline_exec.cpp:219-276 modes):
 * 0 = sequential (sampling and compute on one stream, Mode::sequential);
 * n = 1..12 sampling streams running n batches' samplers concurrently ahead of
 * the compute stream (n + 1 arenas, allocated on first use). Default 12 for
 * trainers of <= 2048 seeds per batch, else 8.
 * Results are identical for every shape (schedule only, pipeline.hpp:107-109). */
a3g_status a3g_trainer_set_pipeline(a3g_trainer* t, int sampling_streams);
/* Attach a communicator for the data-parallel gradient sum (NULL detaches). */
a3g_status a3g_trainer_set_comm(a3g_trainer* t, a3g_comm* comm);

/* One step on one batch: sample_khop -> gather+aggregate -> forward ->
 * backward -> [allreduce] -> sgd (trainer.cpp:385-406). lr < 0 uses the
 * trainer's learning rate; lr = 0 computes gradients only. loss_out (host)
 * may be NULL (no sync). */
a3g_status a3g_train_step(a3g_trainer* t, const uint32_t* seeds, uint32_t n_seeds,
                          int seeds_on_device, double bias_rate, int kind, uint64_t rng_seed,
                          double lr, double* loss_out);

/* K pipelined steps: batch i = seeds[i*B .. (i+1)*B) (host), step seed
 * rng_seeds[i]; sampling of batch i+1 overlaps compute of batch i on a second
 * stream (the CUDA-stream replacement of pipeline_exec.cpp:229-276).
 * losses_out: host f64[K] (read back once at the end). */
a3g_status a3g_train_steps(a3g_trainer* t, const uint32_t* seeds, uint32_t batch_size,
                           uint32_t num_steps, const uint64_t* rng_seeds, double bias_rate,
                           int kind, int seeds_on_device, double* losses_out);

/* As a3g_train_steps with per-step batch sizes (the last batch of an epoch is
 * short, trainer.cpp:338-341): batch i = seeds[offsets[i] .. offsets[i+1]). */
a3g_status a3g_train_steps_v(a3g_trainer* t, const uint32_t* seeds, const uint64_t* offsets,
                             uint32_t num_steps, const uint64_t* rng_seeds, double bias_rate, int kind,
                             int seeds_on_device, double* losses_out);
/* Statistics of the steps of the last a3g_train_steps[_v] call:
 * out[i * A3G_STEP_STATS + A3G_STAT_*] for i < num_steps. */
a3g_status a3g_trainer_step_stats(a3g_trainer* t, uint64_t* out, uint32_t num_steps);

/* evaluate_full_graph (trainer.cpp:241-303) on the device with the trainer's
 * current weights: full-neighbourhood 2-layer mean-GCN over all nodes, argmax
 * accuracy over test_mask (host u8[n]). ConfigError when no test nodes. */
a3g_status a3g_evaluate_full_graph(a3g_trainer* t, const uint8_t* test_mask, double* accuracy);

/* pipeline.hpp:57-60 profile_stage_costs on the device: one probe of
 * sample_khop (host seeds), retrieve_features (the unique rows gathered into
 * HBM) and grad_on_batch (forward + backward, weights unchanged), timed with
 * CUDA events on the compute stream: stage_ms[3] = {t_sample, t_batch,
 * t_train} in ms. */
a3g_status a3g_trainer_profile_step(a3g_trainer* t, const uint32_t* seeds, uint32_t n_seeds, double bias_rate,
                                    int kind, uint64_t rng_seed, double* stage_ms);

/* Per-resource accounting of the gather (bench roofline leg): when on, each
 * step counts the distinct feature rows the fused gather reads by the tier
 * they live in (store placement: HBM shard of rank r < 15, NVLink peer,
 * pinned host = 15; no store: tier 0), after the gather's timing events.
 * a3g_trainer_tier_rows: u64[16] summed over the last a3g_train_steps call. */
a3g_status a3g_trainer_set_tier_accounting(a3g_trainer* t, int on);
a3g_status a3g_trainer_tier_rows(a3g_trainer* t, uint64_t* rows);

/* Debug/parity copy-out of the last step (host f64 buffers; NULL skips):
 * gradients (F*H, H*C), and ForwardResult arrays (trainer.hpp:49-60). */
a3g_status a3g_trainer_last_grads(a3g_trainer* t, double* gw1, double* gw2);
a3g_status a3g_trainer_last_forward(a3g_trainer* t, uint64_t* n_inner, double* logits,
                                    double* agg_inner, double* h1, double* agg_outer);
a3g_sampler* a3g_trainer_sampler(a3g_trainer* t, int slot);

/* Device-time breakdown of the last a3g_train_steps call (CUDA events on the
 * launching streams): total ms, and the average per-launch ms of the
 * gather+aggregation kernel (the roofline kernel) with its algorithmic bytes. */
a3g_status a3g_trainer_timing(a3g_trainer* t, double* total_ms, double* agg_kernel_ms,
                              double* agg_bytes_per_launch, uint64_t* launches_per_step);

/* ------------------------------------------------------- explicit batch --- */
/* The reference's per-batch model calls on an EXPLICIT host batch -- the
 * SampleBatch (sampler.hpp:30-46) and the feats array the caller passes --
 * run through the same device kernels as the pipeline (explicit.cu). Backs
 * the drop-in's train::forward / backward / grad_on_batch
 * (trainer.hpp:63-79, trainer.cpp:59-239). One model per host thread. */
typedef struct a3g_batch_model a3g_batch_model;
a3g_status a3g_batch_model_create(int device, uint32_t feat_dim, uint32_t hidden_dim, uint32_t num_classes,
                                  a3g_batch_model** out);
void a3g_batch_model_destroy(a3g_batch_model* m);
/* Loads unique count, unique-seed count, num_layers layers of (dst_idx,
 * src_idx) pairs (layers >= 2 are ignored, as trainer.cpp does), feats
 * (host f32[n_unique * feat_dim], unique-node order) and the seed labels
 * (host u32[n_seed_unique], NULL = zeros: forward only). n_inner_out = the
 * ForwardResult's |inner_nodes|. */
a3g_status a3g_batch_model_load(a3g_batch_model* m, uint64_t n_unique, uint64_t n_seed_unique,
                                uint32_t num_layers, const uint64_t* layer_ne, const uint32_t* const* layer_dst,
                                const uint32_t* const* layer_src, const float* feats, const uint32_t* seed_labels,
                                uint64_t* n_inner_out);
/* forward + softmax-CE backward with W1 (F x H), W2 (H x C) f64 host: mean
 * loss and gradients (f64 host, NULL skips). Weights are not changed. */
a3g_status a3g_batch_model_run(a3g_batch_model* m, const double* w1, const double* w2, double* loss,
                               double* gw1, double* gw2);
/* ForwardResult (trainer.hpp:49-60) of the last run, host buffers, NULL
 * skips: inner_nodes u32[n_inner], inner_pos i32[n_unique], inner_deg
 * u32[n_inner], outer_deg u32[n_seed_unique], agg_inner f64[n_inner*F],
 * h1 f64[n_inner*H] (post-ReLU), agg_outer f64[n_seed_unique*H], logits
 * f64[n_seed_unique*C]. */
a3g_status a3g_batch_model_forward(a3g_batch_model* m, uint32_t* inner_nodes, int32_t* inner_pos,
                                   uint32_t* inner_deg, uint32_t* outer_deg, double* agg_inner, double* h1,
                                   double* agg_outer, double* logits);
/* trainer.cpp:208-211 sgd_step on the device: w[i] += (-lr) * g[i] in f64,
 * bit-identical to the reference's active kernel table: the first n_fused
 * elements as one fused multiply-add (AVX2 table: n - n % 4), the rest with
 * product and sum rounded separately (scalar table: n_fused = 0). */
a3g_status a3g_sgd_step(int device, double* w, const double* g, uint64_t n, uint64_t n_fused, double lr);
/* trainer.cpp:213-229 sync_gradients on the device: out = (g_0 + ... +
 * g_{k-1}) * (1/k), summed in list order. ParameterError when k == 0. */
a3g_status a3g_mean_gradients(int device, const double* const* grads, uint32_t k, uint64_t n, double* out);

/* Average per-launch ms of the tcgen05 dense update in the last a3g_train_steps
 * call (CUDA events on the compute stream): h1 = ReLU(agg . W1) and dW1 =
 * agg^T . G, when they ran on the tensor cores (H > 16, or A3G_TC_GEMMS=1);
 * launches = number of timed h1 GEMMs (0: the fused / CUDA-core path ran). */
a3g_status a3g_trainer_gemm_timing(a3g_trainer* t, double* h1_ms, double* dw1_ms, uint64_t* launches);

/* ---------------------------------------------------------------- comm --- */
/* NCCL communicator for data-parallel gradient sync (trainer.cpp:213-229 ->
 * allreduce(sum) of n_k-weighted gradients). unique_id is 128 opaque bytes. */
a3g_status a3g_comm_unique_id(uint8_t unique_id[128]);
a3g_status a3g_comm_create(const uint8_t unique_id[128], int nranks, int rank, int device,
                           a3g_comm** out);
/* Host-transport communicator: each step the library hands the packed
 * gradient buffer [n_k dW1 | n_k dW2 | n_k | n_k loss] (f32, `count` values,
 * pinned host memory) to `fn`, which must replace it in place with the
 * element-wise sum over all ranks (a gloo / MPI / shared-memory allreduce) and
 * return 0. The arithmetic around it is the NCCL path's (k_scale_for_sync,
 * k_sgd); for ranks that cannot share an NCCL communicator (several ranks on
 * one GPU) and for CPU-side collectives. */
typedef int (*a3g_allreduce_fn)(float* buf, size_t count, void* user);
a3g_status a3g_comm_create_host(int nranks, int rank, a3g_allreduce_fn fn, void* user, a3g_comm** out);
void a3g_comm_destroy(a3g_comm* c);

#ifdef __cplusplus
}
#endif
#endif /* A3G_H_ */
