/*
 * a3g_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C, single-threaded CPU restatement of the A3GNN reference hot path:
 * counter RNG, locality-aware k-hop sampler, static hotness cache, feature
 * gather, and the fp64 2-layer mean-GCN forward/backward/SGD step loop.
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/...). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load the library built from this file.
 *
 * Parity of this restatement is PINNED against golden vectors produced by the
 * compiled reference itself (oracle/ref_shim.cpp -> oracle/_ref, fixtures in
 * tests/golden/, generator tests/golden/make_golden.py).
 *
 * Build: see oracle/Makefile (gcc -O2, no -ffast-math, no FMA contraction so
 * the fp64 arithmetic order matches the reference's scalar kernel table).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PHI 0x9e3779b97f4a7c15ull
#define INV32 0xffffffffu

/* ---------------------------------------------------------------- RNG ---- */
/* include/a3gnn/rng.hpp:15-22 */
static inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}
/* rng.hpp:24-30 */
static inline uint64_t hash2(uint64_t a, uint64_t b) { return mix64(a ^ mix64(b + PHI)); }
static inline uint64_t hash3(uint64_t a, uint64_t b, uint64_t c) { return hash2(hash2(a, b), c); }

uint64_t orc_mix64(uint64_t z) { return mix64(z); }
uint64_t orc_hash2(uint64_t a, uint64_t b) { return hash2(a, b); }
uint64_t orc_hash3(uint64_t a, uint64_t b, uint64_t c) { return hash3(a, b, c); }

/* rng.hpp:32-83: RngStream{key, counter}; i-th draw = mix64(key + i*phi) */
typedef struct {
  uint64_t key, ctr, draws;
} rng_t;

static rng_t rng_make(uint64_t seed, uint64_t stream) {
  rng_t r = {hash2(seed, stream), 0, 0};
  return r;
}
static inline uint64_t next_u64(rng_t* r) {
  ++r->draws;
  ++r->ctr;
  return mix64(r->key + r->ctr * PHI);
}
/* rng.hpp:49 */
static inline double next_unit(rng_t* r) { return (double)(next_u64(r) >> 11) * 0x1.0p-53; }
/* rng.hpp:52-55 */
static inline uint32_t next_below(rng_t* r, uint32_t bound) {
  return (uint32_t)(((unsigned __int128)next_u64(r) * bound) >> 64);
}

uint64_t orc_stream_key(uint64_t seed, uint64_t stream) { return hash2(seed, stream); }
double orc_next_unit_at(uint64_t key, uint64_t i) {
  return (double)(mix64(key + i * PHI) >> 11) * 0x1.0p-53;
}

/* generators.cpp:12-24 + rng.hpp:60-65: the power-law generator's feature
 * rows for an explicit node list (papers-scale parity of the gathered rows
 * without the 56 GB f32 table). The generator's rng is RngStream(seed,
 * 0x97a3) (generators.cpp:87) and the noise its substream 0xfea7 (rng.hpp:38-
 * 41: key hash2(key, id ^ 0xd6e8feb86659fd93)); element (v, d) is the
 * Box-Muller Gaussian of draws 2(v F + d) + 1, + 2 (two draws per sample, no
 * caching), cast to float, + 1.0f at d == label % F. */
void orc_feature_rows(uint64_t seed, uint32_t F, const uint32_t* ids, uint64_t n, const uint32_t* labels,
                      float* out) {
  const uint64_t noise_key = hash2(hash2(seed, 0x97a3), 0xfea7ull ^ 0xd6e8feb86659fd93ull);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t v = ids[i];
    float* row = out + i * F;
    for (uint32_t d = 0; d < F; ++d) {
      const uint64_t c = 2 * (v * F + d);
      double u1 = (double)(mix64(noise_key + (c + 1) * PHI) >> 11) * 0x1.0p-53;
      const double u2 = (double)(mix64(noise_key + (c + 2) * PHI) >> 11) * 0x1.0p-53;
      if (u1 <= 0.0) u1 = 0x1.0p-53;
      row[d] = (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925 * u2));
    }
    row[labels[v] % F] += 1.0f;
  }
}

/* trainer.cpp:345-348 */
uint64_t orc_sampling_seed(uint64_t base, uint32_t epoch, uint32_t step, uint32_t worker) {
  return hash3(base, hash2(epoch, step), worker);
}

/* trainer.cpp:330-343 (shuffle: rng.hpp:69-74). Writes the shuffled order;
 * batches are consecutive chunks of batch_size. */
void orc_plan_epoch_order(const uint32_t* train_nodes, uint64_t n, uint32_t epoch, uint64_t seed,
                          uint32_t* order) {
  memcpy(order, train_nodes, n * sizeof(uint32_t));
  rng_t rng = rng_make(seed, hash2(0x5f1e, epoch));
  for (uint64_t i = n; i > 1; --i) {
    uint64_t j = next_below(&rng, (uint32_t)i);
    uint32_t t = order[i - 1];
    order[i - 1] = order[j];
    order[j] = t;
  }
}

/* ------------------------------------------------------------ sampler ---- */
/* sampler.cpp:9-42. Returns #sampled, -1 on |w| mismatch (n/a here), -2 m<1,
 * -3 non-positive weight. *ctr is the stream counter (in/out). */
int64_t orc_weighted_reservoir(const uint32_t* nbrs, const double* w, uint64_t n, uint32_t m,
                               uint64_t key, uint64_t* ctr, uint32_t* out) {
  if (m < 1) return -2;
  if (n == 0) return 0;
  rng_t rng = {key, *ctr, 0};
  uint64_t cap = n < m ? n : m;
  double* keys = (double*)malloc(cap * sizeof(double));
  uint64_t cnt = 0, min_pos = 0;
  for (uint64_t j = 0; j < n; ++j) {
    const double wj = w[j];
    if (!(wj > 0.0)) {
      free(keys);
      *ctr = rng.ctr;
      return -3;
    }
    const double k = pow(next_unit(&rng), 1.0 / wj);
    if (cnt < m) {
      out[cnt] = nbrs[j];
      keys[cnt] = k;
      ++cnt;
      if (k < keys[min_pos]) min_pos = cnt - 1;
    } else if (k > keys[min_pos]) { /* strict: ties keep the incumbent */
      out[min_pos] = nbrs[j];
      keys[min_pos] = k;
      uint64_t mp = 0; /* std::min_element: first minimum */
      for (uint64_t t = 1; t < cnt; ++t)
        if (keys[t] < keys[mp]) mp = t;
      min_pos = mp;
    }
  }
  free(keys);
  *ctr = rng.ctr;
  return (int64_t)cnt;
}

/* sampler.cpp:44-58 (Algorithm R) */
int64_t orc_uniform_reservoir(const uint32_t* nbrs, uint64_t n, uint32_t m, uint64_t key,
                              uint64_t* ctr, uint32_t* out) {
  if (m < 1) return -2;
  rng_t rng = {key, *ctr, 0};
  uint64_t cnt = 0;
  for (uint64_t j = 0; j < n; ++j) {
    if (cnt < m) {
      out[cnt++] = nbrs[j];
    } else {
      const uint64_t r = next_below(&rng, (uint32_t)(j + 1));
      if (r < m) out[r] = nbrs[j];
    }
  }
  *ctr = rng.ctr;
  return (int64_t)cnt;
}

/* Batch record, sampler.hpp:30-46 */
typedef struct {
  uint64_t n_seeds;
  uint32_t* seeds;
  uint64_t n_unique, cap_unique, num_seed_unique, dups;
  uint32_t* unique;
  uint32_t num_layers;
  uint64_t* layer_ne;
  uint64_t* layer_cap;
  uint32_t** layer_dst;
  uint32_t** layer_src;
  uint64_t keys_scanned; /* instrumentation: sum of neighbour-list lengths sampled */
} orc_batch;

static void push_unique(orc_batch* b, uint32_t v) {
  if (b->n_unique == b->cap_unique) {
    b->cap_unique = b->cap_unique ? 2 * b->cap_unique : 1024;
    b->unique = (uint32_t*)realloc(b->unique, b->cap_unique * sizeof(uint32_t));
  }
  b->unique[b->n_unique++] = v;
}
static void push_edge(orc_batch* b, uint32_t l, uint32_t d, uint32_t s) {
  if (b->layer_ne[l] == b->layer_cap[l]) {
    b->layer_cap[l] = b->layer_cap[l] ? 2 * b->layer_cap[l] : 1024;
    b->layer_dst[l] = (uint32_t*)realloc(b->layer_dst[l], b->layer_cap[l] * sizeof(uint32_t));
    b->layer_src[l] = (uint32_t*)realloc(b->layer_src[l], b->layer_cap[l] * sizeof(uint32_t));
  }
  b->layer_dst[l][b->layer_ne[l]] = d;
  b->layer_src[l][b->layer_ne[l]] = s;
  ++b->layer_ne[l];
}

void orc_batch_free(orc_batch* b) {
  if (!b) return;
  free(b->seeds);
  free(b->unique);
  for (uint32_t l = 0; l < b->num_layers; ++l) {
    free(b->layer_dst[l]);
    free(b->layer_src[l]);
  }
  free(b->layer_ne);
  free(b->layer_cap);
  free(b->layer_dst);
  free(b->layer_src);
  free(b);
}

/* accessors for ctypes */
uint64_t orc_batch_num_unique(const orc_batch* b) { return b->n_unique; }
uint64_t orc_batch_num_seed_unique(const orc_batch* b) { return b->num_seed_unique; }
uint64_t orc_batch_dups(const orc_batch* b) { return b->dups; }
uint64_t orc_batch_keys_scanned(const orc_batch* b) { return b->keys_scanned; }
const uint32_t* orc_batch_unique(const orc_batch* b) { return b->unique; }
uint64_t orc_batch_layer_ne(const orc_batch* b, uint32_t l) { return b->layer_ne[l]; }
const uint32_t* orc_batch_layer_dst(const orc_batch* b, uint32_t l) { return b->layer_dst[l]; }
const uint32_t* orc_batch_layer_src(const orc_batch* b, uint32_t l) { return b->layer_src[l]; }

/* sampler.cpp:89-137 (+ assign_weights :60-68, Interner :72-85).
 * kind 0 = weighted_reservoir, 1 = uniform_baseline. device_map: i32[n] or
 * NULL (= nothing cached). On error returns NULL and *err:
 *   1 empty seeds, 2 seed out of range, 3 fanout < 1, 4 gamma < 1. */
orc_batch* orc_sample_khop(uint64_t num_nodes, const uint64_t* row_offsets, const uint32_t* col,
                           const uint32_t* seeds, uint64_t n_seeds, const uint32_t* fanouts,
                           uint32_t num_layers, double gamma, int kind, uint64_t rng_seed,
                           const int32_t* device_map, int* err) {
  *err = 0;
  if (n_seeds == 0) {
    *err = 1;
    return NULL;
  }
  for (uint64_t i = 0; i < n_seeds; ++i)
    if (seeds[i] >= num_nodes) {
      *err = 2;
      return NULL;
    }
  orc_batch* b = (orc_batch*)calloc(1, sizeof(orc_batch));
  b->n_seeds = n_seeds;
  b->seeds = (uint32_t*)malloc(n_seeds * sizeof(uint32_t));
  memcpy(b->seeds, seeds, n_seeds * sizeof(uint32_t));
  b->num_layers = num_layers;
  b->layer_ne = (uint64_t*)calloc(num_layers + 1, sizeof(uint64_t));
  b->layer_cap = (uint64_t*)calloc(num_layers + 1, sizeof(uint64_t));
  b->layer_dst = (uint32_t**)calloc(num_layers + 1, sizeof(uint32_t*));
  b->layer_src = (uint32_t**)calloc(num_layers + 1, sizeof(uint32_t*));

  uint32_t* index = (uint32_t*)malloc(num_nodes * sizeof(uint32_t)); /* Interner map */
  memset(index, 0xff, num_nodes * sizeof(uint32_t));
  uint32_t* seen_stamp = (uint32_t*)calloc(num_nodes, sizeof(uint32_t)); /* seen_next */
  uint64_t fcap = n_seeds, fn = 0, nfn = 0, nfcap = 1024;
  uint32_t* frontier = (uint32_t*)malloc(fcap * sizeof(uint32_t));
  uint32_t* next_frontier = (uint32_t*)malloc(nfcap * sizeof(uint32_t));
  uint32_t maxf = 1;
  for (uint32_t l = 0; l < num_layers; ++l)
    if (fanouts[l] > maxf) maxf = fanouts[l];
  uint32_t* sampled = (uint32_t*)malloc(maxf * sizeof(uint32_t));
  double* wbuf = NULL;
  uint64_t wcap = 0;

  for (uint64_t i = 0; i < n_seeds; ++i) { /* :100-105 */
    const uint32_t s = seeds[i];
    if (index[s] == INV32) {
      index[s] = (uint32_t)b->n_unique;
      push_unique(b, s);
      frontier[fn++] = s;
    } else {
      ++b->dups;
    }
  }
  b->num_seed_unique = b->n_unique;

  for (uint32_t layer = 0; layer < num_layers && !*err; ++layer) { /* :107-135 */
    const uint32_t fanout = fanouts[layer];
    if (fanout < 1) {
      *err = 3;
      break;
    }
    nfn = 0;
    for (uint64_t fi = 0; fi < fn; ++fi) {
      const uint32_t dst = frontier[fi];
      const uint64_t beg = row_offsets[dst], end = row_offsets[dst + 1], deg = end - beg;
      if (deg == 0) continue; /* :116 */
      const uint64_t key = hash2(rng_seed, hash2(layer, dst)); /* :117 */
      uint64_t ctr = 0;
      int64_t cnt;
      b->keys_scanned += deg;
      if (kind == 1) {
        cnt = orc_uniform_reservoir(col + beg, deg, fanout, key, &ctr, sampled);
      } else {
        if (gamma < 1.0) { /* assign_weights :62 */
          *err = 4;
          break;
        }
        if (deg > wcap) {
          wcap = deg;
          wbuf = (double*)realloc(wbuf, wcap * sizeof(double));
        }
        for (uint64_t j = 0; j < deg; ++j) {
          const uint32_t v = col[beg + j];
          wbuf[j] = (device_map && device_map[v] != -1) ? gamma : 1.0;
        }
        cnt = orc_weighted_reservoir(col + beg, wbuf, deg, fanout, key, &ctr, sampled);
      }
      const uint32_t dst_idx = index[dst]; /* :125 */
      for (int64_t t = 0; t < cnt; ++t) {
        const uint32_t src = sampled[t];
        uint32_t sidx = index[src];
        if (sidx == INV32) {
          sidx = (uint32_t)b->n_unique;
          index[src] = sidx;
          push_unique(b, src);
        } else {
          ++b->dups;
        }
        push_edge(b, layer, dst_idx, sidx);
        if (seen_stamp[src] != layer + 1) { /* :128-131 */
          seen_stamp[src] = layer + 1;
          if (nfn == nfcap) {
            nfcap *= 2;
            next_frontier = (uint32_t*)realloc(next_frontier, nfcap * sizeof(uint32_t));
          }
          next_frontier[nfn++] = src;
        }
      }
    }
    /* swap frontiers */
    uint32_t* t = frontier;
    frontier = next_frontier;
    next_frontier = t;
    uint64_t tc = fcap;
    fcap = nfcap;
    nfcap = tc;
    if (nfcap < 1024) {
      nfcap = 1024;
      next_frontier = (uint32_t*)realloc(next_frontier, nfcap * sizeof(uint32_t));
    }
    fn = nfn;
  }
  free(index);
  free(seen_stamp);
  free(frontier);
  free(next_frontier);
  free(sampled);
  free(wbuf);
  if (*err) {
    orc_batch_free(b);
    return NULL;
  }
  return b;
}

/* -------------------------------------------------------------- cache ---- */
static const uint64_t* g_sort_ro; /* qsort context (single-threaded oracle) */
static int hot_cmp(const void* pa, const void* pb) {
  const uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
  const uint64_t da = g_sort_ro[a + 1] - g_sort_ro[a], db = g_sort_ro[b + 1] - g_sort_ro[b];
  if (da != db) return da > db ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0);
}

/* cache.cpp:12-46. device_map i32[n] (-1 = miss). Returns #cached, -1 if
 * num_devices < 1. */
int64_t orc_build_static_cache(uint64_t num_nodes, const uint64_t* row_offsets, uint32_t feat_dim,
                               uint64_t volume_bytes, uint32_t num_devices, int32_t* device_map) {
  if (num_devices < 1) return -1;
  for (uint64_t v = 0; v < num_nodes; ++v) device_map[v] = -1;
  const uint64_t node_cost = (uint64_t)feat_dim * 4;
  if (volume_bytes < node_cost) return 0;
  uint32_t* order = (uint32_t*)malloc(num_nodes * sizeof(uint32_t));
  for (uint64_t v = 0; v < num_nodes; ++v) order[v] = (uint32_t)v;
  g_sort_ro = row_offsets;
  qsort(order, num_nodes, sizeof(uint32_t), hot_cmp);
  uint64_t* used = (uint64_t*)calloc(num_devices, sizeof(uint64_t));
  uint32_t device = 0, full = 0;
  int64_t cached = 0;
  for (uint64_t i = 0; i < num_nodes; ++i) {
    if (full == num_devices) break;
    while (used[device] + node_cost > volume_bytes) device = (device + 1) % num_devices;
    device_map[order[i]] = (int32_t)device;
    ++cached;
    used[device] += node_cost;
    if (used[device] + node_cost > volume_bytes) ++full;
    device = (device + 1) % num_devices;
  }
  free(used);
  free(order);
  return cached;
}

/* cache.cpp:48-87 + kernels_scalar.cpp:95-101: gather f32 rows of
 * unique_nodes, count hits/misses, return B (batch bytes). */
uint64_t orc_retrieve_features(const float* features, uint32_t feat_dim, const int32_t* device_map,
                               const orc_batch* b, float* out, uint64_t* hits, uint64_t* misses) {
  uint64_t h = 0, m = 0, ne = 0;
  for (uint64_t i = 0; i < b->n_unique; ++i) {
    const uint32_t v = b->unique[i];
    if (device_map && device_map[v] != -1)
      ++h;
    else
      ++m;
    memcpy(out + i * feat_dim, features + (uint64_t)v * feat_dim, feat_dim * sizeof(float));
  }
  for (uint32_t l = 0; l < b->num_layers; ++l) ne += b->layer_ne[l];
  *hits += h;
  *misses += m;
  return b->n_unique * feat_dim * 4 + ne * 2 * 4;
}

/* ------------------------------------------------------------ trainer ---- */
/* trainer.cpp:12-28 */
int orc_init_model(uint32_t F, uint32_t H, uint32_t C, uint64_t seed, double* w1, double* w2) {
  if (F < 1 || H < 1 || C < 1) return -1;
  rng_t rng = rng_make(seed, 0x6a10);
  double a = sqrt(6.0 / ((double)F + H));
  for (uint64_t i = 0; i < (uint64_t)F * H; ++i) w1[i] = (2.0 * next_unit(&rng) - 1.0) * a;
  a = sqrt(6.0 / ((double)H + C));
  for (uint64_t i = 0; i < (uint64_t)H * C; ++i) w2[i] = (2.0 * next_unit(&rng) - 1.0) * a;
  return 0;
}

/* kernels_scalar.cpp:40-72 scalar semantics */
static void mm_accum(const double* a, const double* b, double* c, uint64_t m, uint64_t k,
                     uint64_t n) {
  for (uint64_t i = 0; i < m; ++i)
    for (uint64_t r = 0; r < k; ++r) {
      const double aik = a[i * k + r];
      const double* brow = b + r * n;
      double* crow = c + i * n;
      for (uint64_t j = 0; j < n; ++j) crow[j] += aik * brow[j];
    }
}
static void mm_at_b_accum(const double* a, const double* b, double* c, uint64_t k, uint64_t m,
                          uint64_t n) {
  for (uint64_t r = 0; r < k; ++r) {
    const double* brow = b + r * n;
    for (uint64_t i = 0; i < m; ++i) {
      const double ari = a[r * m + i];
      double* crow = c + i * n;
      for (uint64_t j = 0; j < n; ++j) crow[j] += ari * brow[j];
    }
  }
}
static void mm_a_bt_accum(const double* a, const double* b, double* c, uint64_t m, uint64_t n,
                          uint64_t k) {
  for (uint64_t i = 0; i < m; ++i) {
    const double* arow = a + i * n;
    for (uint64_t t = 0; t < k; ++t) {
      double s = 0.0;
      const double* brow = b + t * n;
      for (uint64_t x = 0; x < n; ++x) s += arow[x] * brow[x];
      c[i * k + t] += s;
    }
  }
}

/* trainer.cpp:34-55 */
static void mean_aggregate(uint64_t ne, const uint32_t* ed, const uint32_t* es, const double* src,
                           uint64_t dim, const uint32_t* dst_rows_of, const int32_t* src_rows_of,
                           double* dst, uint64_t n_rows, uint32_t* deg) {
  memset(deg, 0, n_rows * sizeof(uint32_t));
  memset(dst, 0, n_rows * dim * sizeof(double));
  for (uint64_t e = 0; e < ne; ++e) {
    const uint32_t row = dst_rows_of[ed[e]];
    if (row == INV32) continue;
    const uint32_t srow = src_rows_of ? (uint32_t)src_rows_of[es[e]] : es[e];
    const double* x = src + (uint64_t)srow * dim;
    double* acc = dst + (uint64_t)row * dim;
    for (uint64_t i = 0; i < dim; ++i) acc[i] += x[i];
    ++deg[row];
  }
  for (uint64_t r = 0; r < n_rows; ++r)
    if (deg[r] > 0) {
      const double s = 1.0 / (double)deg[r];
      for (uint64_t i = 0; i < dim; ++i) dst[r * dim + i] *= s;
    }
}

/* Intermediates of forward() (trainer.hpp:49-60). Caller-sized buffers may
 * be NULL when not wanted; n_inner is returned through *n_inner_out. */
typedef struct {
  uint64_t n_inner;
  double* agg_inner; /* n_inner x F */
  double* h1;        /* n_inner x H */
  double* agg_outer; /* n_seeds x H */
  double* logits;    /* n_seeds x C */
  uint32_t* inner_nodes;
  int32_t* inner_pos;
  uint32_t* inner_deg;
  uint32_t* outer_deg;
} fwd_t;

static void fwd_free(fwd_t* f) {
  free(f->agg_inner);
  free(f->h1);
  free(f->agg_outer);
  free(f->logits);
  free(f->inner_nodes);
  free(f->inner_pos);
  free(f->inner_deg);
  free(f->outer_deg);
}

/* trainer.cpp:59-137. Batch given as arrays (layers[0], layers[1] only). */
static void forward(uint32_t F, uint32_t H, uint32_t C, const double* w1, const double* w2,
                    uint64_t n_unique, uint64_t n_seeds, uint32_t num_layers, const uint64_t* ne,
                    const uint32_t* const* ed, const uint32_t* const* es, const float* feats,
                    fwd_t* o) {
  double* featsd = (double*)malloc(n_unique * F * sizeof(double) + 8);
  for (uint64_t i = 0; i < n_unique * F; ++i) featsd[i] = (double)feats[i];
  o->inner_pos = (int32_t*)malloc(n_unique * sizeof(int32_t) + 4);
  o->inner_nodes = (uint32_t*)malloc(n_unique * sizeof(uint32_t) + 4);
  for (uint64_t i = 0; i < n_unique; ++i) o->inner_pos[i] = -1;
  uint64_t ni = 0;
  for (uint64_t s = 0; s < n_seeds; ++s) {
    o->inner_pos[s] = (int32_t)ni;
    o->inner_nodes[ni++] = (uint32_t)s;
  }
  if (num_layers >= 1)
    for (uint64_t e = 0; e < ne[0]; ++e) {
      const uint32_t s = es[0][e];
      if (o->inner_pos[s] < 0) {
        o->inner_pos[s] = (int32_t)ni;
        o->inner_nodes[ni++] = s;
      }
    }
  o->n_inner = ni;
  o->agg_inner = (double*)malloc(ni * F * sizeof(double) + 8);
  o->inner_deg = (uint32_t*)malloc(ni * sizeof(uint32_t) + 4);
  uint32_t* inner_row_of = (uint32_t*)malloc(n_unique * sizeof(uint32_t) + 4);
  memset(inner_row_of, 0xff, n_unique * sizeof(uint32_t));
  for (uint64_t r = 0; r < ni; ++r) inner_row_of[o->inner_nodes[r]] = (uint32_t)r;
  if (num_layers >= 2)
    mean_aggregate(ne[1], ed[1], es[1], featsd, F, inner_row_of, NULL, o->agg_inner, ni,
                   o->inner_deg);
  else
    mean_aggregate(0, NULL, NULL, featsd, F, inner_row_of, NULL, o->agg_inner, ni, o->inner_deg);
  for (uint64_t r = 0; r < ni; ++r)
    if (o->inner_deg[r] == 0)
      memcpy(o->agg_inner + r * F, featsd + (uint64_t)o->inner_nodes[r] * F, F * sizeof(double));
  o->h1 = (double*)calloc(ni * H + 1, sizeof(double));
  mm_accum(o->agg_inner, w1, o->h1, ni, F, H);
  for (uint64_t i = 0; i < ni * H; ++i) o->h1[i] = o->h1[i] > 0.0 ? o->h1[i] : 0.0;
  o->agg_outer = (double*)malloc(n_seeds * H * sizeof(double) + 8);
  o->outer_deg = (uint32_t*)malloc(n_seeds * sizeof(uint32_t) + 4);
  uint32_t* seed_row_of = (uint32_t*)malloc(n_unique * sizeof(uint32_t) + 4);
  memset(seed_row_of, 0xff, n_unique * sizeof(uint32_t));
  for (uint64_t s = 0; s < n_seeds; ++s) seed_row_of[s] = (uint32_t)s;
  if (num_layers >= 1)
    mean_aggregate(ne[0], ed[0], es[0], o->h1, H, seed_row_of, o->inner_pos, o->agg_outer, n_seeds,
                   o->outer_deg);
  else
    mean_aggregate(0, NULL, NULL, o->h1, H, seed_row_of, o->inner_pos, o->agg_outer, n_seeds,
                   o->outer_deg);
  for (uint64_t s = 0; s < n_seeds; ++s)
    if (o->outer_deg[s] == 0)
      memcpy(o->agg_outer + s * H, o->h1 + (uint64_t)o->inner_pos[s] * H, H * sizeof(double));
  o->logits = (double*)calloc(n_seeds * C + 1, sizeof(double));
  mm_accum(o->agg_outer, w2, o->logits, n_seeds, H, C);
  free(featsd);
  free(inner_row_of);
  free(seed_row_of);
}

/* trainer.cpp:139-206; returns mean loss */
static double backward(uint32_t F, uint32_t H, uint32_t C, const double* w2, uint64_t n_seeds,
                       uint32_t num_layers, const uint64_t* ne, const uint32_t* const* ed,
                       const uint32_t* const* es, const fwd_t* f, const uint32_t* labels,
                       double* gw1, double* gw2) {
  const uint64_t ni = f->n_inner;
  memset(gw1, 0, (uint64_t)F * H * sizeof(double));
  memset(gw2, 0, (uint64_t)H * C * sizeof(double));
  double* dlogits = (double*)malloc(n_seeds * C * sizeof(double) + 8);
  double loss = 0.0;
  const double inv_n = 1.0 / (double)n_seeds;
  for (uint64_t s = 0; s < n_seeds; ++s) {
    const double* row = f->logits + s * C;
    double* drow = dlogits + s * C;
    double mx = row[0];
    for (uint32_t c = 1; c < C; ++c) mx = mx > row[c] ? mx : row[c]; /* std::max */
    double denom = 0.0;
    for (uint32_t c = 0; c < C; ++c) denom += exp(row[c] - mx);
    const uint32_t y = labels[s];
    loss += -(row[y] - mx - log(denom));
    for (uint32_t c = 0; c < C; ++c) {
      const double p = exp(row[c] - mx) / denom;
      drow[c] = (p - (c == y ? 1.0 : 0.0)) * inv_n;
    }
  }
  loss *= inv_n;
  mm_at_b_accum(f->agg_outer, dlogits, gw2, n_seeds, H, C);
  double* dagg = (double*)calloc(n_seeds * H + 1, sizeof(double));
  mm_a_bt_accum(dlogits, w2, dagg, n_seeds, C, H);
  double* dh1 = (double*)calloc(ni * H + 1, sizeof(double));
  if (num_layers >= 1)
    for (uint64_t e = 0; e < ne[0]; ++e) {
      const uint32_t d = ed[0][e], s = es[0][e];
      if (d >= n_seeds) continue;
      const double w = 1.0 / (double)f->outer_deg[d];
      const double* x = dagg + (uint64_t)d * H;
      double* y = dh1 + (uint64_t)f->inner_pos[s] * H;
      for (uint32_t i = 0; i < H; ++i) y[i] += w * x[i];
    }
  for (uint64_t s = 0; s < n_seeds; ++s)
    if (f->outer_deg[s] == 0) {
      const double* x = dagg + s * H;
      double* y = dh1 + (uint64_t)f->inner_pos[s] * H;
      for (uint32_t i = 0; i < H; ++i) y[i] += x[i];
    }
  for (uint64_t i = 0; i < ni * H; ++i)
    if (f->h1[i] <= 0.0) dh1[i] = 0.0;
  mm_at_b_accum(f->agg_inner, dh1, gw1, ni, F, H);
  free(dlogits);
  free(dagg);
  free(dh1);
  return loss;
}

/* grad_on_batch (trainer.cpp:231-239) with optional intermediates out.
 * labels_of_node: u32[num_nodes] (graph labels). Returns loss. */
double orc_grad_on_batch(uint32_t F, uint32_t H, uint32_t C, const double* w1, const double* w2,
                         const orc_batch* b, const float* feats, const uint32_t* labels_of_node,
                         double* gw1, double* gw2, uint64_t* n_inner_out, double* logits_out,
                         double* agg_inner_out, double* h1_out, double* agg_outer_out) {
  fwd_t f;
  memset(&f, 0, sizeof f);
  const uint64_t ns = b->num_seed_unique;
  forward(F, H, C, w1, w2, b->n_unique, ns, b->num_layers, b->layer_ne,
          (const uint32_t* const*)b->layer_dst, (const uint32_t* const*)b->layer_src, feats, &f);
  uint32_t* labels = (uint32_t*)malloc(ns * sizeof(uint32_t) + 4);
  for (uint64_t s = 0; s < ns; ++s) labels[s] = labels_of_node[b->unique[s]];
  const double loss = backward(F, H, C, w2, ns, b->num_layers, b->layer_ne,
                               (const uint32_t* const*)b->layer_dst,
                               (const uint32_t* const*)b->layer_src, &f, labels, gw1, gw2);
  if (n_inner_out) *n_inner_out = f.n_inner;
  if (logits_out) memcpy(logits_out, f.logits, ns * C * sizeof(double));
  if (agg_inner_out) memcpy(agg_inner_out, f.agg_inner, f.n_inner * F * sizeof(double));
  if (h1_out) memcpy(h1_out, f.h1, f.n_inner * H * sizeof(double));
  if (agg_outer_out) memcpy(agg_outer_out, f.agg_outer, ns * H * sizeof(double));
  free(labels);
  fwd_free(&f);
  return loss;
}

/* Explicit-batch forward for hand-built fixtures (test_trainer.cpp:22-35):
 * layers given as flat (dst,src) arrays. */
double orc_grad_on_edges(uint32_t F, uint32_t H, uint32_t C, const double* w1, const double* w2,
                         uint64_t n_unique, uint64_t n_seeds, uint32_t num_layers,
                         const uint64_t* ne, const uint32_t* const* ed, const uint32_t* const* es,
                         const float* feats, const uint32_t* seed_labels, double* gw1, double* gw2,
                         double* logits_out) {
  fwd_t f;
  memset(&f, 0, sizeof f);
  forward(F, H, C, w1, w2, n_unique, n_seeds, num_layers, ne, ed, es, feats, &f);
  const double loss =
      backward(F, H, C, w2, n_seeds, num_layers, ne, ed, es, &f, seed_labels, gw1, gw2);
  if (logits_out) memcpy(logits_out, f.logits, n_seeds * C * sizeof(double));
  fwd_free(&f);
  return loss;
}

/* trainer.cpp:208-211 */
void orc_sgd_step(double* w, const double* g, uint64_t n, double lr) {
  const double a = -lr;
  for (uint64_t i = 0; i < n; ++i) w[i] += a * g[i];
}

/* The u=1 step loop of train() (trainer.cpp:350-407), bounded to `max_steps`
 * steps (spanning epochs). Writes per-step losses; updates w1/w2 in place.
 * Returns #steps run, or <0 on sampler error. */
int64_t orc_train_steps(uint64_t num_nodes, const uint64_t* row_offsets, const uint32_t* col,
                        const float* features, uint32_t F, const uint32_t* labels,
                        const uint8_t* train_mask, const int32_t* device_map,
                        const uint32_t* fanouts, uint32_t num_layers, double gamma, int kind,
                        uint64_t rng_seed, uint32_t batch_size, uint32_t H, uint32_t C, double lr,
                        double* w1, double* w2, uint64_t max_steps, double* losses,
                        uint64_t* hits, uint64_t* misses) {
  uint64_t n_train = 0;
  for (uint64_t v = 0; v < num_nodes; ++v) n_train += train_mask[v] ? 1 : 0;
  if (n_train == 0 || batch_size < 1) return -10;
  uint32_t* train_nodes = (uint32_t*)malloc(n_train * sizeof(uint32_t));
  uint32_t* order = (uint32_t*)malloc(n_train * sizeof(uint32_t));
  n_train = 0;
  for (uint64_t v = 0; v < num_nodes; ++v)
    if (train_mask[v]) train_nodes[n_train++] = (uint32_t)v;
  double* gw1 = (double*)malloc((uint64_t)F * H * sizeof(double));
  double* gw2 = (double*)malloc((uint64_t)H * C * sizeof(double));
  const uint64_t steps_per_epoch = (n_train + batch_size - 1) / batch_size;
  uint64_t done = 0;
  int64_t ret = 0;
  for (uint32_t epoch = 0; done < max_steps; ++epoch) {
    orc_plan_epoch_order(train_nodes, n_train, epoch, hash2(rng_seed, 0), order);
    for (uint64_t step = 0; step < steps_per_epoch && done < max_steps; ++step) {
      const uint64_t beg = step * batch_size;
      const uint64_t nb = (beg + batch_size <= n_train) ? batch_size : n_train - beg;
      int err = 0;
      const uint64_t sseed = orc_sampling_seed(rng_seed, epoch, (uint32_t)step, 0);
      orc_batch* b = orc_sample_khop(num_nodes, row_offsets, col, order + beg, nb, fanouts,
                                     num_layers, gamma, kind, sseed, device_map, &err);
      if (!b) {
        ret = -(int64_t)err;
        goto out;
      }
      float* feats = (float*)malloc(b->n_unique * F * sizeof(float) + 4);
      orc_retrieve_features(features, F, device_map, b, feats, hits, misses);
      losses[done] = orc_grad_on_batch(F, H, C, w1, w2, b, feats, labels, gw1, gw2, NULL, NULL,
                                       NULL, NULL, NULL);
      /* sync_gradients over one worker: 0 + g, then * 1.0 (trainer.cpp:213-229) */
      orc_sgd_step(w1, gw1, (uint64_t)F * H, lr);
      orc_sgd_step(w2, gw2, (uint64_t)H * C, lr);
      free(feats);
      orc_batch_free(b);
      ++done;
    }
  }
  ret = (int64_t)done;
out:
  free(train_nodes);
  free(order);
  free(gw1);
  free(gw2);
  return ret;
}
