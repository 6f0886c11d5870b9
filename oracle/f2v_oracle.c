/* oracle/f2v_oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU checker for the
 * CUDA product path (see f2v_oracle.h for the pinning story).  Compiled with
 * -ffp-contract=off and no -march so each fp64 multiply and add rounds
 * separately, exactly as the reference's Release build does on x86-64.
 * Every block cites the reference file:line it restates. */
#include "f2v_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9e3779b97f4a7c15ull

/* ---------------------------------------------------------------- rng.hpp */
/* rng.hpp:44-49 */
uint64_t orc_mix(uint64_t z) {
  z += GAMMA;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
/* rng.hpp:14-15 */
uint64_t orc_rng_init(uint64_t seed, uint64_t stream) {
  return orc_mix(orc_mix(seed) ^ orc_mix(stream ^ GAMMA));
}
/* rng.hpp:18-24 */
uint64_t orc_rng_keyed(uint64_t seed, const uint64_t* key, int nkey) {
  uint64_t s = orc_mix(seed);
  for (int i = 0; i < nkey; ++i) s = orc_mix(s ^ orc_mix(key[i] ^ GAMMA));
  return s;
}
/* rng.hpp:26-29 */
uint64_t orc_rng_next(uint64_t* st) {
  *st += GAMMA;
  return orc_mix(*st);
}
/* rng.hpp:39-42 */
uint64_t orc_rng_below(uint64_t* st, uint64_t n) {
  return (uint64_t)(((unsigned __int128)orc_rng_next(st) * n) >> 64);
}
/* rng.hpp:32 */
double orc_rng_uniform(uint64_t* st) {
  return (double)(orc_rng_next(st) >> 11) * 0x1.0p-53;
}
void orc_rng_draws(uint64_t st, uint64_t count, uint64_t* out) {
  for (uint64_t i = 0; i < count; ++i) out[i] = orc_rng_next(&st);
}

/* ------------------------------------------------------------- Philox4x32 */
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
  const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  const uint32_t n0 = hi1 ^ c[1] ^ k[0];
  const uint32_t n2 = hi0 ^ c[3] ^ k[1];
  c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  uint32_t k[2] = {key[0], key[1]};
  for (int r = 0; r < 10; ++r) {
    if (r) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
    philox_round(c, k);
  }
  memcpy(out, c, sizeof c);
}
/* Negative k of (epoch, batch, gpu): counter {k, batch_lo, epoch,
 * batch_hi<<16 | gpu}... see DESIGN.md "Samplers" for the exact layout. */
void orc_philox_negatives(uint64_t seed, uint32_t epoch, uint64_t batch, uint32_t gpu,
                          uint32_t n, uint32_t s, uint32_t* out) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (uint32_t k = 0; k < s; ++k) {
    const uint32_t ctr[4] = {k, (uint32_t)batch, epoch,
                             ((uint32_t)(batch >> 32) << 16) | (gpu & 0xffffu)};
    uint32_t r[4];
    orc_philox4x32_10(ctr, key, r);
    const uint64_t draw = ((uint64_t)r[1] << 32) | r[0];
    out[k] = (uint32_t)(((unsigned __int128)draw * n) >> 64);
  }
}
/* sampling.cpp:21-25 with train()'s key (trainer.cpp:222-224) */
void orc_ref_negatives(uint64_t seed, uint32_t epoch, uint64_t batch, uint32_t n,
                       uint32_t s, uint32_t* out) {
  const uint64_t key[3] = {0x33, epoch, batch};
  uint64_t st = orc_rng_keyed(seed, key, 3);
  for (uint32_t k = 0; k < s; ++k) out[k] = (uint32_t)orc_rng_below(&st, n);
}

/* ------------------------------------------------------------ embeddings */
void orc_random_embedding(uint32_t n, uint32_t d, uint64_t seed, float* out) {
  uint64_t st = orc_rng_init(seed, 0);
  const size_t total = (size_t)n * d;
  for (size_t i = 0; i < total; ++i)
    out[i] = (float)(-1.0 + (1.0 - -1.0) * orc_rng_uniform(&st)); /* rng.hpp:35 */
}
void orc_init_embedding(uint32_t n, uint32_t d, uint64_t seed, float* out) {
  const uint64_t key[1] = {0x11};
  uint64_t st = orc_rng_keyed(seed, key, 1);
  const double half = 0.5 / (double)d;
  const size_t total = (size_t)n * d;
  for (size_t i = 0; i < total; ++i)
    out[i] = (float)(-half + (half - -half) * orc_rng_uniform(&st));
}

/* --------------------------------------------------------- sampling.cpp:7 */
int orc_partition(uint32_t n, uint32_t b, uint64_t st, uint32_t* perm) {
  if (b == 0 || b > n) return 1; /* UsageError, sampling.cpp:8 */
  for (uint32_t i = 0; i < n; ++i) perm[i] = i;
  for (uint32_t i = n; i > 1; --i) {
    const uint32_t j = (uint32_t)orc_rng_below(&st, i);
    const uint32_t t = perm[i - 1];
    perm[i - 1] = perm[j];
    perm[j] = t;
  }
  return 0;
}

/* --------------------------------------------------- csr_graph.cpp:57-97 */
static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}
int orc_from_edges(const uint32_t* pairs, uint64_t m, uint32_t n, int symmetrize,
                   uint64_t* rowptr, uint32_t* col, uint64_t* nnz_out,
                   uint64_t* dups_out, uint64_t* loops_out) {
  uint64_t* e = (uint64_t*)malloc(sizeof(uint64_t) * (2 * m + 1));
  uint64_t k = 0, loops = 0;
  for (uint64_t i = 0; i < m; ++i) {
    const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u == v) { ++loops; continue; }
    e[k++] = ((uint64_t)u << 32) | v;
  }
  if (symmetrize) {
    const uint64_t kk = k;
    for (uint64_t i = 0; i < kk; ++i) e[k++] = (e[i] << 32) | (e[i] >> 32);
  }
  qsort(e, k, sizeof(uint64_t), cmp_u64);
  uint64_t w = 0;
  for (uint64_t i = 0; i < k; ++i)
    if (w == 0 || e[i] != e[w - 1]) e[w++] = e[i];
  uint64_t dups = k - w;
  if (symmetrize) dups /= 2;
  for (uint32_t u = 0; u <= n; ++u) rowptr[u] = 0;
  for (uint64_t i = 0; i < w; ++i) {
    const uint32_t u = (uint32_t)(e[i] >> 32), v = (uint32_t)e[i];
    if (u >= n || v >= n) { free(e); return 3; } /* RangeError */
    ++rowptr[u + 1];
  }
  for (uint32_t u = 0; u < n; ++u) rowptr[u + 1] += rowptr[u];
  for (uint64_t i = 0; i < w; ++i) col[i] = (uint32_t)e[i];
  free(e);
  if (nnz_out) *nnz_out = w;
  if (dups_out) *dups_out = dups;
  if (loops_out) *loops_out = loops;
  return 0;
}

/* tests/support/test_graphs.hpp:67-78 */
uint64_t orc_sbm_edges(uint32_t n, int blocks, double p_in, double p_out, uint64_t seed,
                       uint32_t* pairs, uint64_t cap) {
  uint64_t st = orc_rng_init(seed, 0);
  const uint32_t bs = n / (uint32_t)blocks;
  uint64_t m = 0;
  for (uint32_t u = 0; u < n; ++u)
    for (uint32_t v = u + 1; v < n; ++v) {
      const int same = u / bs == v / bs;
      if (orc_rng_uniform(&st) < (same ? p_in : p_out)) {
        if (m < cap) { pairs[2 * m] = u; pairs[2 * m + 1] = v; }
        ++m;
      }
    }
  return m;
}

/* ------------------------------------------------- force_kernels.cpp:30-77 */
static double dot(const float* a, const float* b, uint32_t d) {
  double s = 0.0;
  for (uint32_t i = 0; i < d; ++i) s += (double)a[i] * (double)b[i];
  return s;
}
static double distance(const float* a, const float* b, uint32_t d) {
  double s = 0.0;
  for (uint32_t i = 0; i < d; ++i) {
    const double t = (double)a[i] - (double)b[i];
    s += t * t;
  }
  return sqrt(s);
}
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static void scale_into(double c, const float* v, uint32_t d, double* out) {
  for (uint32_t i = 0; i < d; ++i) out[i] = c * (double)v[i];
}
static void scaled_unit_diff(double scalar, const float* zu, const float* zo, double t,
                             double eps, uint32_t d, double* out) {
  if (t < eps) {
    for (uint32_t i = 0; i < d; ++i) out[i] = 0.0;
    if (d) out[0] = scalar;
    return;
  }
  for (uint32_t i = 0; i < d; ++i)
    out[i] = scalar * ((double)zu[i] - (double)zo[i]) / t;
}
static void clamp_magnitude(float capf, double magnitude, uint32_t d, double* out) {
  if (isnan(capf)) return; /* repulsion_cap unset (std::nullopt); 0 still clamps */
  const double cap = (double)capf;
  if (magnitude <= cap || magnitude == 0.0) return;
  const double scale = cap / magnitude;
  for (uint32_t i = 0; i < d; ++i) out[i] = out[i] * scale;
}
/* force_kernels.hpp:25-29 */
double orc_stable_sigmoid(double x) {
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  const double e = exp(x);
  return e / (1.0 + e);
}

/* force_kernels.cpp:79-169 */
int orc_pair_grad(int kind, float epsf, float cap, const float* zu, const float* zo,
                  uint32_t d, int attractive, double* out) {
  const double eps = (double)epsf;
  if (kind == ORC_SIGMOID) {
    if (attractive) { /* 79-86 */
      const double coef = orc_stable_sigmoid(dot(zu, zo, d)) - 1.0;
      scale_into(coef, zo, d, out);
    } else { /* 88-97 */
      const double coef = orc_stable_sigmoid(dot(zu, zo, d));
      scale_into(coef, zo, d, out);
      const double norm_w = sqrt(dot(zo, zo, d));
      clamp_magnitude(cap, coef * norm_w, d, out);
    }
    return 0;
  }
  if (kind == ORC_TDIST) {
    if (attractive) { /* 99-107 */
      const double t = distance(zu, zo, d);
      const double scalar = 2.0 * t / (1.0 + t * t);
      scaled_unit_diff(scalar, zu, zo, t, eps, d, out);
    } else { /* 109-119 */
      const double t_raw = distance(zu, zo, d);
      const double t = dmax(t_raw, eps);
      const double scalar = -2.0 / (t * (1.0 + t * t));
      scaled_unit_diff(scalar, zu, zo, t_raw, eps, d, out);
      clamp_magnitude(cap, fabs(scalar), d, out);
    }
    return 0;
  }
  if (kind < ORC_FR || kind > ORC_LINLOG) return 6; /* UnsupportedError */
  { /* 121-147 */
    const double r_raw = distance(zu, zo, d);
    double scalar;
    if (attractive) {
      if (kind == ORC_FR) scalar = r_raw * r_raw;
      else if (kind == ORC_FA) scalar = r_raw;
      else scalar = log1p(r_raw);
      scaled_unit_diff(scalar, zu, zo, r_raw, eps, d, out);
      return 0;
    }
    scalar = -1.0 / dmax(r_raw, eps);
    scaled_unit_diff(scalar, zu, zo, r_raw, eps, d, out);
    clamp_magnitude(cap, fabs(scalar), d, out);
  }
  return 0;
}

/* force_kernels.cpp:211-231 */
int orc_pair_loss(int kind, float epsf, float cap, const float* zu, const float* zv,
                  uint32_t d, int attractive, double* out) {
  (void)cap;
  if (kind == ORC_SIGMOID) {
    const double x = dot(zu, zv, d);
    if (attractive)
      *out = x >= 0 ? log1p(exp(-x)) : -x + log1p(exp(x));
    else
      *out = x >= 0 ? x + log1p(exp(-x)) : log1p(exp(x));
    return 0;
  }
  if (kind == ORC_TDIST) {
    const double t = distance(zu, zv, d);
    const double t2 = t * t;
    if (attractive) { *out = log1p(t2); return 0; }
    const double tc = dmax(t2, (double)epsf * (double)epsf);
    *out = -log(tc / (1.0 + tc));
    return 0;
  }
  return 6;
}

/* ---------------------------------------------------- trainer.cpp:108-165 */
typedef struct {
  const uint64_t* rowptr; const uint32_t* col; const float* z; uint32_t d;
  const uint32_t* ids; const uint32_t* negs; uint32_t s; int kind; float eps, cap;
  float* grads; uint32_t lo, hi; uint32_t bad_index; /* first bad batch index */
} grad_job;

static void* grad_worker(void* arg) {
  grad_job* j = (grad_job*)arg;
  const uint32_t d = j->d;
  double* acc = (double*)malloc(sizeof(double) * d);
  double* pair = (double*)malloc(sizeof(double) * d);
  j->bad_index = UINT32_MAX;
  for (uint32_t i = j->lo; i < j->hi && j->bad_index == UINT32_MAX; ++i) {
    const uint32_t u = j->ids[i];
    const float* zu = j->z + (size_t)u * d;
    for (uint32_t c = 0; c < d; ++c) acc[c] = 0.0;
    for (uint64_t e = j->rowptr[u]; e < j->rowptr[u + 1]; ++e) {
      orc_pair_grad(j->kind, j->eps, j->cap, zu, j->z + (size_t)j->col[e] * d, d, 1, pair);
      for (uint32_t c = 0; c < d; ++c) acc[c] += pair[c];
    }
    for (uint32_t k = 0; k < j->s; ++k) {
      orc_pair_grad(j->kind, j->eps, j->cap, zu, j->z + (size_t)j->negs[k] * d, d, 0, pair);
      for (uint32_t c = 0; c < d; ++c) acc[c] += pair[c];
    }
    float* out = j->grads + (size_t)i * d;
    for (uint32_t c = 0; c < d; ++c) {
      const float v = (float)acc[c];
      if (!isfinite(v)) j->bad_index = i;
      out[c] = v;
    }
  }
  free(acc);
  free(pair);
  return NULL;
}

int orc_grad_minibatch(const uint64_t* rowptr, const uint32_t* col, uint32_t n,
                       const float* z, uint32_t d, const uint32_t* ids, uint32_t b,
                       const uint32_t* negs, uint32_t s, int kind, float eps, float cap,
                       int threads, float* grads, uint32_t* bad_vertex) {
  (void)n;
  if (kind < 0 || kind > ORC_LINLOG) return 6;
  if (threads < 1) threads = 1;
  if ((uint32_t)threads > b) threads = b ? (int)b : 1;
  grad_job jobs[256];
  pthread_t tid[256];
  if (threads > 256) threads = 256;
  for (int w = 0; w < threads; ++w) {
    grad_job g = {rowptr, col, z, d, ids, negs, s, kind, eps, cap, grads,
                  (uint32_t)((uint64_t)w * b / threads),
                  (uint32_t)((uint64_t)(w + 1) * b / threads), UINT32_MAX};
    jobs[w] = g;
  }
  for (int w = 1; w < threads; ++w) pthread_create(&tid[w], NULL, grad_worker, &jobs[w]);
  grad_worker(&jobs[0]);
  for (int w = 1; w < threads; ++w) pthread_join(tid[w], NULL);
  for (int w = 0; w < threads; ++w)
    if (jobs[w].bad_index != UINT32_MAX) {
      if (bad_vertex) *bad_vertex = ids[jobs[w].bad_index];
      return 4; /* NumericalError, trainer.cpp:149-152 */
    }
  return 0;
}

/* trainer.cpp:167-175 */
void orc_apply_update(float* z, uint32_t d, const uint32_t* ids, uint32_t b,
                      const float* grads, float eta) {
  for (uint32_t i = 0; i < b; ++i) {
    float* row = z + (size_t)ids[i] * d;
    const float* g = grads + (size_t)i * d;
    for (uint32_t c = 0; c < d; ++c) row[c] -= eta * g[c];
  }
}

/* trainer.cpp:177-190 */
int orc_batch_loss(const uint64_t* rowptr, const uint32_t* col, const float* z,
                   uint32_t d, const uint32_t* ids, uint32_t b, const uint32_t* negs,
                   uint32_t s, int kind, float eps, float cap, double* out) {
  if (kind != ORC_SIGMOID && kind != ORC_TDIST) return 6;
  double total = 0.0, l;
  for (uint32_t i = 0; i < b; ++i) {
    const uint32_t u = ids[i];
    const float* zu = z + (size_t)u * d;
    for (uint64_t e = rowptr[u]; e < rowptr[u + 1]; ++e) {
      orc_pair_loss(kind, eps, cap, zu, z + (size_t)col[e] * d, d, 1, &l);
      total += l;
    }
    for (uint32_t k = 0; k < s; ++k) {
      orc_pair_loss(kind, eps, cap, zu, z + (size_t)negs[k] * d, d, 0, &l);
      total += l;
    }
  }
  *out = total;
  return 0;
}

/* ------------------------------------------------------ trainer.cpp:192-251 */
/* Vertex shards of a G-GPU run (no reference
 * counterpart -- the reference is single-process).  G == 1 is exactly
 * train(): one shard, batch min(batch, n) (trainer.cpp:200).  G > 1:
 *   - contiguous row ranges cut at quantiles of the per-vertex work
 *     w(u) = deg(u) + s (its pair evaluations per epoch): lo[g] is the first u
 *     whose work prefix reaches floor(g W / G), W = nnz + n s, kept strictly
 *     increasing so every shard owns at least one row;
 *   - T = ceil(n / (G batch)) steps; shard g's local batch is
 *     ceil(size_g / T), so every shard finishes in (at most) T steps and the
 *     per-step work is balanced as well as the per-epoch work. */
void orc_shard_layout(const uint64_t* rowptr, uint32_t n, uint32_t G, uint32_t s,
                      uint32_t batch, uint32_t* lo, uint32_t* bs, uint32_t* nb, uint64_t* T) {
  lo[0] = 0;
  lo[G] = n;
  if (G == 1) {
    bs[0] = batch < n ? batch : n;
    nb[0] = (n + bs[0] - 1) / bs[0];
    *T = nb[0];
    return;
  }
  const uint64_t W = rowptr[n] + (uint64_t)n * s;
  for (uint32_t g = 1; g < G; ++g) {
    const uint64_t target = W * g / G;
    uint32_t a = 0, b = n; /* first u in [0, n] with rowptr[u] + u s >= target */
    while (a < b) {
      const uint32_t m = a + (b - a) / 2;
      if (rowptr[m] + (uint64_t)m * s >= target) b = m; else a = m + 1;
    }
    uint32_t x = a;
    if (x < lo[g - 1] + 1) x = lo[g - 1] + 1;
    if (x > n - (G - g)) x = n - (G - g);
    lo[g] = x;
  }
  const uint64_t gb = (uint64_t)G * batch;
  const uint64_t steps = ((uint64_t)n + gb - 1) / gb;
  uint64_t t = 0;
  for (uint32_t g = 0; g < G; ++g) {
    const uint32_t sz = lo[g + 1] - lo[g];
    bs[g] = (uint32_t)(((uint64_t)sz + steps - 1) / steps);
    nb[g] = (sz + bs[g] - 1) / bs[g];
    if (nb[g] > t) t = nb[g];
  }
  *T = t;
}

/* gen_walk (sampling.cpp:27-41): k steps from u on the stream st (one below()
 * per step); a dead end restarts at u; an isolated u yields no walk. */
static void orc_gen_walk(const uint64_t* rowptr, const uint32_t* col, uint32_t u, uint32_t k,
                         uint64_t* st, uint32_t* out) {
  if (rowptr[u + 1] == rowptr[u]) return;
  uint32_t w = u;
  for (uint32_t i = 0; i < k; ++i) {
    if (rowptr[w + 1] == rowptr[w]) w = u; /* dead end: restart */
    const uint64_t deg = rowptr[w + 1] - rowptr[w];
    const uint32_t next = col[rowptr[w] + orc_rng_below(st, deg)];
    out[i] = next;
    w = next;
  }
}

int orc_train(const uint64_t* rowptr, const uint32_t* col, uint32_t n, float* z,
              uint32_t d, uint32_t batch, uint32_t s, float lr, uint32_t epochs,
              int kind, float eps, float cap, uint64_t seed, int lr_decay, int monitor,
              int sampler, uint32_t G, int threads, double* loss_out,
              uint64_t* counters, orc_step_cb cb, void* user, uint32_t* fail_info) {
  return orc_train_mode(rowptr, col, n, z, d, batch, s, lr, epochs, kind, eps, cap, seed,
                        lr_decay, monitor, sampler, G, 0, threads, loss_out, counters, cb, user,
                        fail_info);
}

int orc_train_mode(const uint64_t* rowptr, const uint32_t* col, uint32_t n, float* z,
                   uint32_t d, uint32_t batch, uint32_t s, float lr, uint32_t epochs,
                   int kind, float eps, float cap, uint64_t seed, int lr_decay, int monitor,
                   int sampler, uint32_t G, uint32_t walk_k, int threads, double* loss_out,
                   uint64_t* counters, orc_step_cb cb, void* user, uint32_t* fail_info) {
  if (d < 1 || batch < 1 || s < 1 || !(lr > 0) || epochs < 1 || G < 1 || n < G)
    return 1; /* TrainConfig::validate, trainer.cpp:13-22 */
  /* walk mode (SampleMode::walk(k), sampling.hpp:12-20): the context of u is
   * its k-step walk; layout: ctx row u at k * (non-isolated vertices < u) */
  uint64_t* cptr = NULL;
  uint32_t* ccol = NULL;
  if (walk_k) {
    cptr = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
    cptr[0] = 0;
    for (uint32_t u = 0; u < n; ++u)
      cptr[u + 1] = cptr[u] + (rowptr[u + 1] > rowptr[u] ? walk_k : 0);
    ccol = (uint32_t*)malloc(sizeof(uint32_t) * (cptr[n] ? cptr[n] : 1));
  }
  const uint64_t* xptr = walk_k ? cptr : rowptr; /* the context CSR */
  const uint32_t* xcol = walk_k ? ccol : col;
  if (monitor && kind != ORC_SIGMOID && kind != ORC_TDIST) return 6;
  uint32_t* perms = (uint32_t*)malloc(sizeof(uint32_t) * n);
  uint32_t* lo = (uint32_t*)malloc(sizeof(uint32_t) * (G + 1));
  uint32_t* bs = (uint32_t*)malloc(sizeof(uint32_t) * G);
  uint32_t* nb = (uint32_t*)malloc(sizeof(uint32_t) * G);
  uint32_t* negs = (uint32_t*)malloc(sizeof(uint32_t) * s * G);
  uint32_t bmax = 0;
  uint64_t T = 0;
  orc_shard_layout(rowptr, n, G, s, batch, lo, bs, nb, &T);
  for (uint32_t g = 0; g < G; ++g)
    if (bs[g] > bmax) bmax = bs[g];
  float* grads = (float*)malloc(sizeof(float) * (size_t)bmax * d * G);
  uint64_t attr = 0, rep = 0;
  int rc = 0;
  for (uint32_t epoch = 0; epoch < epochs && rc == 0; ++epoch) {
    float eta = lr;
    if (lr_decay) eta = lr * (1.0f - (float)epoch / (float)epochs); /* 212-214 */
    for (uint32_t g = 0; g < G; ++g) {
      const uint32_t l = lo[g], h = lo[g + 1];
      const uint64_t key1[2] = {0x22, epoch}, keyG[3] = {0x22, epoch, g};
      const uint64_t st = G == 1 ? orc_rng_keyed(seed, key1, 2) : orc_rng_keyed(seed, keyG, 3);
      orc_partition(h - l, bs[g], st, perms + l);
      for (uint32_t i = l; i < h; ++i) perms[i] += l;
    }
    double epoch_loss = 0.0;
    for (uint64_t t = 0; t < T && rc == 0; ++t) {
      /* negatives per shard (sampling.cpp:59) */
      for (uint32_t g = 0; g < G; ++g) {
        /* build_minibatch (sampling.cpp:43-61): walks (walk mode) then the
         * negatives, on one stream (seed,{0x33,epoch,t[,g]}) */
        const uint64_t key3[3] = {0x33, epoch, t}, key4[4] = {0x33, epoch, t, g};
        uint64_t st = G == 1 ? orc_rng_keyed(seed, key3, 3) : orc_rng_keyed(seed, key4, 4);
        if (walk_k && t < nb[g]) {
          const uint32_t l = lo[g], h = lo[g + 1];
          const uint32_t p0 = l + (uint32_t)(t * bs[g]);
          const uint32_t p1 = (uint32_t)((uint64_t)p0 + bs[g] < h ? p0 + bs[g] : h);
          for (uint32_t p = p0; p < p1; ++p)
            orc_gen_walk(rowptr, col, perms[p], walk_k, &st, ccol + cptr[perms[p]]);
        }
        if (sampler == 1) {
          orc_philox_negatives(seed, epoch, t, g, n, s, negs + (size_t)g * s);
        } else {
          for (uint32_t k = 0; k < s; ++k) negs[g * s + k] = (uint32_t)orc_rng_below(&st, n);
        }
      }
      /* gradients of every shard's batch on the same snapshot */
      for (uint32_t g = 0; g < G && rc == 0; ++g) {
        if (t >= nb[g]) continue;
        const uint32_t l = lo[g], h = lo[g + 1];
        const uint32_t p0 = l + (uint32_t)(t * bs[g]);
        const uint32_t p1 = (uint32_t)((uint64_t)p0 + bs[g] < h ? p0 + bs[g] : h);
        uint32_t bad = 0;
        const int r = orc_grad_minibatch(xptr, xcol, n, z, d, perms + p0, p1 - p0,
                                         negs + (size_t)g * s, s, kind, eps, cap, threads,
                                         grads + (size_t)g * bmax * d, &bad);
        if (r) {
          rc = r;
          if (fail_info) { fail_info[0] = epoch; fail_info[1] = (uint32_t)t; fail_info[2] = bad; }
          break;
        }
        for (uint32_t p = p0; p < p1; ++p) attr += xptr[perms[p] + 1] - xptr[perms[p]];
        rep += (uint64_t)(p1 - p0) * s;
        if (monitor) {
          double l2 = 0.0;
          orc_batch_loss(xptr, xcol, z, d, perms + p0, p1 - p0, negs + (size_t)g * s, s,
                         kind, eps, cap, &l2);
          epoch_loss += l2;
        }
      }
      if (rc) break;
      for (uint32_t g = 0; g < G; ++g) {
        if (t >= nb[g]) continue;
        const uint32_t l = lo[g], h = lo[g + 1];
        const uint32_t p0 = l + (uint32_t)(t * bs[g]);
        const uint32_t p1 = (uint32_t)((uint64_t)p0 + bs[g] < h ? p0 + bs[g] : h);
        orc_apply_update(z, d, perms + p0, p1 - p0, grads + (size_t)g * bmax * d, eta);
      }
      if (cb) cb(epoch, t, z, user);
    }
    if (rc == 0 && monitor && loss_out) loss_out[epoch] = epoch_loss;
  }
  if (counters) { counters[0] = attr; counters[1] = rep; }
  free(perms); free(lo); free(bs); free(nb); free(negs); free(grads); free(cptr); free(ccol);
  return rc;
}
