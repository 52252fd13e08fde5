/*
 * gen.c -- seeded synthetic SPS workload generator (inputs only).
 *
 * This module is shared by the oracle side (oracle/, tests/) and the CUDA side
 * (bench.py, GPU tests).  It holds NONE of the method's arithmetic: no norms, no
 * similarity, no selection, no softmax, no weighted sum.  It only draws the
 * inputs whose shape and structure SURVEY.md §8(d) prescribes:
 *
 *   - clustered prompt embeddings (bf16 bits), the paper's premise that
 *     semantically similar prompts share activation patterns;
 *   - Zipf-skewed per-prompt activation tables s~_{l,k} = frec_{l,k} / sum_k frec
 *     with sum_k frec = N_in * N_topk (§IV-B), computed as one
 *     correctly rounded fp32 division of two exact integers;
 *   - query batches (fresh cluster members, exact copies, perturbed copies,
 *     in-batch duplicates).
 *
 * Every value is a pure function of (seed, indices) via a splitmix64 counter
 * hash, so a shard [row0, row0+nrows) of a store is bit-identical to the same
 * rows of the full store, and the host is the only place values are drawn.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* h(seed, stream, a, b): counter hash. */
static inline uint64_t hsh(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  uint64_t z = mix64(seed ^ (stream * 0xD1B54A32D192ED03ull));
  z = mix64(z ^ a);
  z = mix64(z ^ (b * 0x8CB92BA72F3D8DD7ull + 0x632BE59BD9B4E019ull));
  return z;
}

/* uniform in [0,1), 24 bits: exact in fp32 */
static inline double unif(uint64_t h) { return (double)(h >> 40) * (1.0 / 16777216.0); }

/* Irwin-Hall(4) gaussian approximation, unit variance */
static inline double gauss(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b) {
  double s = 0.0;
  for (uint64_t t = 0; t < 4; ++t) s += unif(hsh(seed, stream, a, b * 4u + t));
  return (s - 2.0) * 1.7320508075688772;
}

/* round-to-nearest-even double -> bf16 bits (via fp32, values are finite) */
static inline uint16_t to_bf16(double v) {
  float f = (float)v;
  uint32_t u;
  memcpy(&u, &f, 4);
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb;
  return (uint16_t)(u >> 16);
}

static inline double from_bf16(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

int64_t gen_num_clusters(int64_t n_total) {
  int64_t c = n_total / 1000;
  if (c < 16) c = 16;
  if (c > 16384) c = 16384;
  return c;
}

int64_t gen_cluster_of(uint64_t seed, int64_t n_total, int64_t row) {
  return (int64_t)(hsh(seed, 1, (uint64_t)row, 0) % (uint64_t)gen_num_clusters(n_total));
}

static double noise_scale(uint64_t seed, int64_t row) {
  return 0.25 + 1.25 * unif(hsh(seed, 5, (uint64_t)row, 0));
}

/* ---------------- threading helper ---------------- */
typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct { range_fn fn; void* ctx; int64_t lo, hi; } job_t;
static void* job_run(void* p) { job_t* j = (job_t*)p; j->fn(j->ctx, j->lo, j->hi); return NULL; }

static void parallel_for(int64_t n, int nthreads, range_fn fn, void* ctx) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (n < 4096 || nthreads == 1) { fn(ctx, 0, n); return; }
  pthread_t th[256];
  job_t jobs[256];
  int64_t per = (n + nthreads - 1) / nthreads;
  int used = 0;
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = (int64_t)t * per, hi = lo + per;
    if (lo >= n) break;
    if (hi > n) hi = n;
    jobs[t].fn = fn; jobs[t].ctx = ctx; jobs[t].lo = lo; jobs[t].hi = hi;
    pthread_create(&th[t], NULL, job_run, &jobs[t]);
    used++;
  }
  for (int t = 0; t < used; ++t) pthread_join(th[t], NULL);
}

/* ---------------- embeddings ---------------- */
typedef struct {
  uint64_t seed; int64_t n_total, row0; int dim; const float* centroids; uint16_t* out;
} emb_ctx;

static void emb_rows(void* p, int64_t lo, int64_t hi) {
  emb_ctx* c = (emb_ctx*)p;
  int64_t C = gen_num_clusters(c->n_total);
  for (int64_t r = lo; r < hi; ++r) {
    int64_t j = c->row0 + r;
    int64_t cl = (int64_t)(hsh(c->seed, 1, (uint64_t)j, 0) % (uint64_t)C);
    double eps = noise_scale(c->seed, j);
    const float* mu = c->centroids + cl * (int64_t)c->dim;
    uint16_t* o = c->out + r * (int64_t)c->dim;
    for (int d = 0; d < c->dim; ++d)
      o[d] = to_bf16((double)mu[d] + eps * gauss(c->seed, 3, (uint64_t)j, (uint64_t)d));
  }
}

typedef struct { uint64_t seed; int dim; float* cent; } cent_ctx;
static void cent_rows(void* p, int64_t lo, int64_t hi) {
  cent_ctx* c = (cent_ctx*)p;
  for (int64_t cl = lo; cl < hi; ++cl)
    for (int d = 0; d < c->dim; ++d)
      c->cent[cl * c->dim + d] = (float)gauss(c->seed, 2, (uint64_t)cl, (uint64_t)d);
}

static float* make_centroids(uint64_t seed, int64_t n_total, int dim, int nthreads) {
  int64_t C = gen_num_clusters(n_total);
  float* cent = (float*)malloc(sizeof(float) * (size_t)C * (size_t)dim);
  if (!cent) return NULL;
  cent_ctx cc = {seed, dim, cent};
  parallel_for(C, nthreads, cent_rows, &cc);
  return cent;
}

/* Rows [row0, row0+nrows) of the store of n_total prompts, bf16 bits, row-major. */
int gen_store_emb(uint64_t seed, int64_t n_total, int64_t row0, int64_t nrows, int dim,
                  uint16_t* out, int nthreads) {
  if (dim <= 0 || row0 < 0 || nrows < 0 || row0 + nrows > n_total) return 1;
  float* cent = make_centroids(seed, n_total, dim, nthreads);
  if (!cent) return 2;
  emb_ctx c = {seed, n_total, row0, dim, cent, out};
  parallel_for(nrows, nthreads, emb_rows, &c);
  free(cent);
  return 0;
}

/* ---------------- activation tables ---------------- */
typedef struct {
  uint64_t seed; int64_t n_total, row0; int L, E, topk;
  const int* rank_of;   /* [C][L][E]: Zipf rank of expert e for (cluster, layer) */
  const double* zipf;   /* [E] normalized Zipf weights by rank */
  float* out;
} act_ctx;

static void act_rows(void* p, int64_t lo, int64_t hi) {
  act_ctx* c = (act_ctx*)p;
  int64_t C = gen_num_clusters(c->n_total);
  int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)c->E);
  for (int64_t r = lo; r < hi; ++r) {
    int64_t j = c->row0 + r;
    int64_t cl = (int64_t)(hsh(c->seed, 1, (uint64_t)j, 0) % (uint64_t)C);
    int64_t n_in = 64 + (int64_t)(hsh(c->seed, 9, (uint64_t)j, 0) % 193u);
    double T = (double)(n_in * c->topk);
    for (int l = 0; l < c->L; ++l) {
      const int* rk = c->rank_of + ((int64_t)cl * c->L + l) * c->E;
      int64_t tot = 0;
      for (int e = 0; e < c->E; ++e) {
        double u = unif(hsh(c->seed, 6, (uint64_t)j, (uint64_t)(l * c->E + e)));
        cnt[e] = (int64_t)floor(T * c->zipf[rk[e]] * (0.5 + u));
        tot += cnt[e];
      }
      if (tot == 0) {
        for (int e = 0; e < c->E; ++e) if (rk[e] == 0) cnt[e] = 1;
        tot = 1;
      }
      float* o = c->out + (r * c->L + l) * (int64_t)c->E;
      for (int e = 0; e < c->E; ++e) o[e] = (float)cnt[e] / (float)tot;
    }
  }
  free(cnt);
}

/* Rows [row0, row0+nrows) of the activation table, fp32 [nrows][L][E]. */
int gen_store_act(uint64_t seed, int64_t n_total, int64_t row0, int64_t nrows, int L, int E,
                  int topk, float* out, int nthreads) {
  if (L <= 0 || E <= 0 || topk <= 0 || row0 < 0 || nrows < 0 || row0 + nrows > n_total) return 1;
  int64_t C = gen_num_clusters(n_total);
  int* rank_of = (int*)malloc(sizeof(int) * (size_t)C * (size_t)L * (size_t)E);
  double* zipf = (double*)malloc(sizeof(double) * (size_t)E);
  int* perm = (int*)malloc(sizeof(int) * (size_t)E);
  if (!rank_of || !zipf || !perm) { free(rank_of); free(zipf); free(perm); return 2; }
  double zs = 0.0;
  for (int r = 0; r < E; ++r) { zipf[r] = pow((double)(r + 1), -1.1); zs += zipf[r]; }
  for (int r = 0; r < E; ++r) zipf[r] /= zs;
  for (int64_t cl = 0; cl < C; ++cl) {
    for (int l = 0; l < L; ++l) {
      /* hashed Fisher-Yates: perm[r] = expert with Zipf rank r */
      for (int e = 0; e < E; ++e) perm[e] = e;
      for (int e = E - 1; e > 0; --e) {
        int s = (int)(hsh(seed, 7, (uint64_t)(cl * L + l), (uint64_t)e) % (uint64_t)(e + 1));
        int t = perm[e]; perm[e] = perm[s]; perm[s] = t;
      }
      int* rk = rank_of + (cl * L + l) * (int64_t)E;
      for (int r = 0; r < E; ++r) rk[perm[r]] = r;
    }
  }
  act_ctx c = {seed, n_total, row0, L, E, topk, rank_of, zipf, out};
  parallel_for(nrows, nthreads, act_rows, &c);
  free(rank_of); free(zipf); free(perm);
  return 0;
}

/* ---------------- queries ---------------- */
/*
 * mode 0 (throughput): every query is a fresh cluster member.
 * mode 1 (correctness mix, by i mod 8): 0-3 fresh members, 4-5 exact copies of a
 *   stored row, 6 a perturbed copy (delta = 0.05), 7 a duplicate of query i-1.
 * Copies regenerate the stored row from the store seed (pure function), so the
 * store itself is never read.
 */
typedef struct {
  uint64_t sseed, qseed; int64_t n_total; int dim, mode; const float* cent; uint16_t* out;
} q_ctx;

static void store_row(uint64_t sseed, int64_t n_total, int64_t j, int dim, const float* cent,
                      uint16_t* o) {
  int64_t C = gen_num_clusters(n_total);
  int64_t cl = (int64_t)(hsh(sseed, 1, (uint64_t)j, 0) % (uint64_t)C);
  double eps = noise_scale(sseed, j);
  const float* mu = cent + cl * (int64_t)dim;
  for (int d = 0; d < dim; ++d)
    o[d] = to_bf16((double)mu[d] + eps * gauss(sseed, 3, (uint64_t)j, (uint64_t)d));
}

static void q_rows(void* p, int64_t lo, int64_t hi) {
  q_ctx* c = (q_ctx*)p;
  int64_t C = gen_num_clusters(c->n_total);
  for (int64_t i = lo; i < hi; ++i) {
    uint16_t* o = c->out + i * (int64_t)c->dim;
    int kind = c->mode == 0 ? 0 : (int)(i % 8);
    if (kind <= 3) {
      int64_t cl = (int64_t)(hsh(c->qseed, 1, (uint64_t)i, 0) % (uint64_t)C);
      double eps = 0.25 + 1.25 * unif(hsh(c->qseed, 5, (uint64_t)i, 0));
      const float* mu = c->cent + cl * (int64_t)c->dim;
      for (int d = 0; d < c->dim; ++d)
        o[d] = to_bf16((double)mu[d] + eps * gauss(c->qseed, 4, (uint64_t)i, (uint64_t)d));
    } else if (kind <= 6) {
      int64_t j = (int64_t)(hsh(c->qseed, 7, (uint64_t)i, 0) % (uint64_t)c->n_total);
      store_row(c->sseed, c->n_total, j, c->dim, c->cent, o);
      if (kind == 6)
        for (int d = 0; d < c->dim; ++d)
          o[d] = to_bf16(from_bf16(o[d]) + 0.05 * gauss(c->qseed, 8, (uint64_t)i, (uint64_t)d));
    }
  }
}

int gen_queries(uint64_t store_seed, uint64_t query_seed, int64_t n_total, int dim, int64_t B,
                int mode, uint16_t* out, int nthreads) {
  if (dim <= 0 || B < 0 || n_total <= 0 || (mode != 0 && mode != 1)) return 1;
  float* cent = make_centroids(store_seed, n_total, dim, nthreads);
  if (!cent) return 2;
  q_ctx c = {store_seed, query_seed, n_total, dim, mode, cent, out};
  parallel_for(B, nthreads, q_rows, &c);
  if (mode == 1)  /* duplicates: query i (i%8==7) repeats query i-1 */
    for (int64_t i = 7; i < B; i += 8)
      memcpy(out + i * (int64_t)dim, out + (i - 1) * (int64_t)dim, sizeof(uint16_t) * (size_t)dim);
  free(cent);
  return 0;
}

/* Which stored row a copy-kind query (mode 1, i%8 in {4,5,6}) was copied from; -1 otherwise. */
int64_t gen_query_source_row(uint64_t query_seed, int64_t n_total, int64_t i, int mode) {
  if (mode != 1) return -1;
  int kind = (int)(i % 8);
  if (kind < 4 || kind > 6) return -1;
  return (int64_t)(hsh(query_seed, 7, (uint64_t)i, 0) % (uint64_t)n_total);
}
