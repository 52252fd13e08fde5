/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously correct CPU
 * definition of what the SPS hot path computes.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load this library.  It shares no source, header, table or helper with the CUDA
 * path (paper_2512_18674_b200/csrc), and neither side includes the other.
 *
 * Precision: fp64 throughout; bf16 inputs are widened exactly (bits << 16 -> fp32
 * -> fp64).  Plain scalar loops, no intrinsics, built -O2 without fast-math.
 *
 * Steps, each following one passage of PAPER.md (arXiv 2512.18674):
 *   1. widen            bf16 -> double
 *   2. norms            ||x|| = sqrt(sum_d x_d^2), d ascending       (Eq. 11 denominator)
 *   3. scores           s = (q.x) / (||q|| ||x|| + sigma)            (Eq. 11, reduced
 *                       to prompt vectors: V1^T C V2 = a.b with a = sum of normalized token rows,
 *                       see oracle/scs.py for the literal Gram-matrix form and SURVEY F1)
 *   4. select           order by (s desc, global id asc), first k    (BF top-alpha, PAPER.md:672;
 *                       "top-alpha semantically similar ones are returned")
 *   5. weights          w_r = softmax(s_r / T) over the k retrieved   (T=1 reading)
 *   6. prediction       P[l,e] = sum_r w_r * S~_{id_r}[l,e], r asc
 *   7. plan             per layer the n_cold lowest-utility experts   (u = (N_in +
 *                       N_out N_topk) s~ is a positive multiple of s~, so argmin over u equals argmin
 *                       over s~; ties -> lower expert index, SPEC S:429 reading)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- step 1: exact widening of one bf16 bit pattern ---- */
static double widen(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return (double)f;
}

void oracle_widen_bf16(const uint16_t* in, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = widen(in[i]);
}

/* ---- step 2: norm of one row, d ascending ---- */
static double norm_row(const double* x, int dim) {
  double s = 0.0;
  for (int d = 0; d < dim; ++d) s += x[d] * x[d];
  return sqrt(s);
}

/* ---- step 3: Eq. 11 score of one (query, row) pair ---- */
static double score_pair(const double* q, double qn, const double* x, double xn, int dim,
                         double sigma) {
  double dot = 0.0;
  for (int d = 0; d < dim; ++d) dot += q[d] * x[d];
  return dot / (qn * xn + sigma);
}

/* ---------------- scores over a whole store, threaded over rows ---------------- */
typedef struct {
  const double* q;      /* [B][dim] widened queries */
  const double* qn;     /* [B] */
  int64_t B;
  const void* x;        /* store rows, bf16 bits or doubles */
  int x_is_bf16;
  int dim;
  double sigma;
  double* out;          /* [B][N] */
  int64_t N;
  int64_t lo, hi;
} scores_job;

static void* scores_worker(void* p) {
  scores_job* j = (scores_job*)p;
  double* row = (double*)malloc(sizeof(double) * (size_t)j->dim);
  for (int64_t r = j->lo; r < j->hi; ++r) {
    const double* xr;
    if (j->x_is_bf16) {
      const uint16_t* xb = (const uint16_t*)j->x + r * (int64_t)j->dim;
      for (int d = 0; d < j->dim; ++d) row[d] = widen(xb[d]);
      xr = row;
    } else {
      xr = (const double*)j->x + r * (int64_t)j->dim;
    }
    double xn = norm_row(xr, j->dim);
    for (int64_t i = 0; i < j->B; ++i)
      j->out[i * j->N + r] = score_pair(j->q + i * (int64_t)j->dim, j->qn[i], xr, xn, j->dim, j->sigma);
  }
  free(row);
  return NULL;
}

static void all_scores(const double* q, const double* qn, int64_t B, const void* x, int x_is_bf16,
                       int64_t N, int dim, double sigma, double* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (N < 1024) nthreads = 1;
  pthread_t th[256];
  scores_job jobs[256];
  int64_t per = (N + nthreads - 1) / nthreads;
  int used = 0;
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = (int64_t)t * per, hi = lo + per;
    if (lo >= N) break;
    if (hi > N) hi = N;
    scores_job jb = {q, qn, B, x, x_is_bf16, dim, sigma, out, N, lo, hi};
    jobs[t] = jb;
    if (nthreads == 1) scores_worker(&jobs[t]);
    else pthread_create(&th[t], NULL, scores_worker, &jobs[t]);
    used++;
  }
  if (nthreads > 1)
    for (int t = 0; t < used; ++t) pthread_join(th[t], NULL);
}

/* ---- step 4: selection by full sort on (score desc, id asc) ---- */
typedef struct { double s; int64_t id; } cand_t;

static int cand_cmp(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->s > y->s) return -1;
  if (x->s < y->s) return 1;
  if (x->id < y->id) return -1;
  if (x->id > y->id) return 1;
  return 0;
}

/* s[N] scores of rows with global ids id_offset + j; writes the first k. */
int oracle_select(const double* s, int64_t N, int64_t k, int64_t id_offset, int64_t* ids,
                  double* top) {
  if (k < 1 || k > N) return 1;
  cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)N);
  if (!c) return 2;
  for (int64_t j = 0; j < N; ++j) { c[j].s = s[j]; c[j].id = id_offset + j; }
  qsort(c, (size_t)N, sizeof(cand_t), cand_cmp);
  for (int64_t r = 0; r < k; ++r) {
    ids[r] = c[r].id;
    top[r] = c[r].s == 0.0 ? 0.0 : c[r].s; /* canonical +0 */
  }
  free(c);
  return 0;
}

/* ---- step 5: softmax of the k retrieved scores, temperature T ---- */
int oracle_softmax(const double* s, int64_t k, double T, double* w) {
  if (k < 1 || !(T > 0.0)) return 1;
  double m = s[0];
  for (int64_t r = 1; r < k; ++r) if (s[r] > m) m = s[r];
  double z = 0.0;
  for (int64_t r = 0; r < k; ++r) { w[r] = exp((s[r] - m) / T); z += w[r]; }
  for (int64_t r = 0; r < k; ++r) w[r] /= z;
  return 0;
}

/* ---- step 6: P = sum_r w_r * S~_{id_r}, r ascending ---- */
int oracle_predict(const int64_t* ids, const double* w, int64_t k, const float* act,
                   int64_t id_offset, int64_t n_rows, int64_t LE, double* out) {
  for (int64_t e = 0; e < LE; ++e) out[e] = 0.0;
  for (int64_t r = 0; r < k; ++r) {
    int64_t j = ids[r] - id_offset;
    if (j < 0 || j >= n_rows) return 1;
    const float* a = act + j * LE;
    for (int64_t e = 0; e < LE; ++e) out[e] += w[r] * (double)a[e];
  }
  return 0;
}

/* ---- step 7: cold set per (query, layer): n_cold smallest by (value asc, index asc) ---- */
int oracle_plan(const double* pred, int64_t B, int L, int E, int n_cold, uint8_t* mask) {
  if (n_cold < 0 || n_cold > E || L < 1 || E < 1) return 1;
  int* order = (int*)malloc(sizeof(int) * (size_t)E);
  for (int64_t i = 0; i < B; ++i) {
    for (int l = 0; l < L; ++l) {
      const double* v = pred + (i * L + l) * (int64_t)E;
      uint8_t* m = mask + (i * L + l) * (int64_t)E;
      for (int e = 0; e < E; ++e) order[e] = e;
      /* insertion sort by (v asc, e asc): textbook, E <= 256 */
      for (int a = 1; a < E; ++a) {
        int t = order[a], b = a - 1;
        while (b >= 0 && (v[order[b]] > v[t] || (v[order[b]] == v[t] && order[b] > t))) {
          order[b + 1] = order[b];
          --b;
        }
        order[b + 1] = t;
      }
      for (int e = 0; e < E; ++e) m[e] = 0;
      for (int c = 0; c < n_cold; ++c) m[order[c]] = 1;
    }
  }
  free(order);
  return 0;
}

/* ---------------- whole path ---------------- */
static int sps_core(const double* q, int64_t B, const void* x, int x_is_bf16, int64_t N, int dim,
                    const float* act, int L, int E, double sigma, double T, int64_t k,
                    int64_t id_offset, int64_t* ids, double* scores, double* pred, int nthreads) {
  if (B < 0 || N < 1 || dim < 1 || k < 1 || k > N || !(sigma > 0.0) || !(T > 0.0)) return 1;
  if (B == 0) return 0;
  double* qn = (double*)malloc(sizeof(double) * (size_t)B);
  double* s = (double*)malloc(sizeof(double) * (size_t)B * (size_t)N);
  double* w = (double*)malloc(sizeof(double) * (size_t)k);
  if (!qn || !s || !w) { free(qn); free(s); free(w); return 2; }
  for (int64_t i = 0; i < B; ++i) qn[i] = norm_row(q + i * (int64_t)dim, dim);
  all_scores(q, qn, B, x, x_is_bf16, N, dim, sigma, s, nthreads);
  int rc = 0;
  int64_t LE = (int64_t)L * E;
  for (int64_t i = 0; i < B && rc == 0; ++i) {
    rc = oracle_select(s + i * N, N, k, id_offset, ids + i * k, scores + i * k);
    if (rc == 0 && pred) {
      rc = oracle_softmax(scores + i * k, k, T, w);
      if (rc == 0) rc = oracle_predict(ids + i * k, w, k, act, id_offset, N, LE, pred + i * LE);
    }
  }
  free(qn); free(s); free(w);
  return rc;
}

/* bf16 store and queries (the hot path's inputs). */
int oracle_sps_bf16(const uint16_t* q_bits, int64_t B, const uint16_t* x_bits, int64_t N, int dim,
                    const float* act, int L, int E, double sigma, double T, int64_t k,
                    int64_t id_offset, int64_t* ids, double* scores, double* pred, int nthreads) {
  double* q = (double*)malloc(sizeof(double) * (size_t)(B > 0 ? B : 1) * (size_t)dim);
  if (!q) return 2;
  oracle_widen_bf16(q_bits, B * (int64_t)dim, q);
  int rc = sps_core(q, B, x_bits, 1, N, dim, act, L, E, sigma, T, k, id_offset, ids, scores, pred,
                    nthreads);
  free(q);
  return rc;
}

/* fp64 store and queries (used to pin the Eq. 11 reduction with real-valued vectors). */
int oracle_sps_f64(const double* q, int64_t B, const double* x, int64_t N, int dim,
                   const float* act, int L, int E, double sigma, double T, int64_t k,
                   int64_t id_offset, int64_t* ids, double* scores, double* pred, int nthreads) {
  return sps_core(q, B, x, 0, N, dim, act, L, E, sigma, T, k, id_offset, ids, scores, pred,
                  nthreads);
}

/* All scores s[B][N] (step 3) for bf16 inputs. */
int oracle_scores_bf16(const uint16_t* q_bits, int64_t B, const uint16_t* x_bits, int64_t N,
                       int dim, double sigma, double* out, int nthreads) {
  if (B < 1 || N < 1 || dim < 1 || !(sigma > 0.0)) return 1;
  double* q = (double*)malloc(sizeof(double) * (size_t)B * (size_t)dim);
  double* qn = (double*)malloc(sizeof(double) * (size_t)B);
  if (!q || !qn) { free(q); free(qn); return 2; }
  oracle_widen_bf16(q_bits, B * (int64_t)dim, q);
  for (int64_t i = 0; i < B; ++i) qn[i] = norm_row(q + i * (int64_t)dim, dim);
  all_scores(q, qn, B, x_bits, 1, N, dim, sigma, out, nthreads);
  free(q); free(qn);
  return 0;
}

/* Scores of explicit (query, row) pairs: out[p] = s(q[qi[p]], x[rows[p]]). */
int oracle_pair_scores_bf16(const uint16_t* q_bits, const uint16_t* x_bits, int dim,
                            const int64_t* qi, const int64_t* rows, int64_t n_pairs, double sigma,
                            double* out) {
  double* a = (double*)malloc(sizeof(double) * (size_t)dim);
  double* b = (double*)malloc(sizeof(double) * (size_t)dim);
  if (!a || !b) { free(a); free(b); return 2; }
  for (int64_t p = 0; p < n_pairs; ++p) {
    oracle_widen_bf16(q_bits + qi[p] * (int64_t)dim, dim, a);
    oracle_widen_bf16(x_bits + rows[p] * (int64_t)dim, dim, b);
    out[p] = score_pair(a, norm_row(a, dim), b, norm_row(b, dim), dim, sigma);
  }
  free(a); free(b);
  return 0;
}

/* ---- NEXT-N4: Jensen-Shannon divergence, log base 2 ("JS Divergence of expert
 * activation distributions", P:675 the prediction-accuracy metric; base 2 so the maximum is
 * 1, SPEC S:247 reading), averaged over the L layer rows.  JS(p,q) = KL(p||m)/2 + KL(q||m)/2,
 * m = (p+q)/2, with 0 log 0 = 0. */
double oracle_js_divergence(const double* p, const double* q, int L, int E) {
  double total = 0.0;
  for (int l = 0; l < L; ++l) {
    double js = 0.0;
    for (int e = 0; e < E; ++e) {
      const double a = p[l * E + e], b = q[l * E + e], m = 0.5 * (a + b);
      if (a > 0.0) js += 0.5 * a * log2(a / m);
      if (b > 0.0) js += 0.5 * b * log2(b / m);
    }
    total += js;
  }
  return total / L;
}
