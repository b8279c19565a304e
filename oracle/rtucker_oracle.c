/* rtucker_oracle.c -- CPU restatement of the reference's sketched Tucker-ALS
 * path. TEST INFRASTRUCTURE ONLY (see rtucker_oracle.h): the parity checker,
 * never the measured or shipped path.
 *
 * Build: gcc -std=c99 -O2 -ffp-contract=off -fPIC -shared (oracle/Makefile).
 * -ffp-contract=off plus plain x86-64 SSE2 keeps every multiply and add
 * separately rounded, the same as the reference's g++ -O3 build, so outputs are
 * bit-identical (pinned in tests/test_oracle_pin.py).
 */
#include "rtucker_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* oracle_last_error(void) { return g_err; }

#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_NUMERICAL 3
#define ORC_NOMEM 4

#define CHECK(expr)            \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != ORC_OK) {       \
      status = rc_;            \
      goto done;               \
    }                          \
  } while (0)

static void* xcalloc(size_t n, size_t sz) {
  if (n == 0) n = 1;
  return calloc(n, sz);
}

/* ------------------------------------------------------------------------ */
/* SplitMix64 -- rng.hpp:12-62                                                */

#define SM_GAMMA 0x9e3779b97f4a7c15ULL

static uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t orc_next_u64(orc_rng* r) { /* rng.hpp:16-21 */
  r->state += SM_GAMMA;
  return sm_mix(r->state);
}

double orc_next_double(orc_rng* r) { /* rng.hpp:24-26: top 53 bits x 2^-53 */
  return (double)(orc_next_u64(r) >> 11) * 0x1.0p-53;
}

uint64_t orc_next_below(orc_rng* r, uint64_t bound) { /* rng.hpp:46-52 */
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t v = orc_next_u64(r);
    if (v >= threshold) return v % bound;
  }
}

uint64_t orc_split_seed(orc_rng* r) { /* rng.hpp:56 */
  return orc_next_u64(r) ^ 0x5851f42d4c957f2dULL;
}

uint64_t orc_splitmix_at(uint64_t seed, uint64_t k) {
  return sm_mix(seed + (k + 1) * SM_GAMMA);
}

void orc_splitmix_stream(uint64_t seed, uint64_t n, uint64_t* out) {
  orc_rng r = {seed};
  for (uint64_t i = 0; i < n; ++i) out[i] = orc_next_u64(&r);
}

/* ------------------------------------------------------------------------ */
/* Dense helpers -- dense_matrix.cpp                                          */

static int all_finite(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* t = a^T (dense_matrix.cpp:35-43) */
static void transpose(const double* a, size_t m, size_t n, double* t) {
  for (size_t i = 0; i < m; ++i)
    for (size_t j = 0; j < n; ++j) t[j * m + i] = a[i * n + j];
}

/* c = a b, i-k-j order, zero a_ik skipped (dense_matrix.cpp:45-62). c zeroed here. */
static void matmul(const double* a, size_t m, size_t k, const double* b, size_t n,
                   double* c) {
  memset(c, 0, m * n * sizeof(double));
  for (size_t i = 0; i < m; ++i) {
    for (size_t p = 0; p < k; ++p) {
      const double aik = a[i * k + p];
      if (aik == 0.0) continue;
      const double* brow = b + p * n;
      double* crow = c + i * n;
      for (size_t j = 0; j < n; ++j) crow[j] += aik * brow[j];
    }
  }
}

static double dotv(const double* x, const double* y, size_t n) { /* :132-136 */
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += x[i] * y[i];
  return s;
}

static double norm2sq(const double* x, size_t n) { /* :138-142 */
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += x[i] * x[i];
  return s;
}

/* g = a^T a (d x d), upper triangle then mirror, zero skipped (:91-109). */
static void gram(const double* a, size_t m, size_t n, double* g) {
  memset(g, 0, n * n * sizeof(double));
  for (size_t k = 0; k < m; ++k) {
    const double* row = a + k * n;
    for (size_t i = 0; i < n; ++i) {
      const double rki = row[i];
      if (rki == 0.0) continue;
      for (size_t j = i; j < n; ++j) g[i * n + j] += rki * row[j];
    }
  }
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < i; ++j) g[i * n + j] = g[j * n + i];
}

/* Explicit Kronecker product (:111-124). */
static void kron(const double* a, size_t ar, size_t ac, const double* b, size_t br,
                 size_t bc, double* k) {
  const size_t kc = ac * bc;
  for (size_t ia = 0; ia < ar; ++ia)
    for (size_t ja = 0; ja < ac; ++ja) {
      const double v = a[ia * ac + ja];
      for (size_t ib = 0; ib < br; ++ib)
        for (size_t jb = 0; jb < bc; ++jb)
          k[(ia * br + ib) * kc + ja * bc + jb] = v * b[ib * bc + jb];
    }
}

/* ------------------------------------------------------------------------ */
/* One-sided Jacobi SVD -- svd.cpp:21-129                                     */

typedef struct {
  size_t m, n, rank, kmax; /* kmax = n (tall: columns); rank <= kmax */
  double* u;               /* m x kmax, only first rank cols valid */
  double* s;               /* kmax */
  double* vt;              /* kmax x n */
} orc_svd;

static void svd_free(orc_svd* s) {
  free(s->u);
  free(s->s);
  free(s->vt);
  memset(s, 0, sizeof *s);
}

/* svd.cpp:21-67. w is m x n (m >= n), v is n x n. */
static int jacobi_orthogonalize(double* w, size_t m, size_t n, double* v, double frob_sq) {
  const double threshold = 1e-14 * frob_sq;
  const size_t big = m > n ? m : n;
  const double relative_tol = (double)(big > 16 ? big : 16) * DBL_EPSILON;
  for (int sweep = 0; sweep < 100; ++sweep) {
    int rotated = 0;
    for (size_t p = 0; p + 1 < n; ++p) {
      for (size_t q = p + 1; q < n; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (size_t i = 0; i < m; ++i) {
          const double wp = w[i * n + p], wq = w[i * n + q];
          alpha += wp * wp;
          beta += wq * wq;
          gamma += wp * wq;
        }
        if (fabs(gamma) <= threshold && fabs(gamma) <= relative_tol * sqrt(alpha * beta))
          continue;
        rotated = 1;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t);
        const double s = c * t;
        for (size_t i = 0; i < m; ++i) {
          const double wp = w[i * n + p], wq = w[i * n + q];
          w[i * n + p] = c * wp - s * wq;
          w[i * n + q] = s * wp + c * wq;
        }
        for (size_t i = 0; i < n; ++i) {
          const double vp = v[i * n + p], vq = v[i * n + q];
          v[i * n + p] = c * vp - s * vq;
          v[i * n + q] = s * vp + c * vq;
        }
      }
    }
    if (!rotated) return ORC_OK;
  }
  return fail(ORC_NUMERICAL, "compact_svd: Jacobi sweeps did not converge");
}

/* svd.cpp:69-111 */
static int svd_tall(const double* a, size_t m, size_t n, orc_svd* out) {
  int status = ORC_OK;
  double* w = malloc(m * n * sizeof(double));
  double* v = xcalloc(n * n, sizeof(double));
  double* norms = xcalloc(n, sizeof(double));
  size_t* order = xcalloc(n, sizeof(size_t));
  memset(out, 0, sizeof *out);
  if (!w || !v || !norms || !order) {
    status = fail(ORC_NOMEM, "out of memory");
    goto done;
  }
  memcpy(w, a, m * n * sizeof(double));
  for (size_t i = 0; i < n; ++i) v[i * n + i] = 1.0;
  double frob_sq = 0.0;
  for (size_t i = 0; i < m * n; ++i) frob_sq += a[i] * a[i];
  CHECK(jacobi_orthogonalize(w, m, n, v, frob_sq));
  for (size_t j = 0; j < n; ++j) {
    double s = 0.0;
    for (size_t i = 0; i < m; ++i) s += w[i * n + j] * w[i * n + j];
    norms[j] = sqrt(s);
  }
  /* stable sort of column indices by norm, descending (svd.cpp:81-83) */
  for (size_t j = 0; j < n; ++j) {
    size_t k = j;
    while (k > 0 && norms[order[k - 1]] < norms[j]) {
      order[k] = order[k - 1];
      --k;
    }
    order[k] = j;
  }
  const double sigma_max = n == 0 ? 0.0 : norms[order[0]];
  const double cutoff = (double)(m > n ? m : n) * DBL_EPSILON * sigma_max;
  size_t rank = 0;
  while (rank < n && norms[order[rank]] > cutoff && norms[order[rank]] > 0.0) ++rank;
  out->m = m;
  out->n = n;
  out->kmax = n;
  out->rank = rank;
  out->u = xcalloc(m * n, sizeof(double));
  out->s = xcalloc(n, sizeof(double));
  out->vt = xcalloc(n * n, sizeof(double));
  if (!out->u || !out->s || !out->vt) {
    status = fail(ORC_NOMEM, "out of memory");
    goto done;
  }
  for (size_t k = 0; k < rank; ++k) {
    const size_t j = order[k];
    const double sigma = norms[j];
    out->s[k] = sigma;
    for (size_t i = 0; i < m; ++i) out->u[i * n + k] = w[i * n + j] / sigma;
    for (size_t i = 0; i < n; ++i) out->vt[k * n + i] = v[i * n + j];
  }
done:
  free(w);
  free(v);
  free(norms);
  free(order);
  if (status != ORC_OK) svd_free(out);
  return status;
}

/* svd.cpp:115-129. Result: u is m x kmax, vt is kmax x n, kmax = min(m,n). */
static int compact_svd(const double* a, size_t m, size_t n, orc_svd* out) {
  if (m == 0 || n == 0) return fail(ORC_INVALID, "compact_svd: empty matrix");
  if (m >= n) return svd_tall(a, m, n, out);
  /* wide: factor the transpose and swap the bases */
  double* at = malloc(m * n * sizeof(double));
  if (!at) return fail(ORC_NOMEM, "out of memory");
  transpose(a, m, n, at);
  orc_svd t;
  int status = svd_tall(at, n, m, &t); /* t.u: n x m, t.vt: m x m */
  free(at);
  if (status != ORC_OK) return status;
  memset(out, 0, sizeof *out);
  out->m = m;
  out->n = n;
  out->kmax = m;
  out->rank = t.rank;
  out->s = t.s;
  out->u = xcalloc(m * m, sizeof(double));
  out->vt = xcalloc(m * n, sizeof(double));
  /* u = transpose(t.vt) restricted to rank columns; vt = transpose(t.u) */
  for (size_t k = 0; k < t.rank; ++k) {
    for (size_t i = 0; i < m; ++i) out->u[i * m + k] = t.vt[k * m + i];
    for (size_t i = 0; i < n; ++i) out->vt[k * n + i] = t.u[i * m + k];
  }
  free(t.u);
  free(t.vt);
  return ORC_OK;
}

#define SVD_U(sv, i, k) ((sv)->u[(i) * (sv)->kmax + (k)])
#define SVD_VT(sv, k, j) ((sv)->vt[(k) * (sv)->n + (j)])

int orc_compact_svd(const double* a, size_t m, size_t n, double* u_out, double* s_out,
                    double* vt_out, size_t* rank_out) {
  orc_svd sv;
  int status = compact_svd(a, m, n, &sv);
  if (status != ORC_OK) return status;
  const size_t kmax = sv.kmax;
  memcpy(u_out, sv.u, m * kmax * sizeof(double));
  memcpy(s_out, sv.s, kmax * sizeof(double));
  memcpy(vt_out, sv.vt, kmax * n * sizeof(double));
  *rank_out = sv.rank;
  svd_free(&sv);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Leverage scores and dense solves -- leverage.cpp, linalg.cpp               */

/* ridge_scores(svd, n, lambda), leverage.cpp:16-37 */
static void scores_from_svd(const orc_svd* sv, size_t n, double lambda, double* out) {
  double* weights = xcalloc(sv->rank, sizeof(double));
  for (size_t k = 0; k < sv->rank; ++k) {
    const double s2 = sv->s[k] * sv->s[k];
    weights[k] = s2 / (s2 + lambda);
  }
  for (size_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (size_t k = 0; k < sv->rank; ++k) {
      const double u = SVD_U(sv, i, k);
      s += weights[k] * u * u;
    }
    out[i] = s;
  }
  free(weights);
}

/* ridge_scores(A, lambda), leverage.cpp:39-52 */
int orc_ridge_scores(const double* a, size_t n, size_t d, double lambda, double* scores) {
  if (!all_finite(a, n * d)) return fail(ORC_INVALID, "DenseMatrix: non-finite entry");
  if (lambda < 0.0) return fail(ORC_INVALID, "ridge_scores: lambda must be non-negative");
  int all_zero = 1;
  for (size_t i = 0; i < n * d && all_zero; ++i)
    if (a[i] != 0.0) all_zero = 0;
  if (all_zero) {
    for (size_t i = 0; i < n; ++i) scores[i] = 0.0;
    return ORC_OK;
  }
  orc_svd sv;
  int status = compact_svd(a, n, d, &sv);
  if (status != ORC_OK) return status;
  scores_from_svd(&sv, n, lambda, scores);
  svd_free(&sv);
  return ORC_OK;
}

/* pseudoinverse, linalg.cpp:8-26: V diag(1/s) U^T as a sum of rank-1 terms. */
int orc_pseudoinverse(const double* a, size_t m, size_t n, double* pinv) {
  memset(pinv, 0, n * m * sizeof(double));
  if (m == 0 || n == 0) return ORC_OK;
  orc_svd sv;
  int status = compact_svd(a, m, n, &sv);
  if (status != ORC_OK) return status;
  for (size_t k = 0; k < sv.rank; ++k) {
    const double inv_sigma = 1.0 / sv.s[k];
    for (size_t i = 0; i < n; ++i) {
      const double vik = SVD_VT(&sv, k, i) * inv_sigma;
      if (vik == 0.0) continue;
      for (size_t j = 0; j < m; ++j) pinv[i * m + j] += vik * SVD_U(&sv, j, k);
    }
  }
  svd_free(&sv);
  return ORC_OK;
}

/* solve_ridge_exact, linalg.cpp:28-41 */
int orc_solve_ridge_exact(const double* a, size_t n, size_t d, const double* b,
                          double lambda, double* x) {
  int status = ORC_OK;
  if (!all_finite(a, n * d)) return fail(ORC_INVALID, "DenseMatrix: non-finite entry");
  if (lambda < 0.0) return fail(ORC_INVALID, "solve_ridge_exact: lambda must be non-negative");
  double* normal = xcalloc(d * d, sizeof(double));
  double* inv = xcalloc(d * d, sizeof(double));
  double* atb = xcalloc(d, sizeof(double));
  gram(a, n, d, normal);
  for (size_t i = 0; i < d; ++i) normal[i * d + i] += lambda;
  CHECK(orc_pseudoinverse(normal, d, d, inv));
  /* matvec_transposed (dense_matrix.cpp:79-89) */
  for (size_t i = 0; i < n; ++i) {
    const double xi = b[i];
    if (xi == 0.0) continue;
    for (size_t j = 0; j < d; ++j) atb[j] += xi * a[i * d + j];
  }
  for (size_t i = 0; i < d; ++i) x[i] = dotv(inv + i * d, atb, d); /* matvec */
done:
  free(normal);
  free(inv);
  free(atb);
  return status;
}

/* ------------------------------------------------------------------------ */
/* Sampling -- sketch_ridge.cpp:40-50, sampler.cpp:9-57                       */

int orc_sample_count(double beta_prime, size_t d, double epsilon, double delta,
                     uint64_t* out) {
  if (beta_prime <= 0.0 || epsilon <= 0.0 || epsilon >= 1.0 || delta <= 0.0 ||
      delta >= 1.0 || d == 0)
    return fail(ORC_INVALID, "sample_count: parameters out of range");
  const double dd = (double)d;
  const double log_term = 420.0 * log(4.0 * dd / delta);
  const double tail_term = 1.0 / (delta * epsilon);
  const double s = ceil(4.0 * dd / beta_prime * (log_term > tail_term ? log_term : tail_term));
  *out = (uint64_t)s;
  return ORC_OK;
}

/* upper_bound over an ascending array: first index with cdf[i] > u. */
static size_t upper_bound(const double* cdf, size_t n, double u) {
  size_t lo = 0, len = n;
  while (len > 0) {
    const size_t half = len / 2;
    if (!(u < cdf[lo + half])) {
      lo = lo + half + 1;
      len = len - half - 1;
    } else {
      len = half;
    }
  }
  return lo;
}

typedef struct { /* sampler.cpp:9-40 */
  size_t n, d;
  double* norm_scores;
  double* cumulative;
  double data_mass, aug_mass_per_row, total_mass;
} aug_sampler;

static int aug_sampler_init(aug_sampler* s, const double* cand, size_t n, size_t d,
                            double d_eff_lower) {
  memset(s, 0, sizeof *s);
  if (d == 0) return fail(ORC_INVALID, "AugmentedSampler: d must be positive");
  if (d_eff_lower < 0.0 || d_eff_lower > (double)d)
    return fail(ORC_INVALID, "AugmentedSampler: d_eff_lower outside [0, d]");
  double l1 = 0.0;
  for (size_t i = 0; i < n; ++i) {
    if (!(cand[i] >= 0.0) || !isfinite(cand[i]))
      return fail(ORC_INVALID, "AugmentedSampler: scores must be finite and non-negative");
    l1 += cand[i];
  }
  if (l1 <= 0.0) return fail(ORC_INVALID, "AugmentedSampler: scores must not all be zero");
  s->n = n;
  s->d = d;
  s->norm_scores = xcalloc(n, sizeof(double));
  s->cumulative = xcalloc(n, sizeof(double));
  const double scale = (double)d / l1;
  double running = 0.0;
  for (size_t i = 0; i < n; ++i) {
    s->norm_scores[i] = cand[i] * scale;
    running += s->norm_scores[i];
    s->cumulative[i] = running;
  }
  s->data_mass = running;
  const double m = (double)d - d_eff_lower;
  s->aug_mass_per_row = m < 1.0 ? m : 1.0;
  s->total_mass = s->data_mass + (double)d * s->aug_mass_per_row;
  return ORC_OK;
}

static void aug_sampler_draw(const aug_sampler* s, orc_rng* rng, uint64_t* idx_out,
                             double* prob_out) { /* sampler.cpp:42-57 */
  const double u = orc_next_double(rng) * s->total_mass;
  if (u < s->data_mass || s->aug_mass_per_row == 0.0) {
    size_t idx = upper_bound(s->cumulative, s->n, u < s->data_mass ? u : s->data_mass);
    if (idx >= s->n) idx = s->n - 1;
    while (idx > 0 && s->norm_scores[idx] == 0.0) --idx;
    *idx_out = idx;
    *prob_out = s->norm_scores[idx] / s->total_mass;
    return;
  }
  size_t k = (size_t)((u - s->data_mass) / s->aug_mass_per_row);
  if (k >= s->d) k = s->d - 1;
  *idx_out = s->n + k;
  *prob_out = s->aug_mass_per_row / s->total_mass;
}

static void aug_sampler_free(aug_sampler* s) {
  free(s->norm_scores);
  free(s->cumulative);
}

/* Streaming normal equations + pinv solve + sketched objective of
 * solve_sketched_ridge (sketch_ridge.cpp:105-149), for any row source given as
 * a callback copy_row(ctx, j < n, out). */
typedef void (*row_fn)(const void* ctx, uint64_t j, double* out);

static void augmented_row(row_fn fn, const void* ctx, uint64_t n, size_t d,
                          double root_lambda, uint64_t j, double* out) {
  if (j < n) { /* sketch_ridge.cpp:18-36 */
    fn(ctx, j, out);
    return;
  }
  for (size_t c = 0; c < d; ++c) out[c] = 0.0;
  out[j - n] = root_lambda;
}

static void normal_equations(row_fn fn, const void* ctx, uint64_t n, size_t d,
                             double lambda, uint64_t s, const uint64_t* idx,
                             const double* wts, const double* sampled_b, double* g,
                             double* rhs) {
  const double root_lambda = sqrt(lambda);
  double* row = xcalloc(d, sizeof(double));
  memset(g, 0, d * d * sizeof(double));
  memset(rhs, 0, d * sizeof(double));
  for (uint64_t t = 0; t < s; ++t) {
    const double w = wts[t];
    augmented_row(fn, ctx, n, d, root_lambda, idx[t], row);
    const double w2 = w * w;
    for (size_t p = 0; p < d; ++p) {
      const double v = w2 * row[p];
      if (v == 0.0) continue;
      double* grow = g + p * d;
      for (size_t q = p; q < d; ++q) grow[q] += v * row[q];
    }
    const double wb = w2 * sampled_b[t];
    if (wb != 0.0)
      for (size_t p = 0; p < d; ++p) rhs[p] += wb * row[p];
  }
  for (size_t p = 0; p < d; ++p)
    for (size_t q = 0; q < p; ++q) g[p * d + q] = g[q * d + p];
  free(row);
}

int orc_pinv_solve(const double* g, const double* rhs, size_t d, double* x,
                   size_t* rank_out) { /* sketch_ridge.cpp:130-139 */
  orc_svd sv;
  int status = compact_svd(g, d, d, &sv);
  if (status != ORC_OK) return status;
  for (size_t p = 0; p < d; ++p) x[p] = 0.0;
  for (size_t k = 0; k < sv.rank; ++k) {
    double uk_rhs = 0.0;
    for (size_t p = 0; p < d; ++p) uk_rhs += SVD_U(&sv, p, k) * rhs[p];
    const double coeff = uk_rhs / sv.s[k];
    for (size_t p = 0; p < d; ++p) x[p] += coeff * SVD_VT(&sv, k, p);
  }
  if (rank_out) *rank_out = sv.rank;
  svd_free(&sv);
  return ORC_OK;
}

typedef struct {
  const double* a;
  size_t d;
} matrix_rows;

static void matrix_row(const void* ctx, uint64_t j, double* out) {
  const matrix_rows* m = ctx;
  memcpy(out, m->a + j * m->d, m->d * sizeof(double));
}

/* rtucker_sketched_ridge (capi.cpp:324-362) -> approximate_ridge_regression
 * (sketch_ridge.cpp:153-164) -> solve_sketched_ridge with AugmentedSampler. */
int orc_sketched_ridge(const double* a, uint64_t n, uint64_t d, const double* b,
                       const double* candidate_scores, double lambda,
                       double d_eff_lower, double epsilon, double delta,
                       uint64_t sample_count_override, uint64_t seed, double* x_out,
                       uint64_t* sample_count_out, double* beta_prime_out) {
  int status = ORC_OK;
  double* cand = NULL;
  uint64_t* idx = NULL;
  double *wts = NULL, *sb = NULL, *g = NULL, *rhs = NULL;
  aug_sampler sam;
  memset(&sam, 0, sizeof sam);
  if (!a || !b || !x_out) return fail(ORC_INVALID, "null argument");
  if (!all_finite(a, n * d)) return fail(ORC_INVALID, "DenseMatrix: non-finite entry");
  cand = xcalloc(n, sizeof(double));
  if (candidate_scores)
    memcpy(cand, candidate_scores, n * sizeof(double));
  else
    CHECK(orc_ridge_scores(a, n, d, 0.0, cand)); /* classical_scores */
  CHECK(aug_sampler_init(&sam, cand, n, d, d_eff_lower));
  if (lambda < 0.0) {
    status = fail(ORC_INVALID, "solve_sketched_ridge: lambda must be non-negative");
    goto done;
  }
  const double beta_prime = 1.0 / (1.0 + sam.aug_mass_per_row);
  uint64_t s = sample_count_override;
  if (s == 0) CHECK(orc_sample_count(beta_prime, d, epsilon, delta, &s));
  idx = xcalloc(s, sizeof(uint64_t));
  wts = xcalloc(s, sizeof(double));
  sb = xcalloc(s, sizeof(double));
  g = xcalloc(d * d, sizeof(double));
  rhs = xcalloc(d, sizeof(double));
  if (!idx || !wts || !sb || !g || !rhs) {
    status = fail(ORC_NOMEM, "out of memory");
    goto done;
  }
  orc_rng rng = {seed};
  const double inv_s = 1.0 / (double)s;
  for (uint64_t t = 0; t < s; ++t) {
    double prob;
    aug_sampler_draw(&sam, &rng, &idx[t], &prob);
    wts[t] = sqrt(inv_s / prob);
  }
  for (uint64_t t = 0; t < s; ++t) sb[t] = idx[t] < n ? b[idx[t]] : 0.0;
  matrix_rows mr = {a, d};
  normal_equations(matrix_row, &mr, n, d, lambda, s, idx, wts, sb, g, rhs);
  CHECK(orc_pinv_solve(g, rhs, d, x_out, NULL));
  if (sample_count_out) *sample_count_out = s;
  if (beta_prime_out) *beta_prime_out = beta_prime;
done:
  free(cand);
  free(idx);
  free(wts);
  free(sb);
  free(g);
  free(rhs);
  aug_sampler_free(&sam);
  return status;
}

/* The dense toolkit's RowSketch alone: s draws of AugmentedSampler(cand, d, d_eff_lower)
 * from SplitMix64(seed), weights sqrt((1/s)/prob) (sampler.cpp:9-57,
 * sketch_ridge.cpp:80-90). */
int orc_aug_draw(const double* cand, uint64_t n, uint64_t d, double d_eff_lower, uint64_t seed,
                 uint64_t s, uint64_t* idx_out, double* w_out) {
  aug_sampler sam;
  int status = aug_sampler_init(&sam, cand, n, d, d_eff_lower);
  if (status != ORC_OK) return status;
  orc_rng rng = {seed};
  const double inv_s = 1.0 / (double)s;
  for (uint64_t t = 0; t < s; ++t) {
    double prob;
    aug_sampler_draw(&sam, &rng, &idx_out[t], &prob);
    w_out[t] = sqrt(inv_s / prob);
  }
  aug_sampler_free(&sam);
  return ORC_OK;
}

/* Sketched normal equations of [A; sqrt(lambda) I] (dense rows) from a given RowSketch
 * (sketch_ridge.cpp:105-128 with a MatrixRowSource): g (d x d, full), rhs (d). */
int orc_dense_normal_eq(const double* a, uint64_t n, uint64_t d, const double* b, double lambda,
                        uint64_t s, const uint64_t* idx, const double* w, double* g,
                        double* rhs) {
  double* sb = xcalloc(s ? s : 1, sizeof(double));
  if (!sb) return fail(ORC_NOMEM, "out of memory");
  for (uint64_t t = 0; t < s; ++t) sb[t] = idx[t] < n ? b[idx[t]] : 0.0;
  memset(g, 0, d * d * sizeof(double));
  memset(rhs, 0, d * sizeof(double));
  matrix_rows mr = {a, d};
  normal_equations(matrix_row, &mr, n, d, lambda, s, idx, w, sb, g, rhs);
  free(sb);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Kronecker design -- kronecker.cpp                                          */

/* ImplicitKronecker ctor, one factor (kronecker.cpp:9-35). */
int orc_factor_scores(const double* factor, size_t rows, size_t cols, double* scores,
                      double* cdf, double* sum_out, size_t* rank_out) {
  orc_svd sv;
  int status = compact_svd(factor, rows, cols, &sv);
  if (status != ORC_OK) return status;
  scores_from_svd(&sv, rows, 0.0, scores);
  double running = 0.0;
  for (size_t i = 0; i < rows; ++i) {
    running += scores[i];
    cdf[i] = running;
  }
  *sum_out = running;
  if (rank_out) *rank_out = sv.rank;
  svd_free(&sv);
  return ORC_OK;
}

/* ProductLeverageSampler::draw (kronecker.cpp:172-181) with sample_row_index
 * (kronecker.cpp:125-144) and linearize (kronecker.cpp:37-43). */
int orc_kron_draw(uint32_t order, const uint64_t* rows, uint64_t d,
                  const double* scores_cat, const double* cdf_cat, const double* sums,
                  uint64_t seed, uint64_t s, uint64_t* indices, double* weights,
                  uint64_t* u64_used_out) {
  uint64_t total_rows = 1;
  for (uint32_t n = 0; n < order; ++n) total_rows *= rows[n];
  const double aug_mass = (double)d - 0.0 < 1.0 ? (double)d : 1.0; /* min(1, d - 0) */
  const double p_data = 1.0 / (1.0 + aug_mass);
  orc_rng rng = {seed};
  const double inv_s = 1.0 / (double)s;
  for (uint64_t t = 0; t < s; ++t) {
    double prob;
    uint64_t index;
    if (orc_next_double(&rng) < p_data) {
      double probability = 1.0;
      uint64_t flat = 0;
      size_t off = 0;
      for (uint32_t n = 0; n < order; ++n) {
        if (sums[n] <= 0.0)
          return fail(ORC_INVALID, "ImplicitKronecker: cannot sample, factor has no nonzero rows");
        const double* cdf = cdf_cat + off;
        const double* sc = scores_cat + off;
        const double u = orc_next_double(&rng) * sums[n];
        size_t i = upper_bound(cdf, rows[n], u);
        if (i >= rows[n]) i = rows[n] - 1;
        while (i > 0 && sc[i] == 0.0) --i;
        flat = flat * rows[n] + i;
        probability *= sc[i] / sums[n];
        off += rows[n];
      }
      index = flat;
      prob = probability * p_data;
    } else {
      const uint64_t j = orc_next_below(&rng, d);
      index = total_rows + j;
      prob = (1.0 - p_data) / (double)d;
    }
    indices[t] = index;
    weights[t] = sqrt(inv_s / prob);
  }
  if (u64_used_out) {
    /* state advanced by one gamma per next_u64 call */
    *u64_used_out = (rng.state - seed) / SM_GAMMA;
  }
  return ORC_OK;
}

typedef struct {
  uint32_t order;
  const uint64_t* rows;
  const uint64_t* ranks;
  const double* const* factors;
} kron_rows;

/* KroneckerRowSource::copy_row: delinearize then the iterated outer product
 * growing left to right (kronecker.cpp:44-75, 154-157). */
static void kron_row(const void* ctx, uint64_t j, double* out) {
  const kron_rows* k = ctx;
  uint64_t idx[16] = {0};
  for (uint32_t n = k->order; n-- > 0;) {
    idx[n] = j % k->rows[n];
    j /= k->rows[n];
  }
  size_t width = k->ranks[0];
  const double* first = k->factors[0] + idx[0] * k->ranks[0];
  for (size_t c = 0; c < width; ++c) out[c] = first[c];
  for (uint32_t n = 1; n < k->order; ++n) {
    const double* next = k->factors[n] + idx[n] * k->ranks[n];
    const size_t nw = k->ranks[n];
    for (size_t c = width; c-- > 0;) {
      const double v = out[c];
      double* dst = out + c * nw;
      for (size_t q = 0; q < nw; ++q) dst[q] = v * next[q];
    }
    width *= nw;
  }
}

int orc_kron_sketch_normal_eq(uint32_t order, const uint64_t* rows,
                              const uint64_t* ranks, const double* factors_cat,
                              const double* xvec, double lambda, uint64_t s,
                              const uint64_t* indices, const double* weights,
                              double* g, double* rhs) {
  const double* fptr[16];
  uint64_t n_rows = 1, d = 1;
  size_t off = 0;
  for (uint32_t n = 0; n < order; ++n) {
    fptr[n] = factors_cat + off;
    off += rows[n] * ranks[n];
    n_rows *= rows[n];
    d *= ranks[n];
  }
  kron_rows kr = {order, rows, ranks, fptr};
  double* sb = xcalloc(s, sizeof(double));
  for (uint64_t t = 0; t < s; ++t) sb[t] = indices[t] < n_rows ? xvec[indices[t]] : 0.0;
  normal_equations(kron_row, &kr, n_rows, d, lambda, s, indices, weights, sb, g, rhs);
  free(sb);
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Tensors -- tensor.cpp:44-127                                                */

static uint64_t volume(uint32_t order, const uint64_t* shape) {
  uint64_t v = 1;
  for (uint32_t n = 0; n < order; ++n) v *= shape[n];
  return v;
}

/* unfold (tensor.cpp:52-79), mode 1-based. m: I_n x (size / I_n). */
static void unfold(const double* t, uint32_t order, const uint64_t* shape, uint32_t mode,
                   double* m) {
  const size_t axis = mode - 1;
  const size_t rows = shape[axis];
  const size_t size = volume(order, shape);
  const size_t cols = size / rows;
  size_t inner = 1;
  for (size_t n = axis + 1; n < order; ++n) inner *= shape[n];
  const size_t outer_count = size / (rows * inner);
  for (size_t outer = 0; outer < outer_count; ++outer)
    for (size_t i = 0; i < rows; ++i) {
      const double* block = t + (outer * rows + i) * inner;
      double* dst = m + i * cols + outer * inner;
      for (size_t k = 0; k < inner; ++k) dst[k] = block[k];
    }
}

/* fold (tensor.cpp:81-105) */
static void fold(const double* m, uint32_t mode, uint32_t order, const uint64_t* shape,
                 double* t) {
  const size_t axis = mode - 1;
  const size_t rows = shape[axis];
  const size_t size = volume(order, shape);
  const size_t cols = size / rows;
  size_t inner = 1;
  for (size_t n = axis + 1; n < order; ++n) inner *= shape[n];
  const size_t outer_count = size / (rows * inner);
  for (size_t outer = 0; outer < outer_count; ++outer)
    for (size_t i = 0; i < rows; ++i) {
      const double* src = m + i * cols + outer * inner;
      double* block = t + (outer * rows + i) * inner;
      for (size_t k = 0; k < inner; ++k) block[k] = src[k];
    }
}

/* mode_n_product (tensor.cpp:107-119): t (shape) x_mode mat (mr x I_mode).
 * shape is updated in place to the result shape; returns a new buffer. */
static double* mode_n_product(const double* t, uint32_t order, uint64_t* shape,
                              const double* mat, size_t mr, uint32_t mode) {
  const size_t axis = mode - 1;
  const size_t rows = shape[axis];
  const size_t cols = volume(order, shape) / rows;
  double* unf = malloc(rows * cols * sizeof(double));
  double* prod = malloc(mr * cols * sizeof(double));
  unfold(t, order, shape, mode, unf);
  matmul(mat, mr, rows, unf, cols, prod);
  shape[axis] = mr;
  double* out = malloc(mr * cols * sizeof(double));
  fold(prod, mode, order, shape, out);
  free(unf);
  free(prod);
  return out;
}

/* ------------------------------------------------------------------------ */
/* Tucker -- tucker.cpp                                                        */

static int check_model(uint32_t order, const uint64_t* shape, const uint64_t* ranks) {
  if (order == 0 || order > 8) return fail(ORC_INVALID, "DenseTensor: order must be in [1, 8]");
  for (uint32_t n = 0; n < order; ++n)
    if (shape[n] == 0) return fail(ORC_INVALID, "DenseTensor: zero-length dimension");
  for (uint32_t n = 0; n < order; ++n)
    if (ranks[n] == 0 || ranks[n] > shape[n])
      return fail(ORC_INVALID, "random_model: rank outside [1, I_n]");
  return ORC_OK;
}

static void factor_ptrs(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                        const double* cat, const double** ptrs) {
  size_t off = 0;
  for (uint32_t n = 0; n < order; ++n) {
    ptrs[n] = cat + off;
    off += shape[n] * ranks[n];
  }
}

/* reconstruct (tucker.cpp:47-53) */
int orc_reconstruct(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                    const double* core, const double* factors_cat, double* xhat) {
  const double* f[16];
  factor_ptrs(order, shape, ranks, factors_cat, f);
  uint64_t cur[16];
  for (uint32_t n = 0; n < order; ++n) cur[n] = ranks[n];
  double* out = malloc(volume(order, cur) * sizeof(double));
  memcpy(out, core, volume(order, cur) * sizeof(double));
  for (uint32_t n = 0; n < order; ++n) {
    double* next = mode_n_product(out, order, cur, f[n], shape[n], n + 1);
    free(out);
    out = next;
  }
  memcpy(xhat, out, volume(order, shape) * sizeof(double));
  free(out);
  return ORC_OK;
}

/* regularizer ||G||^2 + sum ||A_n||^2 accumulated as in tucker.cpp:222-226 */
static double model_reg(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                        const double* core, const double* factors_cat) {
  const double* f[16];
  factor_ptrs(order, shape, ranks, factors_cat, f);
  double reg = norm2sq(core, volume(order, ranks));
  for (uint32_t n = 0; n < order; ++n) reg += norm2sq(f[n], shape[n] * ranks[n]);
  return reg;
}

/* evaluate() of als (tucker.cpp:216-229); tucker_loss is the same sum. */
int orc_tucker_loss(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                    const double* core, const double* factors_cat, double lambda,
                    const double* x, double* loss_out, double* rmse_out) {
  const uint64_t size = volume(order, shape);
  double* xhat = malloc(size * sizeof(double));
  orc_reconstruct(order, shape, ranks, core, factors_cat, xhat);
  double residual = 0.0;
  for (uint64_t i = 0; i < size; ++i) {
    const double r = x[i] - xhat[i];
    residual += r * r;
  }
  free(xhat);
  const double reg = model_reg(order, shape, ranks, core, factors_cat);
  if (loss_out) *loss_out = residual + lambda * reg;
  if (rmse_out) *rmse_out = sqrt(residual / (double)size);
  return ORC_OK;
}

/* update_factor (tucker.cpp:70-89) with kron_excluding (tucker.cpp:31-43). */
int orc_update_factor(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                      const double* core, double* factors_cat, double lambda,
                      const double* x, uint32_t mode) {
  int status = ORC_OK;
  if (mode < 1 || mode > order) return fail(ORC_INVALID, "update_factor: mode out of range");
  const double* f[16];
  factor_ptrs(order, shape, ranks, factors_cat, f);
  const size_t axis = mode - 1;
  const size_t rn = ranks[axis], in = shape[axis];
  size_t j_rows = 1, j_cols = 1; /* others: J x prod R_other */
  for (uint32_t n = 0; n < order; ++n)
    if (n != axis) {
      j_rows *= shape[n];
      j_cols *= ranks[n];
    }
  double* g_unf = malloc(rn * j_cols * sizeof(double));
  double* others = NULL;
  double *othersT = NULL, *k = NULL, *kt = NULL, *b = NULL, *gk = NULL, *inv = NULL;
  double *bkt = NULL, *res = NULL;
  unfold(core, order, ranks, mode, g_unf);
  /* kron_excluding: increasing mode order */
  {
    size_t r = 1, c = 1;
    int first = 1;
    for (uint32_t n = 0; n < order; ++n) {
      if (n == axis) continue;
      if (first) {
        others = malloc(shape[n] * ranks[n] * sizeof(double));
        memcpy(others, f[n], shape[n] * ranks[n] * sizeof(double));
        r = shape[n];
        c = ranks[n];
        first = 0;
      } else {
        double* nk = malloc(r * shape[n] * c * ranks[n] * sizeof(double));
        kron(others, r, c, f[n], shape[n], ranks[n], nk);
        free(others);
        others = nk;
        r *= shape[n];
        c *= ranks[n];
      }
    }
    if (first) { /* identity(1) */
      others = malloc(sizeof(double));
      others[0] = 1.0;
    }
  }
  othersT = malloc(j_rows * j_cols * sizeof(double));
  transpose(others, j_rows, j_cols, othersT);
  k = malloc(rn * j_rows * sizeof(double));
  matmul(g_unf, rn, j_cols, othersT, j_rows, k); /* R_n x J */
  b = malloc(in * j_rows * sizeof(double));
  unfold(x, order, shape, mode, b);
  kt = malloc(j_rows * rn * sizeof(double));
  transpose(k, rn, j_rows, kt);
  gk = malloc(rn * rn * sizeof(double));
  gram(kt, j_rows, rn, gk);
  for (size_t i = 0; i < rn; ++i) gk[i * rn + i] += lambda;
  inv = malloc(rn * rn * sizeof(double));
  CHECK(orc_pseudoinverse(gk, rn, rn, inv));
  bkt = malloc(in * rn * sizeof(double));
  matmul(b, in, j_rows, kt, rn, bkt);
  res = malloc(in * rn * sizeof(double));
  matmul(bkt, in, rn, inv, rn, res);
  memcpy((double*)f[axis], res, in * rn * sizeof(double));
done:
  free(g_unf);
  free(others);
  free(othersT);
  free(k);
  free(kt);
  free(b);
  free(gk);
  free(inv);
  free(bkt);
  free(res);
  return status;
}

/* Sketched factor update (perf mode). NOT in the reference:
 * composed from its public pieces as SURVEY 8(c) prescribes, so parity is unpinned
 * by reference tests. The mode-n subproblem min ||K a_i - x_i||^2 + lambda ||a_i||^2
 * (K = (kron_{m!=n} A_m) G_(n)^T, rows indexed like the columns of X_(n): other modes
 * ascending, last fastest; tucker.cpp:31-43,70-89) is solved once per fiber row i with
 * solve_sketched_ridge semantics (sketch_ridge.cpp:52-151) and ONE shared sketch:
 *   draws: ProductLeverageSampler over the other factors' classical scores with the
 *          sqrt(lambda) augmentation over R_n (kronecker.cpp:159-181), s draws from
 *          SplitMix64(seed) -> orc_kron_draw(order - 1, others, d = R_n);
 *   row t: data -> G_(n) z, z = kron_row of the other factors' rows; aug -> sqrt(lambda) e_j;
 *   G = sum w^2 row row^T (upper triangle, mirrored), rhs_i = sum w^2 X_(n)[i, j_t] row;
 *   a_i = pinv(G) rhs_i (sketch_ridge.cpp:130-139).
 * A factor with no nonzero rows among the others cannot be sampled (kronecker.cpp:128-131). */
int orc_update_factor_sketched(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                               const double* core, double* factors_cat, double lambda,
                               const double* x, uint32_t mode, uint64_t s, uint64_t seed,
                               uint64_t* indices_out, double* weights_out) {
  int status = ORC_OK;
  if (mode < 1 || mode > order) return fail(ORC_INVALID, "update_factor: mode out of range");
  if (order < 2) return fail(ORC_INVALID, "sketched factor update needs order >= 2");
  if (s == 0) return fail(ORC_INVALID, "solve_sketched_ridge: sample count must be positive");
  if (lambda < 0.0) return fail(ORC_INVALID, "solve_sketched_ridge: lambda must be non-negative");
  const double* f[16];
  factor_ptrs(order, shape, ranks, factors_cat, f);
  const size_t axis = mode - 1;
  const size_t rn = ranks[axis], in = shape[axis];
  uint64_t orows[16], oranks[16];
  const double* ofac[16];
  uint32_t no = 0;
  uint64_t total_o = 1, width = 1, sum_rows = 0;
  for (uint32_t n = 0; n < order; ++n) {
    if (n == axis) continue;
    orows[no] = shape[n];
    oranks[no] = ranks[n];
    ofac[no] = f[n];
    total_o *= shape[n];
    width *= ranks[n];
    sum_rows += shape[n];
    ++no;
  }
  double* g_unf = malloc(rn * width * sizeof(double));
  unfold(core, order, ranks, mode, g_unf); /* R_n x width, others ascending */
  double* xu = malloc(in * total_o * sizeof(double));
  unfold(x, order, shape, mode, xu); /* I_n x prod_{m!=n} I_m */
  double* scores = xcalloc(sum_rows, sizeof(double));
  double* cdfs = xcalloc(sum_rows, sizeof(double));
  uint64_t* idx = xcalloc(s, sizeof(uint64_t));
  double* wts = xcalloc(s, sizeof(double));
  double* z = xcalloc(width, sizeof(double));
  double* row = xcalloc(rn, sizeof(double));
  double* g = xcalloc(rn * rn, sizeof(double));
  double* rhs = xcalloc(in * rn, sizeof(double));
  double* sol = xcalloc(rn, sizeof(double));
  double sums[16];
  size_t off = 0;
  for (uint32_t m = 0; m < no; ++m) {
    CHECK(orc_factor_scores(ofac[m], orows[m], oranks[m], scores + off, cdfs + off, &sums[m],
                            NULL));
    off += orows[m];
  }
  CHECK(orc_kron_draw(no, orows, rn, scores, cdfs, sums, seed, s, idx, wts, NULL));
  {
    kron_rows kr = {no, orows, oranks, ofac};
    const double root_lambda = sqrt(lambda);
    for (uint64_t t = 0; t < s; ++t) {
      const double w2 = wts[t] * wts[t];
      if (idx[t] < total_o) {
        kron_row(&kr, idx[t], z);
        for (size_t r = 0; r < rn; ++r) row[r] = dotv(g_unf + r * width, z, width);
      } else {
        for (size_t r = 0; r < rn; ++r) row[r] = 0.0;
        row[idx[t] - total_o] = root_lambda;
      }
      for (size_t p = 0; p < rn; ++p) {
        const double v = w2 * row[p];
        if (v == 0.0) continue;
        for (size_t q = p; q < rn; ++q) g[p * rn + q] += v * row[q];
      }
      if (idx[t] < total_o)
        for (size_t i = 0; i < in; ++i) {
          const double wb = w2 * xu[i * total_o + idx[t]];
          if (wb == 0.0) continue;
          for (size_t p = 0; p < rn; ++p) rhs[i * rn + p] += wb * row[p];
        }
    }
    for (size_t p = 0; p < rn; ++p)
      for (size_t q = 0; q < p; ++q) g[p * rn + q] = g[q * rn + p];
  }
  for (size_t i = 0; i < in; ++i) {
    CHECK(orc_pinv_solve(g, rhs + i * rn, rn, sol, NULL));
    memcpy((double*)f[axis] + i * rn, sol, rn * sizeof(double));
  }
  if (indices_out) memcpy(indices_out, idx, s * sizeof(uint64_t));
  if (weights_out) memcpy(weights_out, wts, s * sizeof(double));
done:
  free(g_unf);
  free(xu);
  free(scores);
  free(cdfs);
  free(idx);
  free(wts);
  free(z);
  free(row);
  free(g);
  free(rhs);
  free(sol);
  return status;
}

/* update_core_exact (tucker.cpp:91-129) */
int orc_update_core_exact(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                          const double* core, const double* factors_cat, double lambda,
                          const double* x, double* core_out) {
  (void)core;
  int status = ORC_OK;
  const double* f[16];
  factor_ptrs(order, shape, ranks, factors_cat, f);
  orc_svd svds[16];
  memset(svds, 0, sizeof svds);
  double* w = NULL;
  uint32_t done_svd = 0;
  for (uint32_t n = 0; n < order; ++n) {
    CHECK(compact_svd(f[n], shape[n], ranks[n], &svds[n]));
    done_svd = n + 1;
  }
  for (uint32_t n = 0; n < order; ++n)
    if (svds[n].rank == 0) {
      memset(core_out, 0, volume(order, ranks) * sizeof(double));
      goto done;
    }
  uint64_t cur[16];
  for (uint32_t n = 0; n < order; ++n) cur[n] = shape[n];
  w = malloc(volume(order, shape) * sizeof(double));
  memcpy(w, x, volume(order, shape) * sizeof(double));
  for (uint32_t n = 0; n < order; ++n) {
    /* transpose(U): rank x I_n */
    const orc_svd* sv = &svds[n];
    double* ut = malloc(sv->rank * shape[n] * sizeof(double));
    for (size_t k = 0; k < sv->rank; ++k)
      for (size_t i = 0; i < shape[n]; ++i) ut[k * shape[n] + i] = SVD_U(sv, i, k);
    double* nw = mode_n_product(w, order, cur, ut, sv->rank, n + 1);
    free(ut);
    free(w);
    w = nw;
  }
  {
    uint64_t t[16] = {0};
    const uint64_t size = volume(order, cur);
    for (uint64_t flat = 0; flat < size; ++flat) {
      double sigma = 1.0;
      for (uint32_t n = 0; n < order; ++n) sigma *= svds[n].s[t[n]];
      w[flat] *= sigma / (sigma * sigma + lambda);
      for (uint32_t n = order; n-- > 0;) {
        if (++t[n] < cur[n]) break;
        t[n] = 0;
      }
    }
  }
  for (uint32_t n = 0; n < order; ++n) {
    /* transpose(vt): R_n x rank */
    const orc_svd* sv = &svds[n];
    double* v = malloc(ranks[n] * sv->rank * sizeof(double));
    for (size_t k = 0; k < sv->rank; ++k)
      for (size_t i = 0; i < ranks[n]; ++i) v[i * sv->rank + k] = SVD_VT(sv, k, i);
    double* nw = mode_n_product(w, order, cur, v, ranks[n], n + 1);
    free(v);
    free(w);
    w = nw;
  }
  if (!all_finite(w, volume(order, ranks))) {
    status = fail(ORC_INVALID, "DenseTensor: non-finite entry");
    goto done;
  }
  memcpy(core_out, w, volume(order, ranks) * sizeof(double));
done:
  for (uint32_t n = 0; n < done_svd; ++n) svd_free(&svds[n]);
  free(w);
  return status;
}

/* update_core_fast (tucker.cpp:141-166) -> solve_sketched_ridge
 * (sketch_ridge.cpp:52-151) over the implicit Kronecker design. */
int orc_update_core_fast(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                         const double* core, const double* factors_cat, double lambda,
                         const double* x, uint64_t s_override, double epsilon,
                         double delta, uint64_t seed, double* core_out,
                         uint64_t* indices_out, double* weights_out,
                         int* rank_deficient_out, uint64_t* s_out) {
  (void)core;
  int status = ORC_OK;
  const double* f[16];
  factor_ptrs(order, shape, ranks, factors_cat, f);
  uint64_t total_rows = volume(order, shape);
  uint64_t d = volume(order, ranks);
  double *scores = NULL, *cdfs = NULL, *wts = NULL, *g = NULL, *rhs = NULL;
  uint64_t* idx = NULL;
  double sums[16];
  size_t off = 0, sum_rows = 0;
  for (uint32_t n = 0; n < order; ++n) sum_rows += shape[n];
  scores = xcalloc(sum_rows, sizeof(double));
  cdfs = xcalloc(sum_rows, sizeof(double));
  size_t franks[16];
  for (uint32_t n = 0; n < order; ++n) { /* ImplicitKronecker ctor: all factors first */
    CHECK(orc_factor_scores(f[n], shape[n], ranks[n], scores + off, cdfs + off, &sums[n],
                            &franks[n]));
    off += shape[n];
  }
  for (uint32_t n = 0; n < order; ++n) {
    if (franks[n] == 0) { /* tucker.cpp:148-154: zero factor -> zero core */
      memset(core_out, 0, d * sizeof(double));
      if (s_out) *s_out = 0;
      if (rank_deficient_out) *rank_deficient_out = 0;
      goto done;
    }
  }
  if (lambda < 0.0) {
    status = fail(ORC_INVALID, "solve_sketched_ridge: lambda must be non-negative");
    goto done;
  }
  const double beta_prime = 1.0 / (1.0 + 1.0); /* aug mass min(1, d) = 1 */
  uint64_t s = s_override;
  if (s == 0) CHECK(orc_sample_count(beta_prime, d, epsilon, delta, &s));
  idx = xcalloc(s, sizeof(uint64_t));
  wts = xcalloc(s, sizeof(double));
  g = xcalloc(d * d, sizeof(double));
  rhs = xcalloc(d, sizeof(double));
  if (!idx || !wts || !g || !rhs) {
    status = fail(ORC_NOMEM, "out of memory");
    goto done;
  }
  CHECK(orc_kron_draw(order, shape, d, scores, cdfs, sums, seed, s, idx, wts, NULL));
  CHECK(orc_kron_sketch_normal_eq(order, shape, ranks, factors_cat, x, lambda, s, idx, wts,
                                  g, rhs));
  size_t rank;
  CHECK(orc_pinv_solve(g, rhs, d, core_out, &rank));
  if (!all_finite(core_out, d)) {
    status = fail(ORC_INVALID, "DenseTensor: non-finite entry");
    goto done;
  }
  if (rank_deficient_out) *rank_deficient_out = rank < d;
  if (indices_out) memcpy(indices_out, idx, s * sizeof(uint64_t));
  if (weights_out) memcpy(weights_out, wts, s * sizeof(double));
  if (s_out) *s_out = s;
  (void)total_rows;
done:
  free(scores);
  free(cdfs);
  free(idx);
  free(wts);
  free(g);
  free(rhs);
  return status;
}

/* random_model (tucker.cpp:168-190) */
int orc_random_model(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                     uint64_t seed, double* core, double* factors_cat) {
  orc_rng rng = {seed};
  const uint64_t csize = volume(order, ranks);
  for (uint64_t i = 0; i < csize; ++i) core[i] = orc_next_double(&rng);
  size_t off = 0;
  for (uint32_t n = 0; n < order; ++n) {
    if (ranks[n] == 0 || ranks[n] > shape[n])
      return fail(ORC_INVALID, "random_model: rank outside [1, I_n]");
    for (uint64_t i = 0; i < shape[n] * ranks[n]; ++i)
      factors_cat[off + i] = orc_next_double(&rng);
    off += shape[n] * ranks[n];
  }
  return ORC_OK;
}

/* als (tucker.cpp:192-276) */
int orc_als(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
            const double* x, const orc_als_options* o, double* core,
            double* factors_cat, uint32_t* history_iter, int* history_step,
            double* history_loss, double* history_rmse, uint64_t* history_len_out,
            uint32_t* iterations_out, double* final_loss, double* final_rmse,
            uint64_t* core_seeds_out) {
  return orc_als_fs(order, shape, ranks, x, o, 0, core, factors_cat, history_iter, history_step,
                    history_loss, history_rmse, history_len_out, iterations_out, final_loss,
                    final_rmse, core_seeds_out);
}

/* orc_als with sketched factor updates when factor_samples > 0 (perf mode). Factor
 * sketch seeds: a second split of the seed generator (the first seeds the core
 * sketches, tucker.cpp:206), one next_u64 per (sweep, mode) in update order. */
int orc_als_fs(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
               const double* x, const orc_als_options* o, uint64_t factor_samples,
               double* core, double* factors_cat, uint32_t* history_iter, int* history_step,
               double* history_loss, double* history_rmse, uint64_t* history_len_out,
               uint32_t* iterations_out, double* final_loss, double* final_rmse,
               uint64_t* core_seeds_out) {
  int status = ORC_OK;
  double* new_core = NULL;
  if (o->max_iterations == 0) return fail(ORC_INVALID, "als: max_iterations must be >= 1");
  if (order == 0 || order > 8) return fail(ORC_INVALID, "DenseTensor: order must be in [1, 8]");
  CHECK(check_model(order, shape, ranks));
  if (!all_finite(x, volume(order, shape))) return fail(ORC_INVALID, "DenseTensor: non-finite entry");
  CHECK(orc_random_model(order, shape, ranks, o->seed, core, factors_cat));
  orc_rng seed_rng0 = {o->seed};
  orc_rng sketch_seed_rng = {orc_split_seed(&seed_rng0)};
  orc_rng factor_seed_rng = {orc_split_seed(&seed_rng0)};
  const double lambda = o->lambda;
  uint64_t hl = 0;
  double previous_loss, unused;
  orc_tucker_loss(order, shape, ranks, core, factors_cat, lambda, x, &previous_loss, &unused);
  const uint64_t csize = volume(order, ranks);
  new_core = xcalloc(csize, sizeof(double));
  uint32_t iter;
  for (iter = 1; iter <= o->max_iterations; ++iter) {
    for (uint32_t n = 0; n < order; ++n) {
      if (factor_samples > 0 && order >= 2) {
        const uint64_t fs = orc_next_u64(&factor_seed_rng);
        CHECK(orc_update_factor_sketched(order, shape, ranks, core, factors_cat, lambda, x,
                                         n + 1, factor_samples, fs, NULL, NULL));
      } else {
        CHECK(orc_update_factor(order, shape, ranks, core, factors_cat, lambda, x, n + 1));
      }
      if (o->record_history) {
        history_iter[hl] = iter;
        history_step[hl] = (int)n;
        orc_tucker_loss(order, shape, ranks, core, factors_cat, lambda, x,
                        &history_loss[hl], &history_rmse[hl]);
        ++hl;
      }
    }
    if (o->sketched_core == 0) {
      CHECK(orc_update_core_exact(order, shape, ranks, core, factors_cat, lambda, x,
                                  new_core));
    } else {
      const uint64_t cs = orc_next_u64(&sketch_seed_rng);
      if (core_seeds_out) core_seeds_out[iter - 1] = cs;
      CHECK(orc_update_core_fast(order, shape, ranks, core, factors_cat, lambda, x,
                                 o->sample_count_override, o->epsilon, o->delta, cs,
                                 new_core, NULL, NULL, NULL, NULL));
    }
    memcpy(core, new_core, csize * sizeof(double));
    history_iter[hl] = iter;
    history_step[hl] = (int)order;
    orc_tucker_loss(order, shape, ranks, core, factors_cat, lambda, x, &history_loss[hl],
                    &history_rmse[hl]);
    const double loss = history_loss[hl];
    ++hl;
    *iterations_out = iter;
    const double prev_abs = fabs(previous_loss);
    const double change = fabs(previous_loss - loss) / (prev_abs > 1e-300 ? prev_abs : 1e-300);
    previous_loss = loss;
    if (change < o->tolerance) break;
  }
  *history_len_out = hl;
  *final_loss = history_loss[hl - 1];
  *final_rmse = history_rmse[hl - 1];
done:
  free(new_core);
  return status;
}
