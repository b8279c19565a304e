// verify.cu -- rtucker_verify_suite (ref verify.cpp:85-416, capi.cpp:364-403): the four
// property suites of the reference -- leverage, kronecker, missing, structural -- with the
// reference's check names, bounds, trial counts and trial-size ranges, run against THIS
// library's GPU routines (ridge leverage scores by the device one-sided Jacobi SVD,
// factored Kronecker scores from the per-factor device scores, the AugmentedSampler draws
// of the dense toolkit) and checked against independent host-side formulas (small dense
// eigen/SVD algebra below). The trials' random matrices come from SplitMix64(seed) in this
// file's own order, so they are not the reference's matrices; the properties and bounds
// are. Report: a JSON array of {suite, passed, elapsed_seconds, checks[{name, passed,
// observed, bound}]} as the reference's C API writes it.
#include <algorithm>
#include <chrono>
#include <cfloat>
#include <cmath>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "engine.h"

namespace rtb {

namespace {

struct HRng {  // host SplitMix64 (ref rng.hpp:12-62)
  uint64_t state;
  uint64_t next() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double unit() { return (double)(next() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t b) {
    const uint64_t thr = (0 - b) % b;
    for (;;) {
      const uint64_t r = next();
      if (r >= thr) return r % b;
    }
  }
};

struct Mat {
  size_t r = 0, c = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(size_t rows, size_t cols) : r(rows), c(cols), v(rows * cols, 0.0) {}
  double& operator()(size_t i, size_t j) { return v[i * c + j]; }
  double operator()(size_t i, size_t j) const { return v[i * c + j]; }
};

Mat rand_mat(HRng& g, size_t rows, size_t cols) {
  Mat m(rows, cols);
  for (auto& x : m.v) x = 2.0 * g.unit() - 1.0;
  return m;
}

// cyclic Jacobi eigen of a small symmetric matrix: eigenvalues descending, V columns
void sym_eig(const Mat& a, std::vector<double>& mu, Mat& V) {
  const size_t n = a.r;
  Mat A = a;
  V = Mat(n, n);
  for (size_t i = 0; i < n; ++i) V(i, i) = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (size_t p = 0; p < n; ++p)
      for (size_t q = 0; q < n; ++q) {
        tot += A(p, q) * A(p, q);
        if (p != q) off += A(p, q) * A(p, q);
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (size_t p = 0; p + 1 < n; ++p)
      for (size_t q = p + 1; q < n; ++q) {
        if (A(p, q) == 0.0) continue;
        const double th = (A(q, q) - A(p, p)) / (2.0 * A(p, q));
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(1.0 + th * th));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
        for (size_t k = 0; k < n; ++k) {
          const double ap = A(k, p), aq = A(k, q);
          A(k, p) = cs * ap - sn * aq;
          A(k, q) = sn * ap + cs * aq;
        }
        for (size_t k = 0; k < n; ++k) {
          const double ap = A(p, k), aq = A(q, k);
          A(p, k) = cs * ap - sn * aq;
          A(q, k) = sn * ap + cs * aq;
          const double vp = V(k, p), vq = V(k, q);
          V(k, p) = cs * vp - sn * vq;
          V(k, q) = sn * vp + cs * vq;
        }
      }
  }
  std::vector<size_t> ord(n);
  for (size_t i = 0; i < n; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](size_t x, size_t y) { return A(x, x) > A(y, y); });
  Mat W(n, n);
  mu.resize(n);
  for (size_t k = 0; k < n; ++k) {
    mu[k] = A(ord[k], ord[k]);
    for (size_t i = 0; i < n; ++i) W(i, k) = V(i, ord[k]);
  }
  V = W;
}

// compact SVD of a small matrix from the eigenpairs of its smaller Gram: U (m x rank), sigma
void svd_small(const Mat& a, Mat& U, std::vector<double>& sig) {
  const size_t m = a.r, n = a.c;
  const bool tall = m >= n;
  const size_t k = tall ? n : m;
  Mat g(k, k);
  for (size_t p = 0; p < k; ++p)
    for (size_t q = 0; q < k; ++q) {
      double s = 0.0;
      if (tall)
        for (size_t i = 0; i < m; ++i) s += a(i, p) * a(i, q);
      else
        for (size_t j = 0; j < n; ++j) s += a(p, j) * a(q, j);
      g(p, q) = s;
    }
  std::vector<double> mu;
  Mat V;
  sym_eig(g, mu, V);
  const double smax = std::sqrt(std::max(mu[0], 0.0));
  const double cut = (double)std::max(m, n) * DBL_EPSILON * smax;
  sig.clear();
  for (size_t r = 0; r < k; ++r) {
    const double s = std::sqrt(std::max(mu[r], 0.0));
    if (s > cut && s > 0.0) sig.push_back(s);
  }
  U = Mat(m, sig.size());
  for (size_t r = 0; r < sig.size(); ++r) {
    if (tall) {
      for (size_t i = 0; i < m; ++i) {
        double s = 0.0;
        for (size_t j = 0; j < n; ++j) s += a(i, j) * V(j, r);
        U(i, r) = s / sig[r];
      }
    } else {
      for (size_t i = 0; i < m; ++i) U(i, r) = V(i, r);
    }
  }
}

// cross-score row i: L_ij = sum_k s_k^2 / (s_k^2 + lambda) u_ik u_jk
std::vector<double> cross_row(const Mat& U, const std::vector<double>& s, size_t i, double lam) {
  std::vector<double> row(U.r, 0.0);
  for (size_t k = 0; k < s.size(); ++k) {
    const double w = s[k] * s[k] / (s[k] * s[k] + lam) * U(i, k);
    for (size_t j = 0; j < U.r; ++j) row[j] += w * U(j, k);
  }
  return row;
}

// pinv with the reference cutoff (ref linalg.cpp:8-26) of a small symmetric matrix
Mat pinv_sym(const Mat& a) {
  std::vector<double> mu;
  Mat V;
  sym_eig(a, mu, V);
  double amax = 0.0;
  for (double m : mu) amax = std::max(amax, std::fabs(m));
  const double cut = (double)a.r * DBL_EPSILON * amax;
  Mat p(a.r, a.r);
  for (size_t k = 0; k < a.r; ++k) {
    if (!(std::fabs(mu[k]) > cut) || mu[k] == 0.0) continue;
    for (size_t i = 0; i < a.r; ++i)
      for (size_t j = 0; j < a.r; ++j) p(i, j) += V(i, k) * V(j, k) / mu[k];
  }
  return p;
}

std::vector<double> dev_scores(const Mat& a, double lam) {
  std::vector<double> s(a.r);
  dense_ridge_scores(a.v.data(), a.r, a.c, lam, s.data());
  return s;
}

Mat augmented(const Mat& a, double lam) {
  Mat b(a.r + a.c, a.c);
  for (size_t i = 0; i < a.r; ++i)
    for (size_t j = 0; j < a.c; ++j) b(i, j) = a(i, j);
  for (size_t j = 0; j < a.c; ++j) b(a.r + j, j) = std::sqrt(lam);
  return b;
}

struct Check {
  std::string name;
  bool min_style;
  double observed, bound;
  bool passed;
};
struct Suite {
  std::string name;
  bool passed;
  double seconds;
  std::vector<Check> checks;
};

class Rec {
 public:
  explicit Rec(std::string n) : t0_(std::chrono::steady_clock::now()) { s_.name = std::move(n); }
  void max(const std::string& n, double v, double bound) {
    Check& c = get(n, bound, false);
    if (v > c.observed || std::isnan(v)) c.observed = v;
  }
  void min(const std::string& n, double v, double bound) {
    Check& c = get(n, bound, true);
    if (v < c.observed || std::isnan(v)) c.observed = v;
  }
  Suite done() {
    s_.passed = true;
    for (auto& c : s_.checks) {
      c.passed = c.min_style ? c.observed >= c.bound : c.observed <= c.bound;
      s_.passed &= c.passed;
    }
    s_.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
    return s_;
  }

 private:
  Check& get(const std::string& n, double bound, bool mn) {
    for (auto& c : s_.checks)
      if (c.name == n) return c;
    s_.checks.push_back({n, mn, mn ? std::numeric_limits<double>::infinity()
                                   : -std::numeric_limits<double>::infinity(),
                         bound, false});
    return s_.checks.back();
  }
  Suite s_;
  std::chrono::steady_clock::time_point t0_;
};

Suite leverage_suite(uint64_t seed, int trials) {
  Rec rec("leverage");
  HRng g{seed};
  const double lams[] = {0.0, 0.01, 0.5, 2.0};
  for (int t = 0; t < trials; ++t) {
    const size_t n = 2 + g.below(49), d = 1 + g.below(8);
    const double lam = lams[t % 4];
    const Mat a = rand_mat(g, n, d);
    const std::vector<double> sc = dev_scores(a, lam);   // device: one-sided Jacobi SVD form
    const std::vector<double> cl = dev_scores(a, 0.0);
    // pinv form on the host: a_i^T (A^T A + lambda I)^+ a_i
    Mat nrm(d, d);
    for (size_t p = 0; p < d; ++p)
      for (size_t q = 0; q < d; ++q) {
        double s = 0.0;
        for (size_t i = 0; i < n; ++i) s += a(i, p) * a(i, q);
        nrm(p, q) = s + (p == q ? lam : 0.0);
      }
    const Mat inv = pinv_sym(nrm);
    double diff = 0.0;
    for (size_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (size_t p = 0; p < d; ++p)
        for (size_t q = 0; q < d; ++q) s += a(i, p) * inv(p, q) * a(i, q);
      diff = std::max(diff, std::fabs(sc[i] - s));
    }
    rec.max("svd_form_vs_pinv_form", diff, 1e-9);
    Mat U;
    std::vector<double> sig;
    svd_small(a, U, sig);
    double deff = 0.0, eff = 0.0;
    for (double s : sig) deff += s * s / (s * s + lam);
    for (double s : sc) eff += s;
    rec.max("effective_dimension_vs_singular_sum", std::fabs(eff - deff), 1e-9);
    rec.max("effective_dimension_at_most_rank", eff - (double)sig.size(), 1e-9);
    if (lam > 0.0) {  // ridge scores of A = classical scores of [A; sqrt(lambda) I], first n rows
      const std::vector<double> ab = dev_scores(augmented(a, lam), 0.0);
      double m = 0.0;
      for (size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(sc[i] - ab[i]));
      rec.max("augmented_design_equality", m, 1e-9);
    }
    for (size_t i = 0; i < n; ++i) {
      rec.min("scores_nonnegative", sc[i], -1e-12);
      rec.max("ridge_at_most_classical", sc[i] - cl[i], 1e-12);
      rec.max("classical_at_most_one", cl[i], 1.0 + 1e-12);
    }
    const size_t probe = g.below(n);
    const std::vector<double> row = cross_row(U, sig, probe, lam);
    double ss = 0.0;
    for (double v : row) ss += v * v;
    if (lam == 0.0) rec.max("sum_squared_cross_equality_at_zero", std::fabs(ss - sc[probe]), 1e-10);
    else rec.max("sum_squared_cross_below_score", ss - sc[probe], 1e-12);
  }
  return rec.done();
}

// materialised Kronecker product of factors (rows last-mode fastest, ref kronecker.cpp:54-75)
Mat kron(const std::vector<Mat>& f) {
  Mat k(1, 1);
  k(0, 0) = 1.0;
  for (const Mat& b : f) {
    Mat o(k.r * b.r, k.c * b.c);
    for (size_t i = 0; i < k.r; ++i)
      for (size_t j = 0; j < b.r; ++j)
        for (size_t p = 0; p < k.c; ++p)
          for (size_t q = 0; q < b.c; ++q) o(i * b.r + j, p * b.c + q) = k(i, p) * b(j, q);
    k = o;
  }
  return k;
}

Suite kronecker_suite(uint64_t seed, int trials) {
  Rec rec("kronecker");
  HRng g{seed};
  for (int t = 0; t < trials; ++t) {
    const size_t order = 2 + t % 2;
    std::vector<Mat> f;
    size_t total = 1;
    for (size_t n = 0; n < order; ++n) {
      const size_t rows = 2 + g.below(order == 2 ? 7 : 5), cols = 1 + g.below(3);
      f.push_back(rand_mat(g, rows, cols));
      total *= rows;
    }
    const double lam = 0.1 + g.unit();
    const Mat K = kron(f);
    // factored classical scores (device scores of each factor, multiplied) vs the device
    // scores of the materialised product
    std::vector<std::vector<double>> fsc;
    for (const Mat& m : f) {
      std::vector<double> sc(m.r), cdf(m.r);
      double sum = 0.0;
      uint64_t rank = 0;
      factor_scores(m.v.data(), (int)m.r, (int)m.c, sc.data(), cdf.data(), &sum, &rank);
      fsc.push_back(sc);
    }
    const std::vector<double> ksc = dev_scores(K, 0.0);
    double diff = 0.0;
    for (size_t flat = 0; flat < total; ++flat) {
      size_t rem = flat;
      double s = 1.0;
      for (size_t n = order; n-- > 0;) {
        s *= fsc[n][rem % f[n].r];
        rem /= f[n].r;
      }
      diff = std::max(diff, std::fabs(s - ksc[flat]));
    }
    rec.max("factored_scores_vs_materialized", diff, 1e-9);
    // ridge cross scores from the factor SVDs vs the materialised cross matrix
    std::vector<Mat> Us(order);
    std::vector<std::vector<double>> ss(order);
    for (size_t n = 0; n < order; ++n) svd_small(f[n], Us[n], ss[n]);
    Mat UK;
    std::vector<double> sK;
    svd_small(K, UK, sK);
    auto digits = [&](size_t flat) {
      std::vector<size_t> d(order);
      for (size_t n = order; n-- > 0;) {
        d[n] = flat % f[n].r;
        flat /= f[n].r;
      }
      return d;
    };
    double dmax = 0.0;
    for (int probe = 0; probe < 20; ++probe) {
      const size_t i = g.below(total), j = g.below(total);
      const auto di = digits(i), dj = digits(j);
      double fast = 0.0;
      std::vector<size_t> tt(order, 0);
      bool any = true;
      for (size_t n = 0; n < order; ++n) any &= !ss[n].empty();
      while (any) {
        double s2 = 1.0, ui = 1.0, uj = 1.0;
        for (size_t n = 0; n < order; ++n) {
          s2 *= ss[n][tt[n]] * ss[n][tt[n]];
          ui *= Us[n](di[n], tt[n]);
          uj *= Us[n](dj[n], tt[n]);
        }
        fast += s2 / (s2 + lam) * ui * uj;
        size_t n = order;
        while (n-- > 0) {
          if (++tt[n] < ss[n].size()) break;
          tt[n] = 0;
        }
        if (n == (size_t)-1) break;
      }
      const std::vector<double> row = cross_row(UK, sK, i, lam);
      dmax = std::max(dmax, std::fabs(fast - row[j]));
    }
    rec.max("ridge_cross_scores_vs_materialized", dmax, 1e-9);
    if (total <= 64) {  // eigenvalues of the cross matrix: prod s^2 / (prod s^2 + lambda)
      Mat L(total, total);
      for (size_t i = 0; i < total; ++i) {
        const std::vector<double> row = cross_row(UK, sK, i, lam);
        for (size_t j = 0; j < total; ++j) L(i, j) = row[j];
      }
      std::vector<double> mu;
      Mat V;
      sym_eig(L, mu, V);
      std::vector<double> want;
      std::vector<size_t> tt(order, 0);
      for (;;) {
        double s2 = 1.0;
        for (size_t n = 0; n < order; ++n) s2 *= ss[n][tt[n]] * ss[n][tt[n]];
        want.push_back(s2 / (s2 + lam));
        size_t n = order;
        while (n-- > 0) {
          if (++tt[n] < ss[n].size()) break;
          tt[n] = 0;
        }
        if (n == (size_t)-1) break;
      }
      want.resize(total, 0.0);
      std::sort(want.begin(), want.end(), std::greater<double>());
      double m = 0.0;
      for (size_t i = 0; i < total; ++i) m = std::max(m, std::fabs(mu[i] - want[i]));
      rec.max("cross_matrix_eigenvalue_formula", m, 1e-8);
    }
  }
  return rec.done();
}

Suite missing_suite(uint64_t seed, int trials) {
  Rec rec("missing");
  HRng g{seed};
  for (int t = 0; t < trials; ++t) {
    const size_t n = 6 + g.below(7), d = 2 + g.below(3);
    const Mat a = rand_mat(g, n, d);
    const double lam = 0.05 + 2.0 * g.unit();
    const size_t rc = 1 + g.below(n - 2);
    std::vector<size_t> pool(n), removed;
    for (size_t i = 0; i < n; ++i) pool[i] = i;
    for (size_t k = 0; k < rc; ++k) {
      const size_t j = k + g.below(n - k);
      std::swap(pool[k], pool[j]);
      removed.push_back(pool[k]);
    }
    std::sort(removed.begin(), removed.end());
    std::vector<size_t> kept;
    for (size_t i = 0; i < n; ++i)
      if (!std::binary_search(removed.begin(), removed.end(), i)) kept.push_back(i);
    Mat U;
    std::vector<double> sig;
    svd_small(a, U, sig);
    const std::vector<double> orig = dev_scores(a, lam);
    // Woodbury: l'_i = l_i + v^T (I - L_SS)^-1 v, v = L_{i,S} (ref missing.cpp:50-78)
    Mat LSS(rc, rc);
    for (size_t p = 0; p < rc; ++p) {
      const std::vector<double> row = cross_row(U, sig, removed[p], lam);
      for (size_t q = 0; q < rc; ++q) LSS(p, q) = row[removed[q]];
    }
    Mat corr(rc, rc);
    for (size_t p = 0; p < rc; ++p)
      for (size_t q = 0; q < rc; ++q) corr(p, q) = (p == q ? 1.0 : 0.0) - LSS(p, q);
    const Mat inv = pinv_sym(corr);
    std::vector<double> lmu;
    Mat lv;
    sym_eig(LSS, lmu, lv);
    const double coeff = 1.0 / (1.0 - lmu[0]);
    Mat red(kept.size(), d);
    for (size_t k = 0; k < kept.size(); ++k)
      for (size_t j = 0; j < d; ++j) red(k, j) = a(kept[k], j);
    const std::vector<double> recomputed = dev_scores(red, lam);
    for (size_t k = 0; k < kept.size(); ++k) {
      const std::vector<double> row = cross_row(U, sig, kept[k], lam);
      std::vector<double> v(rc);
      double vv = 0.0;
      for (size_t p = 0; p < rc; ++p) {
        v[p] = row[removed[p]];
        vv += v[p] * v[p];
      }
      double quad = 0.0;
      for (size_t p = 0; p < rc; ++p)
        for (size_t q = 0; q < rc; ++q) quad += v[p] * inv(p, q) * v[q];
      const double upd = orig[kept[k]] + quad, bound = orig[kept[k]] + coeff * vv;
      rec.max("woodbury_update_vs_recomputation", std::fabs(upd - recomputed[k]), 1e-8);
      rec.min("bound_dominates_exact", bound - upd, -1e-9);
      rec.min("scores_never_decrease", upd - orig[kept[k]], -1e-10);
    }
    const size_t probe = g.below(n);
    const std::vector<double> zsc = dev_scores(a, 0.0);
    auto sumsq = [&](double l) {
      const std::vector<double> row = cross_row(U, sig, probe, l);
      double s = 0.0;
      for (double x : row) s += x * x;
      return s;
    };
    rec.max("sum_squared_cross_equality_at_zero", std::fabs(sumsq(0.0) - zsc[probe]), 1e-10);
    rec.max("sum_squared_cross_below_score", sumsq(lam) - orig[probe], 1e-12);
    if (t % 10 == 0) {  // 1 + prod sigma_max^2 / lambda dominates 1 / (1 - lambda_max(L_SS))
      std::vector<Mat> f{rand_mat(g, 3, 2), rand_mat(g, 4, 2)};
      const Mat K = kron(f);
      const double kl = 0.2 + g.unit();
      double prod2 = 1.0;
      for (const Mat& m : f) {
        Mat Um;
        std::vector<double> sm;
        svd_small(m, Um, sm);
        prod2 *= sm.empty() ? 0.0 : sm[0] * sm[0];
      }
      const double kc = 1.0 + prod2 / kl;
      Mat UK;
      std::vector<double> sK;
      svd_small(K, UK, sK);
      for (int rep = 0; rep < 5; ++rep) {
        const size_t rr = 1 + g.below(K.r - 2);
        std::vector<size_t> pl(K.r), rem;
        for (size_t i = 0; i < K.r; ++i) pl[i] = i;
        for (size_t k = 0; k < rr; ++k) {
          const size_t j = k + g.below(K.r - k);
          std::swap(pl[k], pl[j]);
          rem.push_back(pl[k]);
        }
        Mat sub(rr, rr);
        for (size_t p = 0; p < rr; ++p) {
          const std::vector<double> row = cross_row(UK, sK, rem[p], kl);
          for (size_t q = 0; q < rr; ++q) sub(p, q) = row[rem[q]];
        }
        std::vector<double> smu;
        Mat sv;
        sym_eig(sub, smu, sv);
        rec.min("kronecker_coefficient_dominates", kc - 1.0 / (1.0 - smu[0]), -1e-9);
      }
    }
  }
  return rec.done();
}

Suite structural_suite(uint64_t seed, int emb_trials, int sketches) {
  Rec rec("structural");
  HRng g{seed};
  {  // subspace embedding at the formula sample count, 30 x 3, lambda 0.1
    const double delta = 0.25, eps = 0.5, lam = 0.1;
    const Mat a = rand_mat(g, 30, 3);
    const std::vector<double> cand = dev_scores(a, 0.0);
    Mat U;
    std::vector<double> sig;
    svd_small(augmented(a, lam), U, sig);
    const uint64_t s = sample_count_formula(0.5, 3, eps, delta);
    std::vector<uint64_t> idx(s);
    std::vector<double> w(s);
    int hits = 0;
    for (int tr = 0; tr < emb_trials; ++tr) {
      aug_draw(cand.data(), 30, 3, 0.0, g.next(), s, idx.data(), w.data());  // device sampler
      Mat gsu(sig.size(), sig.size());
      for (uint64_t t = 0; t < s; ++t)
        for (size_t p = 0; p < sig.size(); ++p)
          for (size_t q = 0; q < sig.size(); ++q) gsu(p, q) += w[t] * w[t] * U(idx[t], p) * U(idx[t], q);
      std::vector<double> mu;
      Mat V;
      sym_eig(gsu, mu, V);
      if (!mu.empty() && mu.back() >= 1.0 / std::sqrt(2.0)) ++hits;
    }
    rec.min("subspace_embedding_hit_rate", (double)hits / emb_trials, 1.0 - delta);
  }
  {  // approximate matrix multiplication: E ||(S U)^T S bperp||^2 <= r ||bperp||^2 / (beta s)
    const double lam = 0.3;
    const uint64_t s = 32;
    const Mat a = rand_mat(g, 8, 2);
    std::vector<double> b(8);
    for (auto& x : b) x = 2.0 * g.unit() - 1.0;
    const Mat ab = augmented(a, lam);
    std::vector<double> bb(b);
    bb.resize(10, 0.0);
    Mat U;
    std::vector<double> sig;
    svd_small(ab, U, sig);
    const size_t r = sig.size();
    std::vector<double> bp(bb);
    for (size_t k = 0; k < r; ++k) {
      double ub = 0.0;
      for (size_t i = 0; i < 10; ++i) ub += U(i, k) * bb[i];
      for (size_t i = 0; i < 10; ++i) bp[i] -= U(i, k) * ub;
    }
    double bpn = 0.0;
    for (double v : bp) bpn += v * v;
    // sampler probabilities (ref sampler.cpp:9-40, 59-70) and the realised beta
    const std::vector<double> cand = dev_scores(a, 0.0);
    double l1 = 0.0;
    for (double c : cand) l1 += c;
    std::vector<double> prob(10);
    double data = 0.0;
    for (size_t i = 0; i < 8; ++i) data += cand[i] * (2.0 / l1);
    const double total = data + 2.0 * 1.0;
    for (size_t i = 0; i < 8; ++i) prob[i] = cand[i] * (2.0 / l1) / total;
    prob[8] = prob[9] = 1.0 / total;
    const std::vector<double> ex = dev_scores(ab, 0.0);
    double pl1 = 0.0, el1 = 0.0, beta = std::numeric_limits<double>::infinity();
    for (size_t i = 0; i < 10; ++i) {
      pl1 += prob[i];
      el1 += ex[i];
    }
    for (size_t i = 0; i < 10; ++i)
      if (ex[i] > 0.0) beta = std::min(beta, (prob[i] / pl1) / (ex[i] / el1));
    const uint64_t nd = s * (uint64_t)sketches;
    std::vector<uint64_t> idx(nd);
    std::vector<double> w(nd);
    aug_draw(cand.data(), 8, 2, 0.0, g.next(), nd, idx.data(), w.data());  // device sampler
    double mse = 0.0;
    for (int k = 0; k < sketches; ++k) {
      std::vector<double> est(r, 0.0);
      for (uint64_t t = 0; t < s; ++t) {
        const uint64_t j = idx[(uint64_t)k * s + t];
        const double w2 = 1.0 / (prob[j] * (double)s);
        for (size_t q = 0; q < r; ++q) est[q] += w2 * U(j, q) * bp[j];
      }
      for (double v : est) mse += v * v;
    }
    mse /= sketches;
    rec.max("matrix_multiplication_variance_bound", mse, 1.2 * (double)r * bpn / (beta * (double)s));
  }
  return rec.done();
}

std::string json_num(double v) {
  if (std::isnan(v)) return "null";
  if (std::isinf(v)) return v > 0 ? "1e308" : "-1e308";
  std::ostringstream o;
  o.precision(17);
  o << v;
  return o.str();
}

}  // namespace

// runs one suite ("leverage", "kronecker", "missing", "structural") or "all"; returns the
// JSON report and whether every check passed (ref capi.cpp:364-403)
bool verify_suites(const std::string& name, uint64_t seed, std::string& json) {
  std::vector<Suite> out;
  auto run = [&](const std::string& n) {
    if (n == "leverage") out.push_back(leverage_suite(seed, 200));
    else if (n == "kronecker") out.push_back(kronecker_suite(seed, 50));
    else if (n == "missing") out.push_back(missing_suite(seed, 100));
    else if (n == "structural") out.push_back(structural_suite(seed, 200, 10000));
    else throw Error(1, "run_suite: unknown suite " + n);
  };
  if (name == "all") {
    for (const char* n : {"leverage", "kronecker", "missing", "structural"}) run(n);
  } else {
    run(name);
  }
  bool all = true;
  std::ostringstream o;
  o << "[\n";
  for (size_t i = 0; i < out.size(); ++i) {
    const Suite& s = out[i];
    all &= s.passed;
    o << "  {\n    \"checks\": [\n";
    for (size_t k = 0; k < s.checks.size(); ++k) {
      const Check& c = s.checks[k];
      o << "      {\n        \"bound\": " << json_num(c.bound) << ",\n        \"name\": \"" << c.name
        << "\",\n        \"observed\": " << json_num(c.observed) << ",\n        \"passed\": "
        << (c.passed ? "true" : "false") << "\n      }" << (k + 1 < s.checks.size() ? "," : "")
        << "\n";
    }
    o << "    ],\n    \"elapsed_seconds\": " << json_num(s.seconds) << ",\n    \"passed\": "
      << (s.passed ? "true" : "false") << ",\n    \"suite\": \"" << s.name << "\"\n  }"
      << (i + 1 < out.size() ? "," : "") << "\n";
  }
  o << "]";
  json = o.str();
  return all;
}

}  // namespace rtb
