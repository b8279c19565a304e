// ref_harness.cpp -- C entry points into the REFERENCE's own C++ core, compiled
// from /root/reference/proj/src sources into oracle/_ref/librtucker_ref.so by
// oracle/Makefile. TEST/BENCH INFRASTRUCTURE ONLY: used to pin the C
// restatement (oracle/rtucker_oracle.c) and as the "reference" CPU arm of
// bench.py. The reference's C API (rtucker_*) is exported by the same .so
// (capi.cpp is compiled in unchanged).
//
// Each function only calls reference routines (rtucker:: namespace); the
// marshalling between flat buffers and DenseMatrix/DenseTensor is ours.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "kronecker.hpp"
#include "leverage.hpp"
#include "linalg.hpp"
#include "sketch_ridge.hpp"
#include "svd.hpp"
#include "tensor.hpp"
#include "tucker.hpp"

using namespace rtucker;

namespace {

thread_local std::string g_err;

template <typename Fn>
int run(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

TuckerModel make_model(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                       const double* core, const double* factors, double lambda) {
  TuckerModel m;
  m.lambda = lambda;
  std::vector<std::size_t> r(ranks, ranks + order);
  std::size_t csize = 1;
  for (auto v : r) csize *= v;
  m.core = DenseTensor(r, std::vector<double>(core, core + csize));
  std::size_t off = 0;
  for (uint32_t n = 0; n < order; ++n) {
    const std::size_t sz = shape[n] * ranks[n];
    m.factors.emplace_back(shape[n], ranks[n],
                           std::vector<double>(factors + off, factors + off + sz));
    off += sz;
  }
  return m;
}

DenseTensor make_tensor(uint32_t order, const uint64_t* shape, const double* x) {
  std::vector<std::size_t> s(shape, shape + order);
  std::size_t size = 1;
  for (auto v : s) size *= v;
  return DenseTensor(s, std::vector<double>(x, x + size));
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_sample_count(double beta_prime, uint64_t d, double epsilon, double delta,
                     uint64_t* out) {
  return run([&] { *out = sample_count(beta_prime, d, epsilon, delta); });
}

int ref_compact_svd(const double* a, uint64_t m, uint64_t n, double* u, double* s,
                    double* vt, uint64_t* rank) {
  return run([&] {
    DenseMatrix am(m, n, std::vector<double>(a, a + m * n));
    CompactSvd sv = compact_svd(am);
    const std::size_t kmax = std::min(m, n);
    std::memset(u, 0, m * kmax * sizeof(double));
    std::memset(s, 0, kmax * sizeof(double));
    std::memset(vt, 0, kmax * n * sizeof(double));
    for (std::size_t k = 0; k < sv.rank(); ++k) {
      s[k] = sv.singular_values[k];
      for (std::size_t i = 0; i < m; ++i) u[i * kmax + k] = sv.u(i, k);
      for (std::size_t j = 0; j < n; ++j) vt[k * n + j] = sv.vt(k, j);
    }
    *rank = sv.rank();
  });
}

// Per-factor scores exactly as ImplicitKronecker caches them (kronecker.cpp:9-35).
int ref_factor_scores(const double* f, uint64_t rows, uint64_t cols, double* scores,
                      double* sum_out, uint64_t* rank_out) {
  return run([&] {
    ImplicitKronecker k({DenseMatrix(rows, cols, std::vector<double>(f, f + rows * cols))});
    const ScoreVector& sv = k.factor_scores(0);
    std::memcpy(scores, sv.scores.data(), rows * sizeof(double));
    *sum_out = k.score_l1();
    *rank_out = k.factor_svd(0).rank();
  });
}

// The sketched core update, unrolled through the public core API exactly as
// update_core_fast does (tucker.cpp:141-166), returning the RowSketch too.
int ref_core_sketch(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                    const double* core, const double* factors, double lambda,
                    const double* x, uint64_t s, uint64_t seed, double* core_out,
                    uint64_t* indices, double* weights, int* rank_deficient,
                    double* sketched_objective) {
  return run([&] {
    const TuckerModel model = make_model(order, shape, ranks, core, factors, lambda);
    const DenseTensor xt = make_tensor(order, shape, x);
    const ImplicitKronecker k(model.factors);
    for (std::size_t n = 0; n < k.factor_count(); ++n) {
      if (k.factor_svd(n).rank() == 0) throw std::invalid_argument("zero factor");
    }
    const ProductLeverageSampler sampler(k, 0.0);
    const KroneckerRowSource source(k);
    SketchConfig cfg;
    cfg.lambda = lambda;
    cfg.seed = seed;
    cfg.sample_count_override = s;
    const SketchedSolution sol = solve_sketched_ridge(source, xt.values(), sampler, lambda, cfg);
    std::memcpy(core_out, sol.x.data(), sol.x.size() * sizeof(double));
    std::memcpy(indices, sol.sketch.sampled_indices.data(), s * sizeof(uint64_t));
    std::memcpy(weights, sol.sketch.weights.data(), s * sizeof(double));
    *rank_deficient = sol.diagnostics.rank_deficient ? 1 : 0;
    *sketched_objective = sol.diagnostics.sketched_objective;
  });
}

int ref_update_core_fast(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                         const double* core, const double* factors, double lambda,
                         const double* x, uint64_t s, uint64_t seed, double* core_out) {
  return run([&] {
    const TuckerModel model = make_model(order, shape, ranks, core, factors, lambda);
    const DenseTensor xt = make_tensor(order, shape, x);
    SketchConfig cfg;
    cfg.seed = seed;
    if (s != 0) cfg.sample_count_override = s;
    const FastCoreResult r = update_core_fast(model, xt, cfg);
    std::memcpy(core_out, r.core.data(), r.core.size() * sizeof(double));
  });
}

// The dense toolkit's RowSketch as the reference makes it: approximate_ridge_regression
// (sketch_ridge.cpp:153-164) with AugmentedSampler(candidate scores, d_eff_lower).
int ref_aug_sketch(const double* a, uint64_t n, uint64_t d, const double* b, const double* cand,
                   double lambda, double d_eff_lower, uint64_t s, uint64_t seed,
                   uint64_t* indices, double* weights) {
  return run([&] {
    DenseMatrix am(n, d);
    std::memcpy(am.data(), a, n * d * sizeof(double));
    ScoreVector sc;
    sc.scores.assign(cand, cand + n);
    SketchConfig cfg;
    cfg.lambda = lambda;
    cfg.seed = seed;
    cfg.sample_count_override = s;
    const SketchedSolution sol =
        approximate_ridge_regression(am, std::span<const double>(b, n), sc, d_eff_lower, cfg);
    std::memcpy(indices, sol.sketch.sampled_indices.data(), s * sizeof(uint64_t));
    std::memcpy(weights, sol.sketch.weights.data(), s * sizeof(double));
  });
}

// Times the reference's own public update_core_fast (ref tucker.cpp:141-166) on a given
// model (bench.py's reference arm): out[0] = seconds of the call, out[1] = setup (factor
// SVDs, scores, CDFs), out[2] = draws, out[3] = response gather, out[4] = solve (the
// streamed Gram/RHS of sketch_ridge.cpp:105-128 + the Jacobi compact_svd of the d x d Gram
// + the pinv apply), out[5] = data rows among the s draws (the same stream redrawn).
int ref_time_core_fast(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                       const double* core, const double* factors, double lambda,
                       const double* x, uint64_t s, uint64_t seed, double* out) {
  return run([&] {
    const TuckerModel model = make_model(order, shape, ranks, core, factors, lambda);
    const DenseTensor xt = make_tensor(order, shape, x);
    SketchConfig cfg;
    cfg.seed = seed;
    cfg.sample_count_override = s;
    const double t0 = now_s();
    const FastCoreResult r = update_core_fast(model, xt, cfg);
    out[0] = now_s() - t0;
    out[1] = r.setup_seconds;
    out[2] = r.diagnostics.draw_seconds;
    out[3] = r.diagnostics.gather_seconds;
    out[4] = r.diagnostics.solve_seconds;
    const ImplicitKronecker k(model.factors);
    const ProductLeverageSampler sampler(k, 0.0);
    SplitMix64 rng(seed);
    std::size_t n_data = 0;
    for (std::size_t t = 0; t < s; ++t)
      if (sampler.draw(rng).first < k.rows()) ++n_data;
    out[5] = static_cast<double>(n_data);
  });
}

int ref_update_factor(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                      const double* core, const double* factors, double lambda,
                      const double* x, uint32_t mode, double* factor_out) {
  return run([&] {
    const TuckerModel model = make_model(order, shape, ranks, core, factors, lambda);
    const DenseTensor xt = make_tensor(order, shape, x);
    const DenseMatrix f = update_factor(model, xt, mode);
    std::memcpy(factor_out, f.data(), f.size() * sizeof(double));
  });
}

int ref_update_core_exact(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                          const double* core, const double* factors, double lambda,
                          const double* x, double* core_out) {
  return run([&] {
    const TuckerModel model = make_model(order, shape, ranks, core, factors, lambda);
    const DenseTensor xt = make_tensor(order, shape, x);
    const DenseTensor c = update_core_exact(model, xt);
    std::memcpy(core_out, c.data(), c.size() * sizeof(double));
  });
}

int ref_tucker_loss(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                    const double* core, const double* factors, double lambda,
                    const double* x, double* loss) {
  return run([&] {
    const TuckerModel model = make_model(order, shape, ranks, core, factors, lambda);
    const DenseTensor xt = make_tensor(order, shape, x);
    *loss = tucker_loss(model, xt);
  });
}

int ref_random_model(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                     uint64_t seed, double* core, double* factors) {
  return run([&] {
    SplitMix64 rng(seed);
    const TuckerModel m = random_model(std::vector<std::size_t>(shape, shape + order),
                                       std::vector<std::size_t>(ranks, ranks + order), 0.0,
                                       rng);
    std::memcpy(core, m.core.data(), m.core.size() * sizeof(double));
    std::size_t off = 0;
    for (const DenseMatrix& f : m.factors) {
      std::memcpy(factors + off, f.data(), f.size() * sizeof(double));
      off += f.size();
    }
  });
}

// Bench support ("reference" CPU arm): times the reference's own routines for
// the phases of one sketched ALS sweep on bounded samples. out[0..5]:
//   [0] seconds for update_factor(mode) (one mode)
//   [1] seconds for one full loss evaluation (reconstruct + residual)
//   [2] seconds per data sample of the streamed Gram/RHS accumulation
//       (measured on `gram_samples` data draws of the real design)
//   [3] seconds for ImplicitKronecker setup (factor SVDs, scores, CDFs)
//   [4] seconds for compact_svd of an svd_dim x svd_dim SPD Gram
//   [5] number of data draws among the s draws of the sketch (exact count)
int ref_time_sweep_phases(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                          const double* core, const double* factors, double lambda,
                          const double* x, uint64_t s, uint64_t seed, uint32_t mode,
                          uint64_t gram_samples, uint64_t svd_dim, int do_factor,
                          int do_loss, double* out) {
  return run([&] {
    const TuckerModel model = make_model(order, shape, ranks, core, factors, lambda);
    const DenseTensor xt = make_tensor(order, shape, x);
    for (int i = 0; i < 6; ++i) out[i] = 0.0;
    double t0;
    if (do_factor) {
      t0 = now_s();
      const DenseMatrix f = update_factor(model, xt, mode);
      out[0] = now_s() - t0;
      if (!std::isfinite(f.data()[0])) throw std::runtime_error("bad factor");
    }
    if (do_loss) {
      t0 = now_s();
      volatile double l = tucker_loss(model, xt);
      (void)l;
      out[1] = now_s() - t0;
    }
    t0 = now_s();
    const ImplicitKronecker k(model.factors);
    const ProductLeverageSampler sampler(k, 0.0);
    out[3] = now_s() - t0;
    // draw the full sketch (cheap), then stream the Gram over a bounded
    // number of its data rows with the same arithmetic as
    // sketch_ridge.cpp:105-128.
    SplitMix64 rng(seed);
    std::vector<std::pair<std::size_t, double>> draws;
    draws.reserve(s);
    std::size_t n_data = 0;
    for (std::size_t t = 0; t < s; ++t) {
      draws.push_back(sampler.draw(rng));
      if (draws.back().first < k.rows()) ++n_data;
    }
    out[5] = static_cast<double>(n_data);
    const KroneckerRowSource source(k);
    const std::size_t d = k.cols();
    DenseMatrix g(d, d);
    std::vector<double> rhs(d, 0.0), row(d);
    const double inv_s = 1.0 / static_cast<double>(s);
    std::size_t done = 0;
    t0 = now_s();
    for (std::size_t t = 0; t < s && done < gram_samples; ++t) {
      if (draws[t].first >= k.rows()) continue;
      const double w = std::sqrt(inv_s / draws[t].second);
      source.copy_row(draws[t].first, row);
      const double w2 = w * w;
      for (std::size_t p = 0; p < d; ++p) {
        const double v = w2 * row[p];
        if (v == 0.0) continue;
        double* grow = g.data() + p * d;
        for (std::size_t q = p; q < d; ++q) grow[q] += v * row[q];
      }
      const double wb = w2 * xt[draws[t].first];
      if (wb != 0.0)
        for (std::size_t p = 0; p < d; ++p) rhs[p] += wb * row[p];
      ++done;
    }
    out[2] = done ? (now_s() - t0) / static_cast<double>(done) : 0.0;
    if (svd_dim > 0) {
      // SPD test Gram of the requested size built from the design rows seen.
      DenseMatrix a(svd_dim, svd_dim);
      SplitMix64 r2(seed ^ 0x1234);
      for (std::size_t i = 0; i < a.size(); ++i) a.data()[i] = r2.next_double() - 0.5;
      DenseMatrix spd = gram(a);
      for (std::size_t i = 0; i < svd_dim; ++i) spd(i, i) += 1e-3;
      t0 = now_s();
      const CompactSvd sv = compact_svd(spd);
      out[4] = now_s() - t0;
      if (sv.rank() == 0) throw std::runtime_error("bad svd");
    }
  });
}

}  // extern "C"
