/* rtucker_oracle.h -- CPU restatement of the reference's sketched Tucker-ALS
 * hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity checker for the B200 build. Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * legs may load it. The product library (librtucker_b200.so) never links or
 * calls it; there is no CPU fallback.
 *
 * Every routine restates an algorithm of the reference in plain C99 with the
 * same floating-point operation order, so results are bit-identical to the
 * compiled reference (pinned by tests/test_oracle_pin.py against oracle/_ref,
 * which is the reference compiled from /root/reference/proj sources, and by the
 * committed golden vectors in tests/golden/). Citations are
 * /root/reference/proj/<path>:<line>.
 *
 * Layout conventions follow the reference: row-major matrices, tensors in
 * canonical order with the last index fastest (src/core/tensor.hpp:11-15).
 * Status codes follow include/rtucker.h (0 OK, 1 invalid argument,
 * 3 numerical); the message is in oracle_last_error().
 */
#ifndef RTUCKER_ORACLE_H
#define RTUCKER_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* oracle_last_error(void);

/* ---- SplitMix64 (src/core/rng.hpp:12-62) ---- */
typedef struct {
  uint64_t state;
} orc_rng;
uint64_t orc_next_u64(orc_rng* r);
double orc_next_double(orc_rng* r);
uint64_t orc_next_below(orc_rng* r, uint64_t bound);
uint64_t orc_split_seed(orc_rng* r);
/* k-th output of SplitMix64(seed), k >= 0 (counter form of rng.hpp:16-21). */
uint64_t orc_splitmix_at(uint64_t seed, uint64_t k);
/* Fills out[0..n) with consecutive next_u64() values of SplitMix64(seed). */
void orc_splitmix_stream(uint64_t seed, uint64_t n, uint64_t* out);

/* ---- compact SVD by one-sided Jacobi (src/core/svd.cpp:21-129) ----
 * a: m x n row-major. Outputs sized for the full min(m,n) rank:
 * u_out m x min(m,n) (row-major, leading dim = min(m,n)), s_out[min(m,n)],
 * vt_out min(m,n) x n. *rank_out receives the numerical rank; only the first
 * rank columns/rows are meaningful. Returns 0, 1 (empty) or 3 (no convergence). */
int orc_compact_svd(const double* a, size_t m, size_t n, double* u_out, double* s_out,
                    double* vt_out, size_t* rank_out);

/* ---- leverage scores (src/core/leverage.cpp:16-52) ---- */
int orc_ridge_scores(const double* a, size_t n, size_t d, double lambda, double* scores);

/* ---- dense ridge solves (src/core/linalg.cpp:8-41) ---- */
int orc_pseudoinverse(const double* a, size_t m, size_t n, double* pinv /* n x m */);
int orc_solve_ridge_exact(const double* a, size_t n, size_t d, const double* b,
                          double lambda, double* x);

/* ---- sampling (src/core/sketch_ridge.cpp:40-50, sampler.cpp:9-57) ---- */
int orc_sample_count(double beta_prime, size_t d, double epsilon, double delta,
                     uint64_t* out);

/* Dense toolkit path behind rtucker_sketched_ridge (capi.cpp:324-362). */
int orc_aug_draw(const double* cand, uint64_t n, uint64_t d, double d_eff_lower, uint64_t seed,
                 uint64_t s, uint64_t* idx_out, double* w_out);
int orc_dense_normal_eq(const double* a, uint64_t n, uint64_t d, const double* b, double lambda,
                        uint64_t s, const uint64_t* idx, const double* w, double* g,
                        double* rhs);
int orc_sketched_ridge(const double* a, uint64_t n, uint64_t d, const double* b,
                       const double* candidate_scores, double lambda,
                       double d_eff_lower, double epsilon, double delta,
                       uint64_t sample_count_override, uint64_t seed, double* x_out,
                       uint64_t* sample_count_out, double* beta_prime_out);

/* ---- Kronecker product design (src/core/kronecker.cpp) ----
 * Per-factor classical scores, score CDF and score sum, exactly as the
 * ImplicitKronecker constructor builds them (kronecker.cpp:9-35).
 * scores/cdf: length rows; *sum_out = last CDF entry; *rank_out = SVD rank. */
int orc_factor_scores(const double* factor, size_t rows, size_t cols, double* scores,
                      double* cdf, double* sum_out, size_t* rank_out);

/* Draws s rows of the augmented Kronecker design with ProductLeverageSampler
 * (kronecker.cpp:159-181) driven by SplitMix64(seed) as in
 * solve_sketched_ridge (sketch_ridge.cpp:80-90). scores/cdfs/sums are per mode
 * and concatenated (mode n starts at offset sum_{m<n} rows[m]).
 * Outputs: indices[s] in [0, prod rows + d), weights[s]; *u64_used_out = the
 * number of next_u64 calls consumed (the stream length). */
int orc_kron_draw(uint32_t order, const uint64_t* rows, uint64_t d,
                  const double* scores_cat, const double* cdf_cat, const double* sums,
                  uint64_t seed, uint64_t s, uint64_t* indices, double* weights,
                  uint64_t* u64_used_out);

/* Sketched normal equations from a factored sketch of the augmented Kronecker
 * design (sketch_ridge.cpp:105-128): gram d x d (full, mirrored), rhs d.
 * factors_cat: factor n row-major (rows[n] x ranks[n]) concatenated. */
int orc_kron_sketch_normal_eq(uint32_t order, const uint64_t* rows,
                              const uint64_t* ranks, const double* factors_cat,
                              const double* xvec, double lambda, uint64_t s,
                              const uint64_t* indices, const double* weights,
                              double* gram, double* rhs);

/* x = gram^+ rhs through the Jacobi SVD (sketch_ridge.cpp:130-139).
 * *rank_out = numerical rank of gram. */
int orc_pinv_solve(const double* gram, const double* rhs, size_t d, double* x,
                   size_t* rank_out);

/* ---- Tucker (src/core/tucker.cpp) ----
 * A model is (core R_1..R_N, factors I_n x R_n concatenated). */
int orc_reconstruct(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                    const double* core, const double* factors_cat, double* xhat);
int orc_tucker_loss(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                    const double* core, const double* factors_cat, double lambda,
                    const double* x, double* loss_out, double* rmse_out);
/* Overwrites factor `mode` (1-based) in factors_cat (tucker.cpp:70-89). */
int orc_update_factor(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                      const double* core, double* factors_cat, double lambda,
                      const double* x, uint32_t mode);
int orc_update_core_exact(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                          const double* core, const double* factors_cat, double lambda,
                          const double* x, double* core_out);
/* Sketched core (tucker.cpp:141-166). Optional outputs (NULL to skip):
 * indices/weights[s] of the sketch, *rank_deficient_out. */
int orc_update_core_fast(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                         const double* core, const double* factors_cat, double lambda,
                         const double* x, uint64_t s_override, double epsilon,
                         double delta, uint64_t seed, double* core_out,
                         uint64_t* indices, double* weights, int* rank_deficient_out,
                         uint64_t* s_out);
/* Uniform [0,1) init, core first then factors (tucker.cpp:168-190). */
int orc_random_model(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                     uint64_t seed, double* core, double* factors_cat);

/* Full ALS (tucker.cpp:192-276) with the C-API option semantics
 * (capi.cpp:176-201). history arrays are sized max_iterations*(order+1) and
 * filled with *history_len_out rows (step code: n for "F(n+1)", order = "Core").
 * core/factors receive the final model. core_seeds_out (optional, length
 * max_iterations) receives the per-sweep sketch seed. */
typedef struct {
  double lambda;
  int sketched_core;
  double epsilon;
  double delta;
  uint64_t seed;
  uint32_t max_iterations;
  double tolerance;
  uint64_t sample_count_override;
  int record_history;
} orc_als_options;

int orc_als(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
            const double* x, const orc_als_options* opts, double* core,
            double* factors_cat, uint32_t* history_iter, int* history_step,
            double* history_loss, double* history_rmse, uint64_t* history_len_out,
            uint32_t* iterations_out, double* final_loss, double* final_rmse,
            uint64_t* core_seeds_out);

/* Perf mode (not in the reference; parity unpinned): sketched factor update and
 * ALS with it. See rtucker_oracle.c. */
int orc_update_factor_sketched(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
                               const double* core, double* factors_cat, double lambda,
                               const double* x, uint32_t mode, uint64_t s, uint64_t seed,
                               uint64_t* indices_out, double* weights_out);
int orc_als_fs(uint32_t order, const uint64_t* shape, const uint64_t* ranks,
               const double* x, const orc_als_options* opts, uint64_t factor_samples,
               double* core, double* factors_cat, uint32_t* history_iter, int* history_step,
               double* history_loss, double* history_rmse, uint64_t* history_len_out,
               uint32_t* iterations_out, double* final_loss, double* final_rmse,
               uint64_t* core_seeds_out);

#ifdef __cplusplus
}
#endif
#endif /* RTUCKER_ORACLE_H */
