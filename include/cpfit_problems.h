/*
 * cpfit_problems.h — synthetic inputs for the cpfit B200 path (libcpfit_gpu.so, host code).
 * Restates proj/core/include/cpfit/problems.hpp + rng.hpp (problems.cpp:24-145) and adds the
 * BASELINE.json generators (N-way collinear factors, l/100 noise scaling, random COO).
 * Not on the timed path: inputs are generated on the host, then uploaded once.
 */
#ifndef CPFIT_PROBLEMS_H
#define CPFIT_PROBLEMS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
const char* cpfit_problems_last_error(void);
/* Rng (rng.hpp:18-48): first n raw / uniform / normal draws of Rng(seed) (any may be NULL) */
int cpfit_rng_draws(uint64_t seed, int64_t n, uint64_t* out_u64, double* out_uniform, double* out_normal);
uint64_t cpfit_rng_mix(uint64_t x);
/* collinear_factors (problems.hpp:41) generalised to N modes / per-mode sizes; out in pack() layout */
int cpfit_collinear_factors(int order, const int64_t* dims, int64_t rank, double c, uint64_t seed, double* out);
/* full(K) (kruskal.hpp:31) */
int cpfit_full(int order, const int64_t* dims, int64_t rank, const double* u, double* out);
/* dense_test_problem (problems.hpp:54); noise_mode 0 = reference (100/l-1)^(-1/2), 1 = BASELINE l/100 */
int cpfit_dense_test_problem(int order, const int64_t* dims, int64_t rank, double c, double l1, double l2,
                             uint64_t seed, int noise_mode, double* t_out, double* truth_out, double* noise_free_out);
/* uniform_initial_guess (problems.hpp:66) */
int cpfit_uniform_initial_guess(int order, const int64_t* dims, int64_t rank, uint64_t seed, double* out);
/* laplacian_tensor (problems.hpp:60); pass NULL buffers to query *nnz_out */
int cpfit_laplacian_tensor(int d, int64_t s, int64_t* coords, double* values, int64_t* nnz_out);
/* BASELINE config 4 random COO problem (sorted lexicographically, distinct coordinates) */
int cpfit_random_sparse_problem(int order, const int64_t* dims, int64_t nnz, int64_t rank, double noise,
                                uint64_t seed, int64_t* coords, double* values, double* truth_out);
#ifdef __cplusplus
}
#endif
#endif
