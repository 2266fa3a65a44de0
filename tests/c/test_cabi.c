/* Compiled C client of include/cpfit_gpu.h (built by __graft_entry__.build() into
 * tests/c/_build/test_cabi; run by tests/test_cabi_c.py). Proves the header is plain C and
 * that the reference's entry points work through it with no Python in between:
 *   - cpfit_tensor_create_dense + cpfit_mttkrp on the reference's known answer
 *     (test_tensor.cpp:122-127: 2x2x2 ones tensor, unit factors -> [[4],[4]]);
 *   - cpfit_objective_and_gradient at an exact fit (test_kruskal.cpp:95-101: g = 0, f = 0);
 *   - cpfit_ngmres_solve on a rank-2 tensor built from known factors (converges, stop GradTol);
 *   - cpfit_tensor_create_coo with a duplicate, an explicit zero and an out-of-range coordinate
 *     (tensor.cpp:56-103: duplicates summed, zeros dropped, out-of-range -> invalid_argument).
 * Exit code 0 on success; with no visible GPU, 0 if the first device call fails loudly with
 * status 3 (no CPU fallback) and "--expect-gpu" was not given. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "cpfit_gpu.h"

static int fails = 0;
#define CHECK(c, ...)                          \
    do {                                       \
        if (!(c)) {                            \
            fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
            fprintf(stderr, __VA_ARGS__);      \
            fprintf(stderr, "\n");             \
            ++fails;                           \
        }                                      \
    } while (0)

int main(int argc, char** argv) {
    const int expect_gpu = argc > 1 && strcmp(argv[1], "--expect-gpu") == 0;
    const int64_t d2[3] = {2, 2, 2};
    double ones[8];
    for (int i = 0; i < 8; ++i) ones[i] = 1.0;
    cpfit_tensor t = NULL;
    int rc = cpfit_tensor_create_dense(3, d2, ones, &t);
    if (cpfit_device_count() < 1) {
        if (expect_gpu) {
            fprintf(stderr, "no GPU visible\n");
            return 1;
        }
        CHECK(rc == 3, "create without a GPU returned %d (expected 3: CUDA failure, no CPU fallback)", rc);
        printf("no GPU: device entry points fail loudly (status %d: %s)\n", rc, cpfit_last_error());
        return fails ? 1 : 0;
    }
    CHECK(rc == 0, "create_dense: %s", cpfit_last_error());
    /* mttkrp of the ones tensor with unit rank-1 factors: every entry sums 4 ones */
    double u[6] = {1, 1, 1, 1, 1, 1}, m[2];
    for (int mode = 0; mode < 3; ++mode) {
        rc = cpfit_mttkrp(t, 1, u, mode, m);
        CHECK(rc == 0 && m[0] == 4.0 && m[1] == 4.0, "mttkrp mode %d: rc %d, [%g, %g]", mode, rc, m[0], m[1]);
    }
    /* exact fit: T = [[a, b, c]] with a = b = c = (1, 1) -> f = 0, g = 0 */
    double g[6], f = -1.0;
    rc = cpfit_objective_and_gradient(t, 1, u, g, &f);
    CHECK(rc == 0 && fabs(f) <= 1e-14, "objective at exact fit: rc %d f %g", rc, f);
    for (int i = 0; i < 6; ++i) CHECK(fabs(g[i]) <= 1e-13, "gradient[%d] = %g at exact fit", i, g[i]);
    rc = cpfit_mttkrp(t, 1, u, 3, m);
    CHECK(rc == 1, "mode out of range returned %d (expected 1: invalid_argument)", rc);
    cpfit_tensor_destroy(t);

    /* rank-2 tensor 6x5x4 from fixed factors; N-GMRES from a perturbed start */
    const int64_t d3[3] = {6, 5, 4};
    const int R = 2, nu = (6 + 5 + 4) * 2;
    double truth[30], start[30], T[120];
    for (int i = 0; i < nu; ++i) truth[i] = 0.5 + 0.5 * sin(1.0 + 0.7 * i);
    for (int i = 0; i < nu; ++i) start[i] = truth[i] * (1.0 + 0.2 * cos(0.3 * i));
    for (int k = 0; k < 4; ++k)
        for (int j = 0; j < 5; ++j)
            for (int i = 0; i < 6; ++i) {
                double s = 0.0;
                for (int r = 0; r < R; ++r) s += truth[i + 6 * r] * truth[12 + j + 5 * r] * truth[22 + k + 4 * r];
                T[i + 6 * (j + 5 * k)] = s;
            }
    rc = cpfit_tensor_create_dense(3, d3, T, &t);
    CHECK(rc == 0, "create_dense 6x5x4: %s", cpfit_last_error());
    cpfit_ngmres_options o;
    cpfit_default_ngmres_options(&o);
    o.max_iters = 500;
    o.tol_grad = 1e-10;
    double best[30], fbest = -1.0;
    cpfit_trace_row rows[501];
    int64_t nrows = 0;
    int stop = -1;
    rc = cpfit_ngmres_solve(t, R, start, &o, best, &fbest, rows, 501, &nrows, &stop);
    CHECK(rc == 0, "ngmres_solve: %s", cpfit_last_error());
    CHECK(stop == 0, "stop reason %d (expected 0 GradTol)", stop);
    CHECK(nrows >= 2 && rows[0].iter == 0 && rows[nrows - 1].iter == nrows - 1, "trace rows %lld", (long long)nrows);
    CHECK(fbest <= 1e-16, "final f %g", fbest);
    printf("ngmres_solve: %lld iterations, f = %.3e, stop %d\n", (long long)(nrows - 1), fbest, stop);
    cpfit_tensor_destroy(t);

    /* COO canonicalisation through the ABI */
    const int64_t dc[3] = {3, 3, 3};
    int64_t coords[12] = {0, 1, 2, 0, 1, 2, 2, 2, 2, 1, 0, 0}; /* (0,1,2) twice, (2,2,2), (1,0,0) */
    double vals[4] = {1.5, 2.5, 0.0, 3.0};
    int64_t nnz = -1;
    rc = cpfit_tensor_create_coo(3, dc, 4, coords, vals, &t);
    CHECK(rc == 0, "create_coo: %s", cpfit_last_error());
    cpfit_tensor_nnz(t, &nnz);
    CHECK(nnz == 2, "canonical nnz %lld (expected 2: duplicate summed, zero dropped)", (long long)nnz);
    double un[9] = {1, 1, 1, 1, 1, 1, 1, 1, 1}, m0[3];
    rc = cpfit_mttkrp(t, 1, un, 0, m0);
    CHECK(rc == 0 && m0[0] == 4.0 && m0[1] == 3.0 && m0[2] == 0.0, "sparse mttkrp [%g %g %g]", m0[0], m0[1], m0[2]);
    cpfit_tensor_destroy(t);
    coords[0] = 3; /* out of range */
    rc = cpfit_tensor_create_coo(3, dc, 4, coords, vals, &t);
    CHECK(rc == 1, "out-of-range coordinate returned %d (expected 1)", rc);
    vals[0] = NAN;
    coords[0] = 0;
    rc = cpfit_tensor_create_coo(3, dc, 4, coords, vals, &t);
    CHECK(rc == 1, "non-finite value returned %d (expected 1)", rc);
    T[7] = INFINITY;
    rc = cpfit_tensor_create_dense(3, d3, T, &t);
    CHECK(rc == 1, "non-finite dense value returned %d (expected 1)", rc);
    printf(fails ? "FAILED (%d)\n" : "all C-ABI checks passed\n", fails);
    return fails ? 1 : 0;
}
