// Synthetic problem generators (host input side; not on the timed path).
//
// Restates proj/core/src/problems.cpp and include/cpfit/rng.hpp, generalised as BASELINE.json
// requires:
//   * Rng: std::mt19937_64; uniform = top 53 bits * 2^-53; normal = Box–Muller cosine branch,
//     two draws per variate (rng.hpp:18-48); mix = splitmix64 finaliser.
//   * collinear factors: per mode, uniform I_n x R (column-major fill), thin Householder QR
//     with the R-diagonal made nonnegative, times the upper Cholesky factor of
//     (1-c) I + c 11^T (problems.cpp:40-61), for any order and per-mode sizes.
//   * dense test problem: factors -> T0 = full -> N1 -> N2 from one stream (problems.cpp:63-95);
//     noise scale either the reference's (100/l - 1)^(-1/2) (noise_mode 0) or BASELINE's
//     l/100 (noise_mode 1); N2 is drawn even when l2 = 0 so streams match.
//   * uniform_initial_guess: U[0,1] in pack order from Rng(mix(seed)) (problems.cpp:137-145).
//   * laplacian_tensor (problems.cpp:97-135) and the BASELINE random-COO problem.
#include "../../include/cpfit_problems.h"

#include <parallel/algorithm>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_perr;

struct Rng {
    std::mt19937_64 e;
    explicit Rng(uint64_t s) : e(s) {}
    double uniform() { return static_cast<double>(e() >> 11) * 0x1.0p-53; }
    double normal() {
        const double u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log1p(-u1));
        return r * std::cos(2.0 * 3.141592653589793238462643383279502884 * u2);
    }
    static uint64_t mix(uint64_t x) {
        x += 0x9e3779b97f4a7c15ull;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
        return x ^ (x >> 31);
    }
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_perr = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_perr = e.what();
        return 3;
    }
}

void require(bool c, const char* w) {
    if (!c) throw std::invalid_argument(w);
}

double vnorm(const double* x, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * x[i];
    return std::sqrt(s);
}

// ||x|| for large vectors: fixed 64K-element chunks summed on all cores, the chunk sums added
// in order (the result does not depend on the thread count)
double pnorm(const double* x, int64_t n) {
    constexpr int64_t CH = 1 << 16;
    const int64_t nch = (n + CH - 1) / CH;
    std::vector<double> part((size_t)std::max<int64_t>(nch, 1), 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nch; ++c) {
        double s = 0.0;
        const int64_t e = std::min(n, (c + 1) * CH);
        for (int64_t i = c * CH; i < e; ++i) s += x[i] * x[i];
        part[(size_t)c] = s;
    }
    double s = 0.0;
    for (double v : part) s += v;
    return std::sqrt(s);
}

// n normals of rng in stream order (Rng::normal: two engine draws each, rng.hpp:26-33). The
// engine is serial (~1 ns per draw) and runs ahead into a buffer; the Box–Muller transforms
// (log1p, sqrt, cos: the expensive part) run on all cores.
void normals(Rng& rng, double* out, int64_t n) {
    constexpr int64_t CH = 1 << 22;
    std::vector<uint64_t> raw((size_t)(2 * std::min<int64_t>(n, CH)));
    for (int64_t k0 = 0; k0 < n; k0 += CH) {
        const int64_t m = std::min(CH, n - k0);
        for (int64_t i = 0; i < 2 * m; ++i) raw[(size_t)i] = rng.e();
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            const double u1 = static_cast<double>(raw[(size_t)(2 * i)] >> 11) * 0x1.0p-53;
            const double u2 = static_cast<double>(raw[(size_t)(2 * i + 1)] >> 11) * 0x1.0p-53;
            const double r = std::sqrt(-2.0 * std::log1p(-u1));
            out[k0 + i] = r * std::cos(2.0 * 3.141592653589793238462643383279502884 * u2);
        }
    }
}

// Thin Householder QR of a (rows x k, column-major): returns Q (rows x k) with the sign fix
// R(j,j) >= 0 (problems.cpp:52-56).
std::vector<double> thin_q(const std::vector<double>& a, int64_t rows, int64_t k) {
    std::vector<double> qr = a;
    std::vector<double> tau((size_t)k, 0.0), rdiag((size_t)k, 0.0);
    for (int64_t j = 0; j < k; ++j) {
        double* col = qr.data() + j * rows;
        double tail = 0.0;
        for (int64_t i = j + 1; i < rows; ++i) tail += col[i] * col[i];
        const double c0 = col[j];
        double t, beta;
        if (tail <= std::numeric_limits<double>::min()) {
            t = 0.0;
            beta = c0;
            for (int64_t i = j + 1; i < rows; ++i) col[i] = 0.0;
        } else {
            beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            for (int64_t i = j + 1; i < rows; ++i) col[i] /= (c0 - beta);
            t = (beta - c0) / beta;
        }
        col[j] = beta;
        tau[(size_t)j] = t;
        rdiag[(size_t)j] = beta;
        for (int64_t c = j + 1; c < k; ++c) {
            double* cc = qr.data() + c * rows;
            if (t == 0.0) continue;
            double s = cc[j];
            for (int64_t i = j + 1; i < rows; ++i) s += col[i] * cc[i];
            cc[j] -= t * s;
            for (int64_t i = j + 1; i < rows; ++i) cc[i] -= t * col[i] * s;
        }
    }
    // Q = H_0 ... H_{k-1} applied to the first k identity columns
    std::vector<double> q((size_t)(rows * k), 0.0);
    for (int64_t c = 0; c < k; ++c) {
        double* x = q.data() + c * rows;
        x[c] = 1.0;
        for (int64_t j = k - 1; j >= 0; --j) {
            const double t = tau[(size_t)j];
            if (t == 0.0) continue;
            const double* v = qr.data() + j * rows;
            double s = x[j];
            for (int64_t i = j + 1; i < rows; ++i) s += v[i] * x[i];
            x[j] -= t * s;
            for (int64_t i = j + 1; i < rows; ++i) x[i] -= t * v[i] * s;
        }
        if (rdiag[(size_t)c] < 0.0)
            for (int64_t i = 0; i < rows; ++i) x[i] = -x[i];
    }
    return q;
}

// Upper Cholesky factor U (U^T U = K) of K = (1-c) I + c 11^T.
std::vector<double> collin_chol(int64_t R, double c) {
    std::vector<double> l((size_t)(R * R), 0.0);  // lower, row-major
    auto K = [&](int64_t i, int64_t j) { return i == j ? 1.0 : c; };
    for (int64_t k = 0; k < R; ++k) {
        double x = K(k, k);
        for (int64_t j = 0; j < k; ++j) x -= l[(size_t)(k * R + j)] * l[(size_t)(k * R + j)];
        x = std::sqrt(x);
        l[(size_t)(k * R + k)] = x;
        for (int64_t i = k + 1; i < R; ++i) {
            double s = K(i, k);
            for (int64_t j = 0; j < k; ++j) s -= l[(size_t)(i * R + j)] * l[(size_t)(k * R + j)];
            l[(size_t)(i * R + k)] = s / x;
        }
    }
    std::vector<double> u((size_t)(R * R), 0.0);  // column-major U = L^T
    for (int64_t i = 0; i < R; ++i)
        for (int64_t j = 0; j <= i; ++j) u[(size_t)(i * R + j)] = l[(size_t)(i * R + j)];  // U(j,i) = L(i,j)
    return u;
}

void collinear(int order, const int64_t* dims, int64_t R, double c, Rng& rng, double* out) {
    require(c >= 0.0 && c < 1.0, "collinear_factors: collinearity must be in [0, 1)");
    const std::vector<double> U = collin_chol(R, c);
    int64_t at = 0;
    for (int n = 0; n < order; ++n) {
        const int64_t s = dims[n];
        require(R >= 1 && s >= R, "collinear_factors: need s >= rank >= 1");
        std::vector<double> raw((size_t)(s * R));
        for (int64_t col = 0; col < R; ++col)
            for (int64_t r = 0; r < s; ++r) raw[(size_t)(r + col * s)] = rng.uniform();
        const std::vector<double> q = thin_q(raw, s, R);
        for (int64_t j = 0; j < R; ++j)
            for (int64_t i = 0; i < s; ++i) {
                double v = 0.0;
                for (int64_t k = 0; k <= j; ++k) v += q[(size_t)(i + k * s)] * U[(size_t)(k + j * R)];
                out[at + i + j * s] = v;
            }
        at += s * R;
    }
}

// full(K): element (i_0..i_{N-1}) = sum_r prod_n A_n(i_n, r), first mode fastest.
void full_tensor(int order, const int64_t* dims, int64_t R, const double* u, double* out) {
    int64_t K = 1;
    for (int n = 0; n < order; ++n) K *= dims[n];
    std::vector<int64_t> off((size_t)order, 0);
    for (int n = 1; n < order; ++n) off[(size_t)n] = off[(size_t)n - 1] + dims[n - 1] * R;
    const int64_t I0 = dims[0];
    const int64_t J = K / I0;
#pragma omp parallel for schedule(static)
    for (int64_t f = 0; f < J; ++f) {
        std::vector<double> w((size_t)R);
        int64_t rem = f;
        for (int64_t r = 0; r < R; ++r) w[(size_t)r] = 1.0;
        for (int n = 1; n < order; ++n) {
            const int64_t j = rem % dims[n];
            rem /= dims[n];
            for (int64_t r = 0; r < R; ++r) w[(size_t)r] *= u[off[(size_t)n] + j + r * dims[n]];
        }
        for (int64_t i = 0; i < I0; ++i) {
            double s = 0.0;
            for (int64_t r = 0; r < R; ++r) s += u[i + r * I0] * w[(size_t)r];
            out[f * I0 + i] = s;
        }
    }
}

double noise_coef(double l, int mode) { return mode == 0 ? std::pow(100.0 / l - 1.0, -0.5) : l / 100.0; }

}  // namespace

extern "C" {

const char* cpfit_problems_last_error(void) { return g_perr.c_str(); }

int cpfit_rng_draws(uint64_t seed, int64_t n, uint64_t* out_u64, double* out_uniform, double* out_normal) {
    return guard([&] {
        if (out_u64) {
            Rng r(seed);
            for (int64_t i = 0; i < n; ++i) out_u64[i] = r.e();
        }
        if (out_uniform) {
            Rng r(seed);
            for (int64_t i = 0; i < n; ++i) out_uniform[i] = r.uniform();
        }
        if (out_normal) {
            Rng r(seed);
            for (int64_t i = 0; i < n; ++i) out_normal[i] = r.normal();
        }
    });
}

uint64_t cpfit_rng_mix(uint64_t x) { return Rng::mix(x); }

int cpfit_collinear_factors(int order, const int64_t* dims, int64_t rank, double c, uint64_t seed, double* out) {
    return guard([&] {
        Rng rng(seed);
        collinear(order, dims, rank, c, rng, out);
    });
}

int cpfit_full(int order, const int64_t* dims, int64_t rank, const double* u, double* out) {
    return guard([&] { full_tensor(order, dims, rank, u, out); });
}

int cpfit_dense_test_problem(int order, const int64_t* dims, int64_t rank, double c, double l1, double l2,
                             uint64_t seed, int noise_mode, double* t_out, double* truth_out, double* noise_free_out) {
    return guard([&] {
        require(l1 >= 0.0 && l1 < 100.0 && l2 >= 0.0 && l2 < 100.0,
                "dense_test_problem: noise levels must be in [0, 100)");
        Rng rng(seed);
        int64_t nu = 0, K = 1;
        for (int n = 0; n < order; ++n) {
            nu += dims[n] * rank;
            K *= dims[n];
        }
        std::vector<double> truth((size_t)nu);
        collinear(order, dims, rank, c, rng, truth.data());
        full_tensor(order, dims, rank, truth.data(), t_out);
        if (noise_free_out) std::memcpy(noise_free_out, t_out, sizeof(double) * (size_t)K);
        if (truth_out) std::memcpy(truth_out, truth.data(), sizeof(double) * (size_t)nu);
        std::vector<double> n1((size_t)K), n2((size_t)K);
        normals(rng, n1.data(), K);
        normals(rng, n2.data(), K);  // drawn even when l2 = 0 (problems.cpp:74)
        if (l1 > 0.0) {
            const double coef = noise_coef(l1, noise_mode);
            const double s = coef * pnorm(t_out, K) / pnorm(n1.data(), K);
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < K; ++i) t_out[i] += s * n1[(size_t)i];
        }
        if (l2 > 0.0) {
            const double coef = noise_coef(l2, noise_mode);
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < K; ++i) n2[(size_t)i] *= t_out[i];  // mixed = N2 .* T_hat
            const double s = coef * pnorm(t_out, K) / pnorm(n2.data(), K);
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < K; ++i) t_out[i] += s * n2[(size_t)i];
        }
    });
}

int cpfit_uniform_initial_guess(int order, const int64_t* dims, int64_t rank, uint64_t seed, double* out) {
    return guard([&] {
        require(rank >= 1, "uniform_initial_guess: rank must be >= 1");
        Rng rng(Rng::mix(seed));
        int64_t at = 0;
        for (int n = 0; n < order; ++n) {
            for (int64_t c = 0; c < rank; ++c)
                for (int64_t r = 0; r < dims[n]; ++r) out[at + r + c * dims[n]] = rng.uniform();
            at += dims[n] * rank;
        }
    });
}

// problems.cpp:97-135. coords: nnz x 2d (AoS), values nnz; *nnz_out = s^d + 2 d s^(d-1)(s-1).
int cpfit_laplacian_tensor(int d, int64_t s, int64_t* coords, double* values, int64_t* nnz_out) {
    return guard([&] {
        require(d >= 1, "laplacian_tensor: dimension must be >= 1");
        require(s >= 2, "laplacian_tensor: grid size must be >= 2");
        std::vector<int64_t> grid((size_t)d, 0);
        int64_t cnt = 0;
        auto emit = [&](const std::vector<int64_t>& x, const std::vector<int64_t>& y, double v) {
            if (coords) {
                for (int k = 0; k < d; ++k) coords[cnt * 2 * d + k] = x[(size_t)k];
                for (int k = 0; k < d; ++k) coords[cnt * 2 * d + d + k] = y[(size_t)k];
            }
            if (values) values[cnt] = v;
            ++cnt;
        };
        bool more = true;
        while (more) {
            emit(grid, grid, 2.0 * d);
            for (int k = 0; k < d; ++k) {
                if (grid[(size_t)k] + 1 < s) {
                    std::vector<int64_t> nb = grid;
                    ++nb[(size_t)k];
                    emit(grid, nb, -1.0);
                    emit(nb, grid, -1.0);
                }
            }
            more = false;
            for (int k = 0; k < d; ++k) {
                if (++grid[(size_t)k] < s) {
                    more = true;
                    break;
                }
                grid[(size_t)k] = 0;
            }
        }
        *nnz_out = cnt;
    });
}

// BASELINE config 4: nnz distinct uniform coordinates (draw, sort, unique, redraw), values =
// rank-R model with U[0,1] unit-normalised factors + noise: v = m + noise * ||m|| / ||z|| * z.
// Draw order from Rng(seed): factors (pack order), coordinates (N draws each, modulo the mode
// size), redraws, then z (nnz normals in sorted order).
int cpfit_random_sparse_problem(int order, const int64_t* dims, int64_t nnz, int64_t rank, double noise,
                                uint64_t seed, int64_t* coords, double* values, double* truth_out) {
    return guard([&] {
        require(order >= 1 && nnz >= 0 && rank >= 1, "random_sparse_problem: bad arguments");
        Rng rng(seed);
        int64_t nu = 0;
        for (int n = 0; n < order; ++n) nu += dims[n] * rank;
        std::vector<double> u((size_t)nu);
        int64_t at = 0;
        for (int n = 0; n < order; ++n) {
            for (int64_t c = 0; c < rank; ++c) {
                double* col = u.data() + at + c * dims[n];
                for (int64_t r = 0; r < dims[n]; ++r) col[r] = rng.uniform();
                const double nr = vnorm(col, dims[n]);
                for (int64_t r = 0; r < dims[n]; ++r) col[r] /= nr;
            }
            at += dims[n] * rank;
        }
        if (truth_out) std::memcpy(truth_out, u.data(), sizeof(double) * (size_t)nu);
        const size_t N = (size_t)order;
        std::vector<int64_t> lin;  // linear index (first mode fastest) for sort/unique
        std::vector<int64_t> strides(N, 1);
        for (size_t n = 1; n < N; ++n) strides[n] = strides[n - 1] * dims[n - 1];
        auto draw = [&]() {
            int64_t l = 0;
            for (size_t n = 0; n < N; ++n) l += (int64_t)(rng.e() % (uint64_t)dims[n]) * strides[n];
            return l;
        };
        // lexicographic order of (i_0, ..., i_{N-1}) == order of the reversed-stride key
        auto key = [&](int64_t l) {
            int64_t k = 0, mult = 1;
            for (int64_t n = (int64_t)N - 1; n >= 0; --n) {
                const int64_t idx = (l / strides[(size_t)n]) % dims[n];
                k += idx * mult;
                mult *= dims[n];
            }
            return k;
        };
        std::vector<int64_t> keys;
        keys.reserve((size_t)nnz);
        for (int64_t i = 0; i < nnz; ++i) keys.push_back(key(draw()));
        for (;;) {
            __gnu_parallel::sort(keys.begin(), keys.end());
            keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
            if ((int64_t)keys.size() == nnz) break;
            const int64_t miss = nnz - (int64_t)keys.size();
            for (int64_t i = 0; i < miss; ++i) keys.push_back(key(draw()));
        }
        std::vector<int64_t> off(N, 0);
        for (size_t n = 1; n < N; ++n) off[n] = off[n - 1] + dims[n - 1] * rank;
        std::vector<double> m((size_t)nnz);
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < nnz; ++i) {
            int64_t k = keys[(size_t)i];
            int64_t idx[16];
            for (int64_t n = (int64_t)N - 1; n >= 0; --n) {
                idx[(size_t)n] = k % dims[n];
                k /= dims[n];
            }
            double s = 0.0;
            for (int64_t r = 0; r < rank; ++r) {
                double p = 1.0;
                for (size_t n = 0; n < N; ++n) p *= u[(size_t)(off[n] + idx[n] + r * dims[n])];
                s += p;
            }
            m[(size_t)i] = s;
            for (size_t n = 0; n < N; ++n) coords[(size_t)i * N + n] = idx[n];
        }
        std::vector<double> z((size_t)nnz);
        normals(rng, z.data(), nnz);
        const double sc = (nnz > 0) ? noise * pnorm(m.data(), nnz) / pnorm(z.data(), nnz) : 0.0;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < nnz; ++i) values[i] = m[(size_t)i] + sc * z[(size_t)i];
    });
}

}  // extern "C"
