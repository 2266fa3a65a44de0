// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp). Input generators for the CPU side of the
// parity tests and bench.py's reference arm, so that neither needs the product library.
//
// Restates proj/core/include/cpfit/rng.hpp:18-48 (Rng) and proj/core/src/problems.cpp:24-145
// (uniform_matrix, normal_values, collinear_factors, dense_test_problem, uniform_initial_guess),
// with the BASELINE.json deltas SURVEY.md Appendix A asks for: collinear factors for any order
// and per-mode sizes (the reference hard-codes three cubic factors, problems.cpp:51), the noise
// scale l/100 besides the reference's (100/l - 1)^(-1/2) (problems.cpp:83, :88), and the
// BASELINE config-4 random COO problem (not in the reference; BASELINE.json configs[4]).
// Single-threaded, in the reference's draw order.
#include "oracle.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <string>

namespace oracle {
namespace {

// rng.hpp:18-48
class Rng {
public:
    explicit Rng(std::uint64_t seed) : engine_(seed) {}
    double uniform() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
    double normal() {
        const double u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log1p(-u1));
        return r * std::cos(2.0 * kPi * u2);
    }
    std::uint64_t next_u64() { return engine_(); }
    static std::uint64_t mix(std::uint64_t x) {
        x += 0x9e3779b97f4a7c15ull;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
        return x ^ (x >> 31);
    }

private:
    static constexpr double kPi = 3.141592653589793238462643383279502884;
    std::mt19937_64 engine_;
};

void require(bool c, const char* what) {
    if (!c) throw std::invalid_argument(what);
}

// problems.cpp:24-30 (column-major fill order)
Matrix uniform_matrix(index_t rows, index_t cols, Rng& rng) {
    Matrix m(rows, cols);
    for (index_t c = 0; c < cols; ++c)
        for (index_t r = 0; r < rows; ++r) m(r, c) = rng.uniform();
    return m;
}

// Eigen HouseholderQR(raw).householderQ() * Identity(s, rank) with the sign fix R(j,j) >= 0
// (problems.cpp:52-56): reflectors from make_householder, Q applied as H_0 ... H_{k-1} to the
// first k identity columns (last reflector first).
Matrix thin_q_signed(Matrix a) {
    const index_t rows = a.rows, k = a.cols;
    std::vector<double> tau(static_cast<size_t>(k)), rdiag(static_cast<size_t>(k));
    for (index_t j = 0; j < k; ++j) {
        double t = 0.0, beta = 0.0;
        make_householder(a.col(j) + j, rows - j, t, beta);
        a(j, j) = beta;
        tau[static_cast<size_t>(j)] = t;
        rdiag[static_cast<size_t>(j)] = beta;
        apply_householder_left(a, j, rows - j, j + 1, k, a.col(j) + j + 1, t);
    }
    Matrix q(rows, k);
    for (index_t c = 0; c < k; ++c) q(c, c) = 1.0;
    for (index_t j = k - 1; j >= 0; --j) apply_householder_left(q, j, rows - j, 0, k, a.col(j) + j + 1, tau[static_cast<size_t>(j)]);
    for (index_t j = 0; j < k; ++j)
        if (rdiag[static_cast<size_t>(j)] < 0.0)
            for (index_t i = 0; i < rows; ++i) q(i, j) = -q(i, j);
    return q;
}

// problems.cpp:40-61 for any order / per-mode sizes (BASELINE configs[3] is 4-way).
std::vector<Matrix> collinear_factors(const std::vector<index_t>& dims, index_t rank, double c, Rng& rng) {
    require(c >= 0.0 && c < 1.0, "collinear_factors: collinearity must be in [0, 1)");
    Matrix collin(rank, rank, c);
    for (index_t i = 0; i < rank; ++i) collin(i, i) = 1.0;
    const Matrix chol = LLT(collin).matrix_u();  // C^T C = K
    std::vector<Matrix> out;
    for (index_t s : dims) {
        require(rank >= 1 && s >= rank, "collinear_factors: need s >= rank >= 1");
        const Matrix q = thin_q_signed(uniform_matrix(s, rank, rng));
        out.push_back(matmul(q, chol));
    }
    return out;
}

double noise_coef(double l, int mode) { return mode == 0 ? std::pow(100.0 / l - 1.0, -0.5) : l / 100.0; }

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

}  // namespace
}  // namespace oracle

using namespace oracle;

extern "C" {

const char* oracle_problems_last_error() { return oracle::g_err.c_str(); }

// problems.cpp:63-95. noise_mode 0: the reference's (100/l - 1)^(-1/2); 1: BASELINE's l/100.
// t_out: K values first-mode-fastest; truth_out (may be null): the generating factors, pack order.
int oracle_dense_test_problem(int order, const int64_t* dims, int64_t rank, double c, double l1, double l2,
                              uint64_t seed, int noise_mode, double* t_out, double* truth_out) {
    return oracle::guard([&] {
        require(order >= 1, "dense_test_problem: order must be >= 1");
        require(l1 >= 0.0 && l1 < 100.0 && l2 >= 0.0 && l2 < 100.0,
                "dense_test_problem: noise levels must be in [0, 100)");
        Rng rng(seed);
        std::vector<index_t> d(dims, dims + order);
        KruskalTensor truth(collinear_factors(d, rank, c, rng));
        const DenseTensor noise_free = full(truth);
        const index_t k = noise_free.shape.num_elements();
        std::vector<double> n1(static_cast<size_t>(k)), n2(static_cast<size_t>(k));
        for (auto& x : n1) x = rng.normal();
        for (auto& x : n2) x = rng.normal();  // drawn even when l2 = 0 (problems.cpp:74)
        std::vector<double> t = noise_free.values;
        if (l1 > 0.0) {
            const double s = noise_coef(l1, noise_mode) * norm(t) / norm(n1);
            for (index_t i = 0; i < k; ++i) t[static_cast<size_t>(i)] += s * n1[static_cast<size_t>(i)];
        }
        if (l2 > 0.0) {
            std::vector<double> mixed(static_cast<size_t>(k));
            for (index_t i = 0; i < k; ++i) mixed[static_cast<size_t>(i)] = n2[static_cast<size_t>(i)] * t[static_cast<size_t>(i)];
            const double s = noise_coef(l2, noise_mode) * norm(t) / norm(mixed);
            for (index_t i = 0; i < k; ++i) t[static_cast<size_t>(i)] += s * mixed[static_cast<size_t>(i)];
        }
        std::memcpy(t_out, t.data(), sizeof(double) * static_cast<size_t>(k));
        if (truth_out) {
            const Vector p = pack(truth);
            std::memcpy(truth_out, p.data(), sizeof(double) * p.size());
        }
    });
}

// problems.cpp:137-145: U[0,1] factors in pack order from Rng(mix(seed)).
int oracle_uniform_initial_guess(int order, const int64_t* dims, int64_t rank, uint64_t seed, double* out) {
    return oracle::guard([&] {
        require(rank >= 1, "uniform_initial_guess: rank must be >= 1");
        Rng rng(Rng::mix(seed));
        std::vector<Matrix> f;
        for (int n = 0; n < order; ++n) f.push_back(uniform_matrix(dims[n], rank, rng));
        const Vector p = pack(KruskalTensor(std::move(f)));
        std::memcpy(out, p.data(), sizeof(double) * p.size());
    });
}

// BASELINE.json configs[4]: nnz distinct uniform coordinates, lexicographically sorted; values =
// rank-R model with U[0,1] unit-normalised columns + noise * ||m|| / ||z|| * z. Draw order from
// Rng(seed): factors (pack order, each column normalised), one draw per mode per coordinate
// (modulo the mode size), redraws for the coordinates lost to duplicates, then z in sorted order.
int oracle_random_sparse_problem(int order, const int64_t* dims, int64_t nnz, int64_t rank, double noise,
                                 uint64_t seed, int64_t* coords, double* values) {
    return oracle::guard([&] {
        require(order >= 1 && nnz >= 0 && rank >= 1, "random_sparse_problem: bad arguments");
        Rng rng(seed);
        std::vector<Matrix> f;
        for (int n = 0; n < order; ++n) {
            Matrix a = uniform_matrix(dims[n], rank, rng);
            for (index_t c = 0; c < rank; ++c) {
                const double nr = norm(a.col(c), a.rows);
                for (index_t r = 0; r < a.rows; ++r) a(r, c) /= nr;
            }
            f.push_back(std::move(a));
        }
        // key: lexicographic rank of (i_0, ..., i_{N-1}) (mode 0 most significant)
        auto draw_key = [&] {
            std::vector<index_t> idx(static_cast<size_t>(order));
            for (int n = 0; n < order; ++n) idx[static_cast<size_t>(n)] = static_cast<index_t>(rng.next_u64() % static_cast<uint64_t>(dims[n]));
            index_t key = 0;
            for (int n = 0; n < order; ++n) key = key * dims[n] + idx[static_cast<size_t>(n)];
            return key;
        };
        std::vector<index_t> keys;
        keys.reserve(static_cast<size_t>(nnz));
        for (index_t i = 0; i < nnz; ++i) keys.push_back(draw_key());
        for (;;) {
            std::sort(keys.begin(), keys.end());
            keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
            if (static_cast<index_t>(keys.size()) == nnz) break;
            const index_t miss = nnz - static_cast<index_t>(keys.size());
            for (index_t i = 0; i < miss; ++i) keys.push_back(draw_key());
        }
        std::vector<double> m(static_cast<size_t>(nnz));
        std::vector<index_t> idx(static_cast<size_t>(order));
        for (index_t i = 0; i < nnz; ++i) {
            index_t k = keys[static_cast<size_t>(i)];
            for (int n = order - 1; n >= 0; --n) {
                idx[static_cast<size_t>(n)] = k % dims[n];
                k /= dims[n];
            }
            double s = 0.0;
            for (index_t r = 0; r < rank; ++r) {
                double p = 1.0;
                for (int n = 0; n < order; ++n) p *= f[static_cast<size_t>(n)](idx[static_cast<size_t>(n)], r);
                s += p;
            }
            m[static_cast<size_t>(i)] = s;
            for (int n = 0; n < order; ++n) coords[i * order + n] = idx[static_cast<size_t>(n)];
        }
        std::vector<double> z(static_cast<size_t>(nnz));
        for (auto& x : z) x = rng.normal();
        const double sc = nnz > 0 ? noise * norm(m) / norm(z) : 0.0;
        for (index_t i = 0; i < nnz; ++i) values[i] = m[static_cast<size_t>(i)] + sc * z[static_cast<size_t>(i)];
    });
}

}  // extern "C"
