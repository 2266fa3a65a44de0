// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp). Small dense LA standing in for Eigen.
#include "oracle.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

namespace oracle {

bool Matrix::all_finite() const {
    for (double x : v)
        if (!std::isfinite(x)) return false;
    return true;
}

Matrix matmul(const Matrix& a, const Matrix& b) {
    if (a.cols != b.rows) throw std::invalid_argument("matmul: shape");
    Matrix c(a.rows, b.cols);
    for (index_t j = 0; j < b.cols; ++j)
        for (index_t p = 0; p < a.cols; ++p) {
            const double s = b(p, j);
            const double* ac = a.col(p);
            double* cc = c.col(j);
            for (index_t i = 0; i < a.rows; ++i) cc[i] += ac[i] * s;
        }
    return c;
}

Matrix matmul_tn(const Matrix& a, const Matrix& b) {
    if (a.rows != b.rows) throw std::invalid_argument("matmul_tn: shape");
    Matrix c(a.cols, b.cols);
    for (index_t j = 0; j < b.cols; ++j)
        for (index_t i = 0; i < a.cols; ++i) {
            double s = 0.0;
            const double* ac = a.col(i);
            const double* bc = b.col(j);
            for (index_t p = 0; p < a.rows; ++p) s += ac[p] * bc[p];
            c(i, j) = s;
        }
    return c;
}

double dot(const Vector& a, const Vector& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}

double norm(const double* x, index_t n) {
    double s = 0.0;
    for (index_t i = 0; i < n; ++i) s += x[i] * x[i];
    return std::sqrt(s);
}

double norm(const Vector& a) { return norm(a.data(), static_cast<index_t>(a.size())); }

// Eigen llt_inplace<double, Lower>::unblocked (used for n < 32): column k pivot
// x = a_kk - |L_k,0:k|^2, fail when x <= 0, then scale the column below.
LLT::LLT(const Matrix& a) : l(a) {
    const index_t n = a.rows;
    // Eigen reads only the lower triangle.
    for (index_t j = 0; j < n; ++j)
        for (index_t i = 0; i < j; ++i) l(i, j) = 0.0;
    ok = true;
    for (index_t k = 0; k < n; ++k) {
        double x = l(k, k);
        for (index_t j = 0; j < k; ++j) x -= l(k, j) * l(k, j);
        if (x <= 0.0) {
            ok = false;
            return;
        }
        x = std::sqrt(x);
        l(k, k) = x;
        for (index_t i = k + 1; i < n; ++i) {
            double s = l(i, k);
            for (index_t j = 0; j < k; ++j) s -= l(i, j) * l(k, j);
            l(i, k) = s / x;
        }
    }
}

Matrix LLT::solve(const Matrix& b) const {
    const index_t n = l.rows;
    Matrix x = b;
    for (index_t c = 0; c < b.cols; ++c) {
        double* xc = x.col(c);
        for (index_t i = 0; i < n; ++i) {  // L y = b
            double s = xc[i];
            for (index_t j = 0; j < i; ++j) s -= l(i, j) * xc[j];
            xc[i] = s / l(i, i);
        }
        for (index_t i = n - 1; i >= 0; --i) {  // L^T x = y
            double s = xc[i];
            for (index_t j = i + 1; j < n; ++j) s -= l(j, i) * xc[j];
            xc[i] = s / l(i, i);
        }
    }
    return x;
}

Matrix LLT::matrix_u() const {
    Matrix u(l.cols, l.rows);
    for (index_t i = 0; i < l.rows; ++i)
        for (index_t j = 0; j <= i; ++j) u(j, i) = l(i, j);
    return u;
}

// Eigen MatrixBase::makeHouseholder on x[0..n): returns tau, beta, essential in x[1..n).
void make_householder(double* x, index_t n, double& tau, double& beta) {
    double tail = 0.0;
    for (index_t i = 1; i < n; ++i) tail += x[i] * x[i];
    const double c0 = x[0];
    const double tol = std::numeric_limits<double>::min();
    if (tail <= tol) {
        tau = 0.0;
        beta = c0;
        for (index_t i = 1; i < n; ++i) x[i] = 0.0;
        return;
    }
    beta = std::sqrt(c0 * c0 + tail);
    if (c0 >= 0.0) beta = -beta;
    for (index_t i = 1; i < n; ++i) x[i] /= (c0 - beta);
    tau = (beta - c0) / beta;
}

// Eigen applyHouseholderOnTheLeft: rows r0..r0+n of columns [c0, c1) of m, reflector
// v = [1; ess], I - tau v v^T.
void apply_householder_left(Matrix& m, index_t r0, index_t n, index_t c0, index_t c1,
                            const double* ess, double tau) {
    if (n == 1) {
        for (index_t j = c0; j < c1; ++j) m(r0, j) *= (1.0 - tau);
        return;
    }
    if (tau == 0.0) return;
    for (index_t j = c0; j < c1; ++j) {
        double t = 0.0;
        for (index_t i = 1; i < n; ++i) t += ess[i - 1] * m(r0 + i, j);
        t += m(r0, j);
        m(r0, j) -= tau * t;
        for (index_t i = 1; i < n; ++i) m(r0 + i, j) -= tau * ess[i - 1] * t;
    }
}

// Eigen ColPivHouseholderQR::computeInPlace + _solve_impl (single rhs).
Vector colpiv_qr_solve(const Matrix& a, const Vector& b) {
    const index_t rows = a.rows, cols = a.cols, size = std::min(rows, cols);
    Matrix qr = a;
    std::vector<double> hcoeffs(static_cast<size_t>(size), 0.0);
    std::vector<index_t> transp(static_cast<size_t>(size));
    std::vector<double> upd(static_cast<size_t>(cols)), direct(static_cast<size_t>(cols));
    for (index_t j = 0; j < cols; ++j) {
        direct[static_cast<size_t>(j)] = norm(qr.col(j), rows);
        upd[static_cast<size_t>(j)] = direct[static_cast<size_t>(j)];
    }
    const double eps = std::numeric_limits<double>::epsilon();
    double maxcol = 0.0;
    for (double x : upd) maxcol = std::max(maxcol, x);
    const double threshold_helper = (maxcol * eps) * (maxcol * eps) / static_cast<double>(rows);
    const double downdate_thr = std::sqrt(eps);
    index_t nonzero_pivots = size;
    double maxpivot = 0.0;
    std::vector<index_t> perm(static_cast<size_t>(cols));
    for (index_t j = 0; j < cols; ++j) perm[static_cast<size_t>(j)] = j;
    std::vector<double> ess(static_cast<size_t>(rows));
    for (index_t k = 0; k < size; ++k) {
        index_t big = k;
        for (index_t j = k + 1; j < cols; ++j)
            if (upd[static_cast<size_t>(j)] > upd[static_cast<size_t>(big)]) big = j;
        const double big_sq = upd[static_cast<size_t>(big)] * upd[static_cast<size_t>(big)];
        if (nonzero_pivots == size && big_sq < threshold_helper * static_cast<double>(rows - k))
            nonzero_pivots = k;
        transp[static_cast<size_t>(k)] = big;
        if (k != big) {
            for (index_t i = 0; i < rows; ++i) std::swap(qr(i, k), qr(i, big));
            std::swap(upd[static_cast<size_t>(k)], upd[static_cast<size_t>(big)]);
            std::swap(direct[static_cast<size_t>(k)], direct[static_cast<size_t>(big)]);
        }
        double tau = 0.0, beta = 0.0;
        make_householder(qr.col(k) + k, rows - k, tau, beta);
        qr(k, k) = beta;
        hcoeffs[static_cast<size_t>(k)] = tau;
        if (std::abs(beta) > maxpivot) maxpivot = std::abs(beta);
        for (index_t i = 0; i < rows - k - 1; ++i) ess[static_cast<size_t>(i)] = qr(k + 1 + i, k);
        apply_householder_left(qr, k, rows - k, k + 1, cols, ess.data(), tau);
        for (index_t j = k + 1; j < cols; ++j) {
            double& u = upd[static_cast<size_t>(j)];
            if (u != 0.0) {
                double t = std::abs(qr(k, j)) / u;
                t = (1.0 + t) * (1.0 - t);
                if (t < 0.0) t = 0.0;
                const double ratio = u / direct[static_cast<size_t>(j)];
                const double t2 = t * ratio * ratio;
                if (t2 <= downdate_thr) {
                    direct[static_cast<size_t>(j)] = norm(qr.col(j) + k + 1, rows - k - 1);
                    u = direct[static_cast<size_t>(j)];
                } else {
                    u *= std::sqrt(t);
                }
            }
        }
    }
    for (index_t k = 0; k < size; ++k) std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(transp[static_cast<size_t>(k)])]);
    // nonzeroPivots(): |r_ii| > maxpivot * (eps * diagSize) among the first m_nonzero_pivots
    const double thr = maxpivot * eps * static_cast<double>(size);
    index_t nz = 0;
    for (index_t i = 0; i < nonzero_pivots; ++i) nz += (std::abs(qr(i, i)) > thr) ? 1 : 0;
    Vector x(static_cast<size_t>(cols), 0.0);
    if (nz == 0) return x;
    // c = Q^T b using the first nz reflectors
    Vector c = b;
    for (index_t k = 0; k < nz; ++k) {
        const double tau = hcoeffs[static_cast<size_t>(k)];
        const index_t n = rows - k;
        if (n == 1) {
            c[static_cast<size_t>(k)] *= (1.0 - tau);
            continue;
        }
        if (tau == 0.0) continue;
        double t = c[static_cast<size_t>(k)];
        for (index_t i = 1; i < n; ++i) t += qr(k + i, k) * c[static_cast<size_t>(k + i)];
        c[static_cast<size_t>(k)] -= tau * t;
        for (index_t i = 1; i < n; ++i) c[static_cast<size_t>(k + i)] -= tau * qr(k + i, k) * t;
    }
    for (index_t i = nz - 1; i >= 0; --i) {  // upper-triangular solve
        double s = c[static_cast<size_t>(i)];
        for (index_t j = i + 1; j < nz; ++j) s -= qr(i, j) * c[static_cast<size_t>(j)];
        c[static_cast<size_t>(i)] = s / qr(i, i);
    }
    for (index_t i = 0; i < nz; ++i) x[static_cast<size_t>(perm[static_cast<size_t>(i)])] = c[static_cast<size_t>(i)];
    return x;
}

}  // namespace oracle
