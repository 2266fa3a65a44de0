// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Restates proj/core/src/tensor.cpp and proj/core/src/kruskal.cpp.
#include "oracle.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>

namespace oracle {

namespace {
void require(bool c, const char* w) {
    if (!c) throw std::invalid_argument(w);
}
}  // namespace

// tensor.cpp:23-32
Shape::Shape(std::vector<index_t> dims) : dims_(std::move(dims)) {
    require(!dims_.empty(), "Shape: order must be >= 1");
    k_ = 1;
    for (index_t d : dims_) {
        require(d >= 1, "Shape: every mode size must be >= 1");
        require(k_ <= std::numeric_limits<index_t>::max() / d, "Shape: element count overflows");
        k_ *= d;
    }
}

// tensor.cpp:34-42 (first mode fastest)
index_t Shape::offset(const index_t* c) const {
    index_t off = 0, stride = 1;
    for (int n = 0; n < order(); ++n) {
        off += c[n] * stride;
        stride *= dim(n);
    }
    return off;
}

// tensor.cpp:44-49
DenseTensor::DenseTensor(Shape s, std::vector<double> v) : shape(std::move(s)), values(std::move(v)) {
    require(static_cast<index_t>(values.size()) == shape.num_elements(), "DenseTensor: value count");
    for (double x : values) require(std::isfinite(x), "DenseTensor: entries must be finite");
}

// tensor.cpp:56-103: validate, stable lexicographic sort, sum duplicates, drop zeros.
SparseTensor::SparseTensor(Shape s, std::vector<index_t> c, std::vector<double> v) : shape(std::move(s)) {
    const size_t n = static_cast<size_t>(shape.order());
    require(c.size() == v.size() * n, "SparseTensor: coords/values size mismatch");
    for (double x : v) require(std::isfinite(x), "SparseTensor: entries must be finite");
    const size_t nnz = v.size();
    for (size_t i = 0; i < nnz; ++i)
        for (size_t k = 0; k < n; ++k)
            require(c[i * n + k] >= 0 && c[i * n + k] < shape.dim(static_cast<int>(k)),
                    "SparseTensor: coordinate out of bounds");
    std::vector<size_t> ord(nnz);
    std::iota(ord.begin(), ord.end(), size_t{0});
    auto less = [&](size_t a, size_t b) {
        return std::lexicographical_compare(c.begin() + static_cast<std::ptrdiff_t>(a * n),
                                            c.begin() + static_cast<std::ptrdiff_t>(a * n + n),
                                            c.begin() + static_cast<std::ptrdiff_t>(b * n),
                                            c.begin() + static_cast<std::ptrdiff_t>(b * n + n));
    };
    auto same = [&](size_t a, size_t b) {
        return std::equal(c.begin() + static_cast<std::ptrdiff_t>(a * n),
                          c.begin() + static_cast<std::ptrdiff_t>(a * n + n),
                          c.begin() + static_cast<std::ptrdiff_t>(b * n));
    };
    std::stable_sort(ord.begin(), ord.end(), less);
    for (size_t i = 0; i < nnz;) {
        double sum = v[ord[i]];
        size_t j = i + 1;
        while (j < nnz && same(ord[i], ord[j])) sum += v[ord[j++]];
        if (sum != 0.0) {
            coords.insert(coords.end(), c.begin() + static_cast<std::ptrdiff_t>(ord[i] * n),
                          c.begin() + static_cast<std::ptrdiff_t>(ord[i] * n + n));
            values.push_back(sum);
        }
        i = j;
    }
}

DenseTensor SparseTensor::densify() const {
    std::vector<double> out(static_cast<size_t>(shape.num_elements()), 0.0);
    const size_t n = static_cast<size_t>(shape.order());
    for (index_t i = 0; i < nnz(); ++i)
        out[static_cast<size_t>(shape.offset(coords.data() + static_cast<size_t>(i) * n))] =
            values[static_cast<size_t>(i)];
    return DenseTensor(shape, std::move(out));
}

// tensor.cpp:171-187 — first listed matrix's row index fastest.
Matrix khatri_rao(const std::vector<const Matrix*>& mats) {
    require(!mats.empty(), "khatri_rao: need at least one matrix");
    const index_t r = mats[0]->cols;
    for (auto* m : mats) require(m->cols == r, "khatri_rao: column counts must match");
    Matrix out = *mats[0];
    for (size_t k = 1; k < mats.size(); ++k) {
        const Matrix& nx = *mats[k];
        Matrix g(out.rows * nx.rows, r);
        for (index_t c = 0; c < r; ++c)
            for (index_t j = 0; j < nx.rows; ++j) {
                const double s = nx(j, c);
                for (index_t i = 0; i < out.rows; ++i) g(j * out.rows + i, c) = s * out(i, c);
            }
        out = std::move(g);
    }
    return out;
}

// tensor.cpp:139-158
Matrix matricize(const DenseTensor& t, int mode) {
    const Shape& s = t.shape;
    require(mode >= 0 && mode < s.order(), "matricize: mode out of range");
    const index_t rows = s.dim(mode), cols = s.co_size(mode);
    index_t inner = 1;
    for (int m = 0; m < mode; ++m) inner *= s.dim(m);
    const index_t outer = cols / inner;
    Matrix out(rows, cols);
    for (index_t b = 0; b < outer; ++b)
        for (index_t r = 0; r < rows; ++r)
            for (index_t a = 0; a < inner; ++a) out(r, a + b * inner) = t.values[static_cast<size_t>(a + r * inner + b * inner * rows)];
    return out;
}

namespace {
void check_factor_shapes(const Shape& s, const std::vector<Matrix>& f, int mode) {
    require(mode >= 0 && mode < s.order(), "mttkrp: mode out of range");
    require(static_cast<int>(f.size()) == s.order(), "mttkrp: need one factor per mode");
    for (int n = 0; n < s.order(); ++n) {
        require(f[static_cast<size_t>(n)].rows == s.dim(n), "mttkrp: factor row count does not match tensor mode size");
        require(f[static_cast<size_t>(n)].cols == f[0].cols, "mttkrp: factors must share a column count");
    }
}
std::vector<const Matrix*> ptrs(const std::vector<Matrix>& f, size_t lo, size_t hi) {
    std::vector<const Matrix*> p;
    for (size_t i = lo; i < hi; ++i) p.push_back(&f[i]);
    return p;
}
}  // namespace

// tensor.cpp:206-240. Mode 0: unf * KR(factors[1:]); last mode: unf^T * KR(factors[:n]);
// middle: per trailing slab b, (slab^T * lead) row-scaled by trail.row(b).
Matrix mttkrp(const DenseTensor& t, const std::vector<Matrix>& factors, int mode) {
    const Shape& s = t.shape;
    check_factor_shapes(s, factors, mode);
    const int n = s.order();
    const index_t rows = s.dim(mode), r = factors[0].cols;
    const double* v = t.values.data();
    if (n == 1) {
        Matrix out(rows, r);
        for (index_t c = 0; c < r; ++c)
            for (index_t i = 0; i < rows; ++i) out(i, c) = v[i];
        return out;
    }
    if (mode == 0) {
        const Matrix kr = khatri_rao(ptrs(factors, 1, factors.size()));
        const index_t co = s.co_size(0);
        Matrix out(rows, r);
        for (index_t p = 0; p < co; ++p) {
            const double* col = v + p * rows;
            for (index_t c = 0; c < r; ++c) {
                const double k = kr(p, c);
                double* o = out.col(c);
                for (index_t i = 0; i < rows; ++i) o[i] += col[i] * k;
            }
        }
        return out;
    }
    if (mode == n - 1) {
        const Matrix kr = khatri_rao(ptrs(factors, 0, static_cast<size_t>(mode)));
        const index_t co = s.co_size(mode);
        Matrix out(rows, r);
        constexpr index_t kb = 256;
        for (index_t p0 = 0; p0 < co; p0 += kb) {
            const index_t p1 = std::min(co, p0 + kb);
            for (index_t i = 0; i < rows; ++i) {
                const double* col = v + i * co;
                for (index_t c = 0; c < r; ++c) {
                    const double* kc = kr.col(c);
                    double acc = 0.0;
                    for (index_t p = p0; p < p1; ++p) acc += col[p] * kc[p];
                    out(i, c) += acc;
                }
            }
        }
        return out;
    }
    index_t inner = 1;
    for (int m = 0; m < mode; ++m) inner *= s.dim(m);
    const index_t outer = s.co_size(mode) / inner;
    const Matrix lead = khatri_rao(ptrs(factors, 0, static_cast<size_t>(mode)));
    const Matrix trail = khatri_rao(ptrs(factors, static_cast<size_t>(mode) + 1, factors.size()));
    Matrix out(rows, r);
    for (index_t b = 0; b < outer; ++b) {
        const double* slab = v + b * inner * rows;  // inner x rows, col-major
        for (index_t c = 0; c < r; ++c) {
            const double* lc = lead.col(c);
            const double tr = trail(b, c);
            for (index_t i = 0; i < rows; ++i) {
                const double* sc = slab + i * inner;
                double acc = 0.0;
                for (index_t a = 0; a < inner; ++a) acc += sc[a] * lc[a];
                out(i, c) += acc * tr;
            }
        }
    }
    return out;
}

// tensor.cpp:242-259
Matrix mttkrp(const SparseTensor& t, const std::vector<Matrix>& factors, int mode) {
    const Shape& s = t.shape;
    check_factor_shapes(s, factors, mode);
    const int n = s.order();
    const index_t r = factors[0].cols;
    Matrix out(s.dim(mode), r);
    std::vector<double> prod(static_cast<size_t>(r));
    for (index_t i = 0; i < t.nnz(); ++i) {
        const index_t* c = t.coords.data() + static_cast<size_t>(i) * static_cast<size_t>(n);
        std::fill(prod.begin(), prod.end(), t.values[static_cast<size_t>(i)]);
        for (int k = 0; k < n; ++k) {
            if (k == mode) continue;
            const Matrix& f = factors[static_cast<size_t>(k)];
            for (index_t q = 0; q < r; ++q) prod[static_cast<size_t>(q)] *= f(c[k], q);
        }
        for (index_t q = 0; q < r; ++q) out(c[mode], q) += prod[static_cast<size_t>(q)];
    }
    return out;
}

// tensor.cpp:261-274
Matrix gram_hadamard(const std::vector<Matrix>& factors, int skip) {
    require(!factors.empty(), "gram_hadamard: need at least one factor");
    const index_t r = factors[0].cols;
    Matrix out(r, r, 1.0);
    for (int n = 0; n < static_cast<int>(factors.size()); ++n) {
        if (n == skip) continue;
        const Matrix g = matmul_tn(factors[static_cast<size_t>(n)], factors[static_cast<size_t>(n)]);
        for (index_t i = 0; i < r * r; ++i) out.v[static_cast<size_t>(i)] *= g.v[static_cast<size_t>(i)];
    }
    Matrix sym(r, r);
    for (index_t j = 0; j < r; ++j)
        for (index_t i = 0; i < r; ++i) sym(i, j) = (out(i, j) + out(j, i)) / 2.0;
    return sym;
}

// tensor.cpp:276-293
DataTensor::DataTensor(DenseTensor t) : dense_(std::move(t)) {
    norm_ = oracle::norm(dense_->values);
    norm_sq_ = norm_ * norm_;
}
DataTensor::DataTensor(SparseTensor t) : sparse_(std::move(t)) {
    norm_ = oracle::norm(sparse_->values);
    norm_sq_ = norm_ * norm_;
}
Matrix DataTensor::mttkrp(const std::vector<Matrix>& f, int mode) const {
    return is_sparse() ? oracle::mttkrp(*sparse_, f, mode) : oracle::mttkrp(*dense_, f, mode);
}

// ---- kruskal.cpp -----------------------------------------------------------------------

KruskalTensor::KruskalTensor(std::vector<Matrix> f) : factors(std::move(f)) {
    require(!factors.empty(), "KruskalTensor: need at least one factor");
    require(factors[0].cols >= 1, "KruskalTensor: rank must be >= 1");
    for (const Matrix& a : factors) {
        require(a.cols == factors[0].cols, "KruskalTensor: factors must share a column count");
        require(a.rows >= 1, "KruskalTensor: factor must have rows");
        require(a.all_finite(), "KruskalTensor: entries must be finite");
    }
}

Shape KruskalTensor::shape() const {
    std::vector<index_t> d;
    for (const Matrix& a : factors) d.push_back(a.rows);
    return Shape(d);
}

// kruskal.cpp:35-48
DenseTensor full(const KruskalTensor& k) {
    const Shape s = k.shape();
    std::vector<double> flat(static_cast<size_t>(s.num_elements()), 0.0);
    const index_t rows = s.dim(0), cols = s.co_size(0), r = k.rank();
    if (k.order() == 1) {
        for (index_t i = 0; i < rows; ++i) {
            double acc = 0.0;
            for (index_t c = 0; c < r; ++c) acc += k.factors[0](i, c);
            flat[static_cast<size_t>(i)] = acc;
        }
    } else {
        const Matrix trail = khatri_rao(ptrs(k.factors, 1, k.factors.size()));
        for (index_t p = 0; p < cols; ++p)
            for (index_t c = 0; c < r; ++c) {
                const double w = trail(p, c);
                const double* a = k.factors[0].col(c);
                for (index_t i = 0; i < rows; ++i) flat[static_cast<size_t>(p * rows + i)] += a[i] * w;
            }
    }
    return DenseTensor(s, std::move(flat));
}

namespace {

// kruskal.cpp:54-72
struct GramSet {
    std::vector<Matrix> grams;
    explicit GramSet(const std::vector<Matrix>& f) {
        for (const Matrix& a : f) grams.push_back(matmul_tn(a, a));
    }
    Matrix hadamard_skipping(int skip) const {
        const index_t r = grams[0].rows;
        Matrix out(r, r, 1.0);
        for (int n = 0; n < static_cast<int>(grams.size()); ++n) {
            if (n == skip) continue;
            for (index_t i = 0; i < r * r; ++i) out.v[static_cast<size_t>(i)] *= grams[static_cast<size_t>(n)].v[static_cast<size_t>(i)];
        }
        Matrix sym(r, r);
        for (index_t j = 0; j < r; ++j)
            for (index_t i = 0; i < r; ++i) sym(i, j) = (out(i, j) + out(j, i)) / 2.0;
        return sym;
    }
};

// kruskal.cpp:83-102: residual streamed in 256-column blocks of the mode-1 unfolding.
double dense_residual_objective(const DenseTensor& t, const KruskalTensor& k) {
    const index_t rows = t.shape.dim(0), cols = t.shape.co_size(0), r = k.rank();
    const double* data = t.values.data();
    if (k.order() == 1) {
        double s = 0.0;
        for (index_t i = 0; i < rows; ++i) {
            double m = 0.0;
            for (index_t c = 0; c < r; ++c) m += k.factors[0](i, c);
            const double d = data[i] - m;
            s += d * d;
        }
        return 0.5 * s;
    }
    const Matrix trail = khatri_rao(ptrs(k.factors, 1, k.factors.size()));
    constexpr index_t kb = 256;
    std::vector<double> buf(static_cast<size_t>(rows * std::min(cols, kb)));
    double sum = 0.0;
    for (index_t at = 0; at < cols; at += kb) {
        const index_t w = std::min(kb, cols - at);
        std::fill(buf.begin(), buf.end(), 0.0);
        for (index_t p = 0; p < w; ++p)
            for (index_t c = 0; c < r; ++c) {
                const double tw = trail(at + p, c);
                const double* a = k.factors[0].col(c);
                double* b = buf.data() + p * rows;
                for (index_t i = 0; i < rows; ++i) b[i] += a[i] * tw;
            }
        for (index_t p = 0; p < w; ++p)
            for (index_t i = 0; i < rows; ++i) {
                const double d = data[(at + p) * rows + i] - buf[static_cast<size_t>(p * rows + i)];
                sum += d * d;
            }
    }
    return 0.5 * sum;
}

// kruskal.cpp:106-111
double sparse_objective(const DataTensor& t, const KruskalTensor& k) {
    const Matrix m0 = t.mttkrp(k.factors, 0);
    double inner = 0.0;
    for (index_t i = 0; i < m0.size(); ++i) inner += m0.v[static_cast<size_t>(i)] * k.factors[0].v[static_cast<size_t>(i)];
    const Matrix gam = gram_hadamard(k.factors);
    double gs = 0.0;
    for (double x : gam.v) gs += x;
    return 0.5 * t.norm_squared() - inner + 0.5 * gs;
}

void check_shapes(const DataTensor& t, const KruskalTensor& k) {
    require(t.shape() == k.shape(), "tensor and Kruskal model shapes must match");
}

}  // namespace

double objective(const DataTensor& t, const KruskalTensor& k) {
    check_shapes(t, k);
    if (!t.is_sparse()) return dense_residual_objective(t.dense(), k);
    return sparse_objective(t, k);
}

// kruskal.cpp:127-149
double objective_and_gradient(const DataTensor& t, const KruskalTensor& k, Vector& grad) {
    check_shapes(t, k);
    const GramSet grams(k.factors);
    index_t total = 0;
    for (const Matrix& a : k.factors) total += a.size();
    grad.assign(static_cast<size_t>(total), 0.0);
    double inner = 0.0;
    index_t at = 0;
    for (int n = 0; n < k.order(); ++n) {
        const Matrix m = t.mttkrp(k.factors, n);
        if (n == 0)
            for (index_t i = 0; i < m.size(); ++i) inner += m.v[static_cast<size_t>(i)] * k.factors[0].v[static_cast<size_t>(i)];
        const Matrix ag = matmul(k.factors[static_cast<size_t>(n)], grams.hadamard_skipping(n));
        for (index_t i = 0; i < m.size(); ++i) grad[static_cast<size_t>(at + i)] = -m.v[static_cast<size_t>(i)] + ag.v[static_cast<size_t>(i)];
        at += m.size();
    }
    if (!t.is_sparse()) return dense_residual_objective(t.dense(), k);
    const Matrix gam = grams.hadamard_skipping(-1);
    double gs = 0.0;
    for (double x : gam.v) gs += x;
    return 0.5 * t.norm_squared() - inner + 0.5 * gs;
}

// kruskal.cpp:151-154
double fit_h(const DataTensor& t, const KruskalTensor& k) {
    require(t.norm() > 0.0, "fit_h: data tensor must be nonzero");
    return std::sqrt(std::max(2.0 * objective(t, k), 0.0)) / t.norm();
}

// kruskal.cpp:156-193
KruskalTensor normalize_and_reorder(const KruskalTensor& k) {
    const int order = k.order();
    const index_t rank = k.rank();
    Matrix norms(order, rank);
    for (int n = 0; n < order; ++n)
        for (index_t r = 0; r < rank; ++r) norms(n, r) = norm(k.factors[static_cast<size_t>(n)].col(r), k.factors[static_cast<size_t>(n)].rows);
    std::vector<double> lambda(static_cast<size_t>(rank), 1.0);
    for (index_t r = 0; r < rank; ++r) {
        double l = 1.0;
        for (int n = 0; n < order; ++n) l *= norms(n, r);
        lambda[static_cast<size_t>(r)] = l;
    }
    std::vector<index_t> perm(static_cast<size_t>(rank));
    std::iota(perm.begin(), perm.end(), index_t{0});
    std::stable_sort(perm.begin(), perm.end(), [&](index_t a, index_t b) {
        return lambda[static_cast<size_t>(a)] > lambda[static_cast<size_t>(b)];
    });
    std::vector<Matrix> out;
    for (int n = 0; n < order; ++n) {
        const Matrix& src = k.factors[static_cast<size_t>(n)];
        Matrix a(src.rows, rank);
        for (index_t r = 0; r < rank; ++r) {
            const index_t s = perm[static_cast<size_t>(r)];
            const double l = lambda[static_cast<size_t>(s)];
            const double scale = (l == 0.0) ? 1.0 : std::pow(l, 1.0 / order) / norms(n, s);
            for (index_t i = 0; i < src.rows; ++i) a(i, r) = (l == 0.0) ? src(i, s) : src(i, s) * scale;
        }
        out.push_back(std::move(a));
    }
    return KruskalTensor(std::move(out));
}

// kruskal.cpp:195-221
Vector pack(const KruskalTensor& k) {
    Vector v;
    for (const Matrix& a : k.factors) v.insert(v.end(), a.v.begin(), a.v.end());
    return v;
}

KruskalTensor unpack(const Vector& v, const Shape& s, index_t rank) {
    index_t total = 0;
    for (int n = 0; n < s.order(); ++n) total += s.dim(n) * rank;
    require(static_cast<index_t>(v.size()) == total, "unpack: vector length does not match shape and rank");
    std::vector<Matrix> f;
    index_t at = 0;
    for (int n = 0; n < s.order(); ++n) {
        Matrix a(s.dim(n), rank);
        std::copy(v.begin() + at, v.begin() + at + a.size(), a.v.begin());
        at += a.size();
        f.push_back(std::move(a));
    }
    return KruskalTensor(std::move(f));
}

}  // namespace oracle
