// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference C++ implementation (arxiv/paper_1105_5331, proj/core/)
// used as the parity checker for the B200 path. Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it. The product library never
// links or calls anything in oracle/.
//
// The reference itself cannot be compiled here: Eigen3 (its only numerical dependency,
// `find_package(Eigen3 3.3 REQUIRED)` at proj/core/CMakeLists.txt:1, version unpinned) is
// absent, as are GTest and CLI11. This restatement therefore carries its
// own small column-major dense linear algebra that reproduces the published Eigen
// algorithms used on the path: plain GEMM, the unblocked LLT (Eigen's llt_inplace for
// sizes < 32, failure on a non-positive pivot), Householder QR with makeHouseholder /
// applyHouseholderOnTheLeft semantics, and ColPivHouseholderQR (norm downdating,
// rank threshold epsilon*diagSize) for the damped least-squares solve in accelerate().
// Parity is pinned by the reference's own known-answer tests restated in
// tests/test_oracle_known_answers.py; bit-level Eigen rounding is
// not reproducible without Eigen and is not claimed.
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using index_t = std::int64_t;

// Column-major dense matrix (stands in for Eigen::MatrixXd, tensor.hpp:13).
struct Matrix {
    index_t rows = 0, cols = 0;
    std::vector<double> v;
    Matrix() = default;
    Matrix(index_t r, index_t c, double fill = 0.0) : rows(r), cols(c), v(static_cast<size_t>(r * c), fill) {}
    double& operator()(index_t i, index_t j) { return v[static_cast<size_t>(i + j * rows)]; }
    double operator()(index_t i, index_t j) const { return v[static_cast<size_t>(i + j * rows)]; }
    double* col(index_t j) { return v.data() + j * rows; }
    const double* col(index_t j) const { return v.data() + j * rows; }
    index_t size() const { return rows * cols; }
    bool all_finite() const;
};
using Vector = std::vector<double>;

// ---- small dense LA (Eigen stand-ins) -------------------------------------------------
Matrix matmul(const Matrix& a, const Matrix& b);     // a * b
Matrix matmul_tn(const Matrix& a, const Matrix& b);  // a^T * b
double dot(const Vector& a, const Vector& b);
double norm(const Vector& a);                        // Eigen norm(): sqrt(squaredNorm())
double norm(const double* x, index_t n);

// Eigen::LLT<MatrixXd> (lower), unblocked path used for n < 32. Returns false on a
// non-positive pivot (x <= 0), exactly Eigen's info() != Success criterion.
struct LLT {
    Matrix l;
    bool ok = false;
    explicit LLT(const Matrix& a);
    // Solve A X = B (B is n x k).
    Matrix solve(const Matrix& b) const;
    Matrix matrix_u() const;  // L^T
};

// Eigen makeHouseholder on x[0..n) (tau, beta; essential part left in x[1..n)) and
// applyHouseholderOnTheLeft on rows r0..r0+n of columns [c0, c1) of m.
void make_householder(double* x, index_t n, double& tau, double& beta);
void apply_householder_left(Matrix& m, index_t r0, index_t n, index_t c0, index_t c1, const double* ess, double tau);

// Eigen::ColPivHouseholderQR<MatrixXd>(a).solve(b) for a single right-hand side.
Vector colpiv_qr_solve(const Matrix& a, const Vector& b);

// ---- tensor.hpp -----------------------------------------------------------------------
class Shape {
public:
    explicit Shape(std::vector<index_t> dims);
    int order() const { return static_cast<int>(dims_.size()); }
    index_t dim(int mode) const { return dims_[static_cast<size_t>(mode)]; }
    const std::vector<index_t>& dims() const { return dims_; }
    index_t num_elements() const { return k_; }
    index_t co_size(int mode) const { return k_ / dim(mode); }
    index_t offset(const index_t* coords) const;
    bool operator==(const Shape& o) const { return dims_ == o.dims_; }

private:
    std::vector<index_t> dims_;
    index_t k_ = 0;
};

struct DenseTensor {
    Shape shape;
    std::vector<double> values;
    DenseTensor(Shape s, std::vector<double> v);
};

struct SparseTensor {
    Shape shape;
    std::vector<index_t> coords;  // nnz*N, AoS
    std::vector<double> values;
    SparseTensor(Shape s, std::vector<index_t> c, std::vector<double> v);  // canonicalizes
    index_t nnz() const { return static_cast<index_t>(values.size()); }
    DenseTensor densify() const;
};

Matrix khatri_rao(const std::vector<const Matrix*>& mats);
Matrix matricize(const DenseTensor& t, int mode);
Matrix mttkrp(const DenseTensor& t, const std::vector<Matrix>& factors, int mode);
Matrix mttkrp(const SparseTensor& t, const std::vector<Matrix>& factors, int mode);
Matrix gram_hadamard(const std::vector<Matrix>& factors, int skip = -1);

class DataTensor {
public:
    explicit DataTensor(DenseTensor t);
    explicit DataTensor(SparseTensor t);
    const Shape& shape() const { return dense_ ? dense_->shape : sparse_->shape; }
    bool is_sparse() const { return sparse_.has_value(); }
    const DenseTensor& dense() const { return *dense_; }
    const SparseTensor& sparse() const { return *sparse_; }
    double norm() const { return norm_; }
    double norm_squared() const { return norm_sq_; }
    Matrix mttkrp(const std::vector<Matrix>& factors, int mode) const;

private:
    std::optional<DenseTensor> dense_;
    std::optional<SparseTensor> sparse_;
    double norm_ = 0, norm_sq_ = 0;
};

// ---- kruskal.hpp ----------------------------------------------------------------------
struct KruskalTensor {
    std::vector<Matrix> factors;
    explicit KruskalTensor(std::vector<Matrix> f);
    int order() const { return static_cast<int>(factors.size()); }
    index_t rank() const { return factors[0].cols; }
    Shape shape() const;
};

DenseTensor full(const KruskalTensor& k);
double objective(const DataTensor& t, const KruskalTensor& k);
double objective_and_gradient(const DataTensor& t, const KruskalTensor& k, Vector& grad);
double fit_h(const DataTensor& t, const KruskalTensor& k);
KruskalTensor normalize_and_reorder(const KruskalTensor& k);
Vector pack(const KruskalTensor& k);
KruskalTensor unpack(const Vector& v, const Shape& shape, index_t rank);

// ---- errors / trace -------------------------------------------------------------------
struct numerical_error : std::runtime_error {
    explicit numerical_error(const std::string& w) : std::runtime_error(w) {}
};
enum class StopReason { GradTol = 0, MaxIters = 1, Stalled = 2 };
struct TraceRecord {
    int iter = 0;
    double time_s = 0;
    double f = 0, h = 0, gnorm_rel = 0;
    long fevals = 0, gevals = 0;
    int precond_calls = 0;
    bool restart = false;
    double beta = 0;
};

// ---- als ------------------------------------------------------------------------------
KruskalTensor als_sweep(const DataTensor& t, const KruskalTensor& k);
struct AlsOptions {
    double tol_grad = 1e-9;
    int max_iters = 2000;
};
struct SolveResult {
    KruskalTensor solution;
    std::vector<TraceRecord> trace;
    StopReason stop;
};
SolveResult als_solve(const DataTensor& t, const KruskalTensor& initial, const AlsOptions& o);

// ---- line search ----------------------------------------------------------------------
struct LineSearchParams {
    double ftol = 1e-4, gtol = 1e-2, initial_step = 1.0;
    int max_evals = 20;
    double step_min = 0.0, step_max = 1e20;
};
enum class LineSearchStatus { Converged = 0, MaxEvals = 1, NotDescent = 2, NumericalStall = 3 };
struct LineSearchResult {
    double step = 0, f = 0, dg = 0;
    LineSearchStatus status = LineSearchStatus::NotDescent;
    int evals = 0;
};
using LineSearchEval = std::function<void(double, double&, double&)>;
LineSearchResult more_thuente(const LineSearchEval& eval, double phi0, double dphi0,
                              const LineSearchParams& p);

// ---- ngmres ---------------------------------------------------------------------------
struct AccelWindow {
    size_t capacity;
    std::vector<std::pair<Vector, Vector>> entries;  // oldest first
    explicit AccelWindow(size_t cap);
    void push(Vector u, Vector g);
    void reset(Vector u, Vector g);
    size_t size() const { return entries.size(); }
};
struct AccelOutcome {
    Vector u_hat, alpha;
    double system_residual_rel = 0;
};
AccelOutcome accelerate(const AccelWindow& w, const Vector& u_bar, const Vector& g_bar, double eps);

struct NgmresOptions {
    int window = 20;
    double epsilon_reg = 1e-12;
    double tol_grad = 1e-9;
    int max_iters = 2000;
    LineSearchParams line_search{};
    bool restart_on_ascent = true;
};
struct NgmresProblem {
    std::function<double(const Vector&, Vector&)> eval;
    std::function<Vector(const Vector&)> precondition;
    std::function<Vector(const Vector&)> canonicalize;
    double gradient_scale = 1.0;
    std::function<double(double)> fit_from_f;
    std::optional<double> fixed_step;
    std::function<void(const AccelWindow&, const Vector&, const Vector&, const Vector&)> observer;
};
struct MinimizeResult {
    Vector u;
    double f = 0;
    std::vector<TraceRecord> trace;
    StopReason stop = StopReason::MaxIters;
    // Iterate log (test instrumentation, not in the reference): the accepted iterate after
    // each iteration, recorded when record_iterates is set.
    std::vector<Vector> iterates;
};
struct NgmresState {
    AccelWindow window;
    Vector u, g;
    double f = 0;
    long fevals = 0, gevals = 0;
};
struct NgmresStepReport {
    bool restart = false, stalled = false;
    double beta = 0;
};
NgmresState ngmres_init(const NgmresProblem& p, const Vector& initial, const NgmresOptions& o);
NgmresStepReport ngmres_step(const NgmresProblem& p, NgmresState& s, const NgmresOptions& o);
MinimizeResult ngmres_minimize(const NgmresProblem& p, const Vector& initial, const NgmresOptions& o,
                               int record_iterates = 0);
// The CP instantiation (ngmres.cpp:202-226) with an explicit gradient scale so the
// BASELINE stop rule (||g||/(R*sum I_n)) can be used.
MinimizeResult ngmres_cp(const DataTensor& t, const KruskalTensor& initial, const NgmresOptions& o,
                         double gradient_scale, int record_iterates = 0);

// ---- ncg ------------------------------------------------------------------------------
struct NcgOptions {
    double tol_grad = 1e-9;
    int max_iters = 2000;
    LineSearchParams line_search{};
};
MinimizeResult ncg_minimize(const std::function<double(const Vector&, Vector&)>& eval,
                            const Vector& initial, const NcgOptions& o, double gradient_scale,
                            const std::function<double(double)>& fit_from_f);

}  // namespace oracle
