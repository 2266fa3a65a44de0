// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Restates proj/core/src/als.cpp, line_search.cpp, ngmres.cpp and ncg.cpp.
#include "oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>

namespace oracle {

namespace {

// als.cpp:16-34 — X * G = B via LLT(G).solve(B^T)^T, one ridge retry (1e-12 * trace).
Matrix solve_normal(const Matrix& gram, const Matrix& rhs) {
    auto attempt = [&](const Matrix& g, Matrix& x) {
        LLT llt(g);
        if (!llt.ok) return false;
        Matrix bt(rhs.cols, rhs.rows);
        for (index_t i = 0; i < rhs.rows; ++i)
            for (index_t j = 0; j < rhs.cols; ++j) bt(j, i) = rhs(i, j);
        const Matrix xt = llt.solve(bt);
        x = Matrix(rhs.rows, rhs.cols);
        for (index_t i = 0; i < rhs.rows; ++i)
            for (index_t j = 0; j < rhs.cols; ++j) x(i, j) = xt(j, i);
        return x.all_finite();
    };
    Matrix x;
    if (attempt(gram, x)) return x;
    double tr = 0.0;
    for (index_t i = 0; i < gram.rows; ++i) tr += gram(i, i);
    const double ridge = 1e-12 * tr;
    if (ridge > 0.0) {
        Matrix reg = gram;
        for (index_t i = 0; i < gram.rows; ++i) reg(i, i) += ridge;
        if (attempt(reg, x)) return x;
    }
    throw numerical_error("als_sweep: normal matrix is singular after regularization "
                          "(structurally rank-deficient iterate)");
}

}  // namespace

// als.cpp:38-48 — Gauss-Seidel over modes 0..N-1, then normalize_and_reorder.
KruskalTensor als_sweep(const DataTensor& t, const KruskalTensor& k) {
    if (!(t.shape() == k.shape())) throw std::invalid_argument("als_sweep: tensor and model shapes must match");
    KruskalTensor cur = k;
    for (int n = 0; n < cur.order(); ++n) {
        const Matrix rhs = t.mttkrp(cur.factors, n);
        const Matrix gram = gram_hadamard(cur.factors, n);
        cur.factors[static_cast<size_t>(n)] = solve_normal(gram, rhs);
    }
    return normalize_and_reorder(cur);
}

// als.cpp:50-96
SolveResult als_solve(const DataTensor& t, const KruskalTensor& initial, const AlsOptions& o) {
    KruskalTensor cur = normalize_and_reorder(initial);
    Vector g;
    double f = objective_and_gradient(t, cur, g);
    long fevals = 1, gevals = 1;
    std::vector<TraceRecord> trace;
    auto record = [&](int it, double fv, double gn, int pc) {
        trace.push_back({it, 0.0, fv, std::sqrt(std::max(2.0 * fv, 0.0)) / t.norm(), gn / t.norm(), fevals, gevals, pc, false, 0.0});
    };
    double gn = norm(g);
    record(0, f, gn, 0);
    KruskalTensor best = cur;
    double best_f = f;
    StopReason stop = StopReason::MaxIters;
    if (gn / t.norm() <= o.tol_grad) return {best, trace, StopReason::GradTol};
    for (int it = 1; it <= o.max_iters; ++it) {
        cur = als_sweep(t, cur);
        f = objective_and_gradient(t, cur, g);
        ++fevals;
        ++gevals;
        gn = norm(g);
        record(it, f, gn, it);
        if (f < best_f) {
            best_f = f;
            best = cur;
        }
        if (gn / t.norm() <= o.tol_grad) {
            stop = StopReason::GradTol;
            break;
        }
    }
    return {best, trace, stop};
}

// ---- line_search.cpp -------------------------------------------------------------------

namespace {

// line_search.cpp:16-108 — the four-case cubic/quadratic trial step on the interval of
// uncertainty; (sx,fx,gx) best endpoint, (sy,fy,gy) other endpoint, (sp,fp,gp) trial.
double trial_step(double& sx, double& fx, double& gx, double& sy, double& fy, double& gy, double sp,
                  double fp, double gp, bool& bracketed, double lo, double hi) {
    const double sgnd = gp * (gx >= 0.0 ? 1.0 : -1.0);
    double next = sp;
    auto cubic_gamma = [](double theta, double a, double b, bool clamp0) {
        const double s = std::max({std::abs(theta), std::abs(a), std::abs(b)});
        const double disc = (theta / s) * (theta / s) - (a / s) * (b / s);
        return s * std::sqrt(clamp0 ? std::max(0.0, disc) : disc);
    };
    if (fp > fx) {  // case 1
        const double theta = 3.0 * (fx - fp) / (sp - sx) + gx + gp;
        double gamma = cubic_gamma(theta, gx, gp, false);
        if (sp < sx) gamma = -gamma;
        const double p = (gamma - gx) + theta;
        const double q = ((gamma - gx) + gamma) + gp;
        const double stpc = sx + (p / q) * (sp - sx);
        const double stpq = sx + ((gx / ((fx - fp) / (sp - sx) + gx)) / 2.0) * (sp - sx);
        next = (std::abs(stpc - sx) < std::abs(stpq - sx)) ? stpc : stpc + (stpq - stpc) / 2.0;
        bracketed = true;
    } else if (sgnd < 0.0) {  // case 2
        const double theta = 3.0 * (fx - fp) / (sp - sx) + gx + gp;
        double gamma = cubic_gamma(theta, gx, gp, false);
        if (sp > sx) gamma = -gamma;
        const double p = (gamma - gp) + theta;
        const double q = ((gamma - gp) + gamma) + gx;
        const double stpc = sp + (p / q) * (sx - sp);
        const double stpq = sp + (gp / (gp - gx)) * (sx - sp);
        next = (std::abs(stpc - sp) > std::abs(stpq - sp)) ? stpc : stpq;
        bracketed = true;
    } else if (std::abs(gp) < std::abs(gx)) {  // case 3
        const double theta = 3.0 * (fx - fp) / (sp - sx) + gx + gp;
        double gamma = cubic_gamma(theta, gx, gp, true);
        if (sp > sx) gamma = -gamma;
        const double p = (gamma - gp) + theta;
        const double q = (gamma + (gx - gp)) + gamma;
        const double r = p / q;
        double stpc;
        if (r < 0.0 && gamma != 0.0)
            stpc = sp + r * (sx - sp);
        else if (sp > sx)
            stpc = hi;
        else
            stpc = lo;
        const double stpq = sp + (gp / (gp - gx)) * (sx - sp);
        if (bracketed) {
            next = (std::abs(stpc - sp) < std::abs(stpq - sp)) ? stpc : stpq;
            next = (sp > sx) ? std::min(sp + 0.66 * (sy - sp), next) : std::max(sp + 0.66 * (sy - sp), next);
        } else {
            next = (std::abs(stpc - sp) > std::abs(stpq - sp)) ? stpc : stpq;
            next = std::clamp(next, lo, hi);
        }
    } else {  // case 4
        if (bracketed) {
            const double theta = 3.0 * (fp - fy) / (sy - sp) + gy + gp;
            double gamma = cubic_gamma(theta, gy, gp, false);
            if (sp > sy) gamma = -gamma;
            const double p = (gamma - gp) + theta;
            const double q = ((gamma - gp) + gamma) + gy;
            next = sp + (p / q) * (sy - sp);
        } else {
            next = (sp > sx) ? hi : lo;
        }
    }
    if (fp > fx) {
        sy = sp;
        fy = fp;
        gy = gp;
    } else {
        if (sgnd < 0.0) {
            sy = sx;
            fy = fx;
            gy = gx;
        }
        sx = sp;
        fx = fp;
        gx = gp;
    }
    return next;
}

}  // namespace

// line_search.cpp:112-224
LineSearchResult more_thuente(const LineSearchEval& eval, double phi0, double dphi0,
                              const LineSearchParams& p) {
    if (!(p.ftol > 0.0 && p.ftol < p.gtol && p.gtol < 1.0)) throw std::invalid_argument("more_thuente: need 0 < ftol < gtol < 1");
    if (!(p.initial_step > 0.0)) throw std::invalid_argument("more_thuente: initial_step must be > 0");
    if (p.max_evals < 1) throw std::invalid_argument("more_thuente: max_evals must be >= 1");
    if (!(p.step_min >= 0.0 && p.step_min < p.step_max)) throw std::invalid_argument("more_thuente: need 0 <= step_min < step_max");
    if (dphi0 >= 0.0) return {0.0, phi0, dphi0, LineSearchStatus::NotDescent, 0};
    const double xtol = 1e-15, xlo = 1.1, xhi = 4.0;
    const double gtest = p.ftol * dphi0;
    double width = p.step_max - p.step_min, width1 = 2.0 * width;
    double sx = 0.0, fx = phi0, gx = dphi0, sy = 0.0, fy = phi0, gy = dphi0;
    double stp = std::clamp(p.initial_step, std::max(p.step_min, 1e-300), p.step_max);
    double lo = 0.0, hi = stp + xhi * stp;
    bool bracketed = false, stage1 = true;
    double best_s = 0.0, best_f = phi0, best_g = dphi0;
    int evals = 0;
    for (;;) {
        double f = 0.0, g = 0.0;
        eval(stp, f, g);
        ++evals;
        if (f < best_f) {
            best_s = stp;
            best_f = f;
            best_g = g;
        }
        const double ftest = phi0 + stp * gtest;
        if (stage1 && f <= ftest && g >= std::min(p.ftol, p.gtol) * dphi0) stage1 = false;
        if (f <= ftest && std::abs(g) <= p.gtol * (-dphi0)) return {stp, f, g, LineSearchStatus::Converged, evals};
        if (evals >= p.max_evals) return {best_s, best_f, best_g, LineSearchStatus::MaxEvals, evals};
        if (bracketed && (stp <= lo || stp >= hi)) return {best_s, best_f, best_g, LineSearchStatus::NumericalStall, evals};
        if (bracketed && hi - lo <= xtol * hi) return {best_s, best_f, best_g, LineSearchStatus::NumericalStall, evals};
        if (stp == p.step_max && f <= ftest && g <= gtest) return {best_s, best_f, best_g, LineSearchStatus::MaxEvals, evals};
        if (stp == p.step_min && (f > ftest || g >= gtest)) return {best_s, best_f, best_g, LineSearchStatus::NumericalStall, evals};
        if (stage1 && f <= fx && f > ftest) {
            double fm = f - stp * gtest, fxm = fx - sx * gtest, fym = fy - sy * gtest;
            double gm = g - gtest, gxm = gx - gtest, gym = gy - gtest;
            stp = trial_step(sx, fxm, gxm, sy, fym, gym, stp, fm, gm, bracketed, lo, hi);
            fx = fxm + sx * gtest;
            fy = fym + sy * gtest;
            gx = gxm + gtest;
            gy = gym + gtest;
        } else {
            stp = trial_step(sx, fx, gx, sy, fy, gy, stp, f, g, bracketed, lo, hi);
        }
        if (bracketed) {
            if (std::abs(sy - sx) >= 0.66 * width1) stp = sx + 0.5 * (sy - sx);
            width1 = width;
            width = std::abs(sy - sx);
            lo = std::min(sx, sy);
            hi = std::max(sx, sy);
        } else {
            lo = stp + xlo * (stp - sx);
            hi = stp + xhi * (stp - sx);
        }
        stp = std::clamp(stp, p.step_min, p.step_max);
        if ((bracketed && (stp <= lo || stp >= hi)) || (bracketed && hi - lo <= xtol * hi)) stp = sx;
        if (stp <= 0.0) stp = (hi > 0.0) ? 0.5 * hi : p.initial_step;
    }
}

// ---- ngmres.cpp ------------------------------------------------------------------------

AccelWindow::AccelWindow(size_t cap) : capacity(cap) {
    if (cap < 1) throw std::invalid_argument("AccelWindow: capacity must be >= 1");
}
void AccelWindow::push(Vector u, Vector g) {
    entries.emplace_back(std::move(u), std::move(g));
    while (entries.size() > capacity) entries.erase(entries.begin());
}
void AccelWindow::reset(Vector u, Vector g) {
    entries.clear();
    entries.emplace_back(std::move(u), std::move(g));
}

// ngmres.cpp:27-63
AccelOutcome accelerate(const AccelWindow& w, const Vector& ub, const Vector& gb, double eps) {
    if (w.size() == 0) throw std::invalid_argument("accelerate: window must be nonempty");
    const index_t m = static_cast<index_t>(w.size()), n = static_cast<index_t>(gb.size());
    Matrix p(n, m);
    for (index_t j = 0; j < m; ++j)
        for (index_t i = 0; i < n; ++i) p(i, j) = gb[static_cast<size_t>(i)] - w.entries[static_cast<size_t>(j)].second[static_cast<size_t>(i)];
    Matrix lhs = matmul_tn(p, p);
    double dmax = lhs(0, 0);
    for (index_t j = 1; j < m; ++j) dmax = std::max(dmax, lhs(j, j));
    const double delta = (dmax > 0.0) ? eps * dmax : eps;
    for (index_t j = 0; j < m; ++j) lhs(j, j) += delta;
    Vector rhs(static_cast<size_t>(m));
    for (index_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (index_t i = 0; i < n; ++i) s += p(i, j) * gb[static_cast<size_t>(i)];
        rhs[static_cast<size_t>(j)] = -s;
    }
    Vector alpha(static_cast<size_t>(m), 0.0);
    double resid = 0.0;
    if (norm(rhs) != 0.0) {
        Matrix st(n + m, m);
        for (index_t j = 0; j < m; ++j) {
            for (index_t i = 0; i < n; ++i) st(i, j) = p(i, j);
            st(n + j, j) = std::sqrt(delta);
        }
        Vector srhs(static_cast<size_t>(n + m), 0.0);
        for (index_t i = 0; i < n; ++i) srhs[static_cast<size_t>(i)] = -gb[static_cast<size_t>(i)];
        alpha = colpiv_qr_solve(st, srhs);
        Vector r(static_cast<size_t>(m));
        for (index_t i = 0; i < m; ++i) {
            double s = 0.0;
            for (index_t j = 0; j < m; ++j) s += lhs(i, j) * alpha[static_cast<size_t>(j)];
            r[static_cast<size_t>(i)] = s - rhs[static_cast<size_t>(i)];
        }
        resid = norm(r) / norm(rhs);
    }
    Vector uh = ub;
    for (index_t j = 0; j < m; ++j) {
        const Vector& uj = w.entries[static_cast<size_t>(j)].first;
        const double a = alpha[static_cast<size_t>(j)];
        for (index_t i = 0; i < n; ++i) uh[static_cast<size_t>(i)] += a * (ub[static_cast<size_t>(i)] - uj[static_cast<size_t>(i)]);
    }
    return {uh, alpha, resid};
}

namespace {
Vector canonical(const NgmresProblem& p, const Vector& u) { return p.canonicalize ? p.canonicalize(u) : u; }
Vector axpy(const Vector& x, double a, const Vector& d) {
    Vector y = x;
    for (size_t i = 0; i < y.size(); ++i) y[i] += a * d[i];
    return y;
}
}  // namespace

// ngmres.cpp:73-85
NgmresState ngmres_init(const NgmresProblem& p, const Vector& initial, const NgmresOptions& o) {
    if (o.window < 1) throw std::invalid_argument("ngmres: window must be >= 1");
    if (!(o.tol_grad > 0.0)) throw std::invalid_argument("ngmres: tol_grad must be > 0");
    if (o.epsilon_reg < 0.0) throw std::invalid_argument("ngmres: epsilon_reg must be >= 0");
    NgmresState s{AccelWindow(static_cast<size_t>(o.window)), canonical(p, initial), {}, 0.0, 0, 0};
    s.f = p.eval(s.u, s.g);
    s.fevals = s.gevals = 1;
    s.window.push(s.u, s.g);
    return s;
}

// ngmres.cpp:87-158
NgmresStepReport ngmres_step(const NgmresProblem& p, NgmresState& s, const NgmresOptions& o) {
    const Vector ub = p.precondition(s.u);
    Vector gb;
    const double fb = p.eval(ub, gb);
    ++s.fevals;
    ++s.gevals;
    const AccelOutcome acc = accelerate(s.window, ub, gb, o.epsilon_reg);
    if (p.observer) p.observer(s.window, ub, gb, acc.u_hat);
    Vector d(ub.size());
    for (size_t i = 0; i < d.size(); ++i) d[i] = acc.u_hat[i] - ub[i];
    const double slope = dot(gb, d);
    NgmresStepReport rep;
    Vector un, gn;
    double fn;
    if (o.restart_on_ascent && slope >= 0.0) {
        rep.restart = true;
        un = ub;
        fn = fb;
        gn = gb;
    } else if (p.fixed_step) {
        rep.beta = *p.fixed_step;
        un = canonical(p, axpy(ub, rep.beta, d));
        fn = p.eval(un, gn);
        ++s.fevals;
        ++s.gevals;
    } else if (slope >= 0.0) {
        un = ub;
        fn = fb;
        gn = gb;
    } else {
        Vector gt;
        auto phi = [&](double step, double& fv, double& dg) {
            fv = p.eval(axpy(ub, step, d), gt);
            dg = dot(gt, d);
        };
        const LineSearchResult ls = more_thuente(phi, fb, slope, o.line_search);
        s.fevals += ls.evals;
        s.gevals += ls.evals;
        if (ls.status == LineSearchStatus::NumericalStall) rep.stalled = true;
        if (ls.step > 0.0 && ls.f <= fb) {
            rep.beta = ls.step;
            un = canonical(p, axpy(ub, rep.beta, d));
            fn = p.eval(un, gn);
            ++s.fevals;
            ++s.gevals;
        } else {
            un = ub;
            fn = fb;
            gn = gb;
        }
    }
    if (rep.restart)
        s.window.reset(un, gn);
    else
        s.window.push(un, gn);
    s.u = std::move(un);
    s.f = fn;
    s.g = std::move(gn);
    return rep;
}

// ngmres.cpp:160-200
MinimizeResult ngmres_minimize(const NgmresProblem& p, const Vector& initial, const NgmresOptions& o,
                               int record_iterates) {
    auto fit = [&](double f) { return p.fit_from_f ? p.fit_from_f(f) : 0.0; };
    const auto t0 = std::chrono::steady_clock::now();  // ngmres.cpp:162-164
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    NgmresState s = ngmres_init(p, initial, o);
    MinimizeResult res;
    auto record = [&](int it, bool restart, double beta) {
        res.trace.push_back({it, elapsed(), s.f, fit(s.f), norm(s.g) / p.gradient_scale, s.fevals, s.gevals, it, restart, beta});
    };
    record(0, false, 0.0);
    if (record_iterates > 0) res.iterates.push_back(s.u);
    Vector best_u = s.u;
    double best_f = s.f;
    StopReason stop = StopReason::MaxIters;
    int stalls = 0;
    for (int it = 1; it <= o.max_iters; ++it) {
        const NgmresStepReport rep = ngmres_step(p, s, o);
        record(it, rep.restart, rep.beta);
        if (static_cast<int>(res.iterates.size()) < record_iterates) res.iterates.push_back(s.u);
        if (s.f < best_f) {
            best_f = s.f;
            best_u = s.u;
        }
        stalls = rep.stalled ? stalls + 1 : 0;
        if (stalls >= 2) {
            stop = StopReason::Stalled;
            break;
        }
        if (norm(s.g) / p.gradient_scale <= o.tol_grad) {
            stop = StopReason::GradTol;
            break;
        }
    }
    res.u = best_u;
    res.f = best_f;
    res.stop = stop;
    return res;
}

// ngmres.cpp:202-226 with gradient_scale as a parameter.
MinimizeResult ngmres_cp(const DataTensor& t, const KruskalTensor& initial, const NgmresOptions& o,
                         double gradient_scale, int record_iterates) {
    const Shape shape = initial.shape();
    const index_t rank = initial.rank();
    if (!(t.shape() == shape)) throw std::invalid_argument("ngmres_solve: tensor and model shapes must match");
    NgmresProblem p;
    p.eval = [&t, shape, rank](const Vector& u, Vector& g) { return objective_and_gradient(t, unpack(u, shape, rank), g); };
    p.precondition = [&t, shape, rank](const Vector& u) { return pack(als_sweep(t, unpack(u, shape, rank))); };
    p.canonicalize = [shape, rank](const Vector& u) { return pack(normalize_and_reorder(unpack(u, shape, rank))); };
    p.gradient_scale = gradient_scale;
    p.fit_from_f = [sc = t.norm()](double f) { return std::sqrt(std::max(2.0 * f, 0.0)) / sc; };
    return ngmres_minimize(p, pack(initial), o, record_iterates);
}

// ---- ncg.cpp ---------------------------------------------------------------------------
MinimizeResult ncg_minimize(const std::function<double(const Vector&, Vector&)>& eval, const Vector& initial,
                            const NcgOptions& o, double gs, const std::function<double(double)>& fit_from_f) {
    if (!(o.tol_grad > 0.0)) throw std::invalid_argument("ncg: tol_grad must be > 0");
    auto fit = [&](double f) { return fit_from_f ? fit_from_f(f) : 0.0; };
    Vector u = initial, g;
    double f = eval(u, g);
    long fe = 1, ge = 1;
    MinimizeResult res;
    auto record = [&](int it, double fv, double gn, bool reset, double beta) {
        res.trace.push_back({it, 0.0, fv, fit(fv), gn / gs, fe, ge, 0, reset, beta});
    };
    record(0, f, norm(g), false, 0.0);
    Vector best_u = u;
    double best_f = f;
    res.stop = StopReason::MaxIters;
    if (norm(g) / gs <= o.tol_grad) {
        res.u = best_u;
        res.f = best_f;
        res.stop = StopReason::GradTol;
        return res;
    }
    Vector dir(g.size());
    for (size_t i = 0; i < g.size(); ++i) dir[i] = -g[i];
    int stalls = 0;
    for (int it = 1; it <= o.max_iters; ++it) {
        bool reset = false;
        double slope = dot(dir, g);
        if (slope >= 0.0) {
            for (size_t i = 0; i < g.size(); ++i) dir[i] = -g[i];
            slope = -dot(g, g);
            reset = true;
        }
        Vector gt;
        double last = -1.0;
        auto phi = [&](double step, double& fv, double& dg) {
            fv = eval(axpy(u, step, dir), gt);
            dg = dot(gt, dir);
            last = step;
        };
        const LineSearchResult ls = more_thuente(phi, f, slope, o.line_search);
        fe += ls.evals;
        ge += ls.evals;
        if (ls.step <= 0.0 || ls.f >= f) {
            if (++stalls >= 2) {
                res.stop = StopReason::Stalled;
                break;
            }
            for (size_t i = 0; i < g.size(); ++i) dir[i] = -g[i];
            continue;
        }
        stalls = 0;
        Vector un = axpy(u, ls.step, dir), gn;
        if (last == ls.step) {
            gn = gt;
        } else {
            eval(un, gn);
            ++fe;
            ++ge;
        }
        double num = 0.0;
        for (size_t i = 0; i < g.size(); ++i) num += gn[i] * (gn[i] - g[i]);
        const double pr = std::max(0.0, num / dot(g, g));
        for (size_t i = 0; i < g.size(); ++i) dir[i] = -gn[i] + pr * dir[i];
        u = std::move(un);
        f = ls.f;
        g = std::move(gn);
        const double gnorm = norm(g);
        record(it, f, gnorm, reset, ls.step);
        if (f < best_f) {
            best_f = f;
            best_u = u;
        }
        if (gnorm / gs <= o.tol_grad) {
            res.stop = StopReason::GradTol;
            break;
        }
    }
    res.u = best_u;
    res.f = best_f;
    return res;
}

}  // namespace oracle
