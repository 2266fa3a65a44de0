// Moré–Thuente strong-Wolfe line search as a resumable state machine
// (line_search.cpp:16-224), compiled for host and device.
//
// The reference runs the search as a loop around a callback. On the B200 every trial
// evaluation is a sequence of kernels inside a CUDA-graph WHILE node, so the search is
// re-expressed as begin() -> [caller evaluates phi(stp), phi'(stp)] -> update() until
// done: same constants, same branch order, same interval updates. The host C++ entry
// point cpfit::more_thuente drives the same object with a host callback.
#pragma once

#include <cmath>

namespace cpfit_gpu {

enum LsStatus : int { LS_CONVERGED = 0, LS_MAXEVALS = 1, LS_NOTDESCENT = 2, LS_STALL = 3, LS_RUNNING = -1 };

struct LsParams {
    double ftol = 1e-4, gtol = 1e-2, initial_step = 1.0;
    int max_evals = 20;
    double step_min = 0.0, step_max = 1e20;
};

struct MoreThuente {
    LsParams p;
    double phi0, dphi0, gtest, width, width1;
    double stx, fx, gx, sty, fy, gy;
    double stp, lo, hi;
    int bracketed, stage1;
    double best_s, best_f, best_g;
    int evals;
    int last_improved;
    int status;
    double out_step, out_f, out_g;

    __host__ __device__ static double dmax3(double a, double b, double c) { return fmax(a, fmax(b, c)); }
    __host__ __device__ static double clampd(double v, double a, double b) { return v < a ? a : (b < v ? b : v); }

    // line_search.cpp:129-147; returns false when no evaluation is needed (NotDescent).
    __host__ __device__ bool begin(const LsParams& prm, double f0, double g0) {
        p = prm;
        phi0 = f0;
        dphi0 = g0;
        evals = 0;
        if (g0 >= 0.0) {
            status = LS_NOTDESCENT;
            out_step = 0.0;
            out_f = f0;
            out_g = g0;
            return false;
        }
        status = LS_RUNNING;
        gtest = p.ftol * g0;
        width = p.step_max - p.step_min;
        width1 = 2.0 * width;
        stx = 0.0;
        fx = f0;
        gx = g0;
        sty = 0.0;
        fy = f0;
        gy = g0;
        stp = clampd(p.initial_step, fmax(p.step_min, 1e-300), p.step_max);
        lo = 0.0;
        hi = stp + 4.0 * stp;
        bracketed = 0;
        stage1 = 1;
        best_s = 0.0;
        best_f = f0;
        best_g = g0;
        return true;
    }

    __host__ __device__ void finish(int st, double s, double f, double g) {
        status = st;
        out_step = s;
        out_f = f;
        out_g = g;
    }

    // One trial result (f, g) at the current stp (line_search.cpp:160-222). Returns true
    // when the search has terminated (status/out_* set); otherwise stp holds the next trial.
    __host__ __device__ bool update(double f, double g) {
        ++evals;
        last_improved = (f < best_f) ? 1 : 0;  // lets the caller keep the best trial's data
        if (f < best_f) {
            best_s = stp;
            best_f = f;
            best_g = g;
        }
        const double ftest = phi0 + stp * gtest;
        if (stage1 && f <= ftest && g >= fmin(p.ftol, p.gtol) * dphi0) stage1 = 0;
        if (f <= ftest && fabs(g) <= p.gtol * (-dphi0)) {
            finish(LS_CONVERGED, stp, f, g);
            return true;
        }
        if (evals >= p.max_evals) {
            finish(LS_MAXEVALS, best_s, best_f, best_g);
            return true;
        }
        if (bracketed && (stp <= lo || stp >= hi)) {
            finish(LS_STALL, best_s, best_f, best_g);
            return true;
        }
        if (bracketed && hi - lo <= 1e-15 * hi) {
            finish(LS_STALL, best_s, best_f, best_g);
            return true;
        }
        if (stp == p.step_max && f <= ftest && g <= gtest) {
            finish(LS_MAXEVALS, best_s, best_f, best_g);
            return true;
        }
        if (stp == p.step_min && (f > ftest || g >= gtest)) {
            finish(LS_STALL, best_s, best_f, best_g);
            return true;
        }
        if (stage1 && f <= fx && f > ftest) {
            // modified function psi(s) = phi(s) - phi0 - s*gtest in stage 1
            double fm = f - stp * gtest, fxm = fx - stx * gtest, fym = fy - sty * gtest;
            double gm = g - gtest, gxm = gx - gtest, gym = gy - gtest;
            stp = cstep(stx, fxm, gxm, sty, fym, gym, stp, fm, gm);
            fx = fxm + stx * gtest;
            fy = fym + sty * gtest;
            gx = gxm + gtest;
            gy = gym + gtest;
        } else {
            stp = cstep(stx, fx, gx, sty, fy, gy, stp, f, g);
        }
        if (bracketed) {
            if (fabs(sty - stx) >= 0.66 * width1) stp = stx + 0.5 * (sty - stx);
            width1 = width;
            width = fabs(sty - stx);
            lo = fmin(stx, sty);
            hi = fmax(stx, sty);
        } else {
            lo = stp + 1.1 * (stp - stx);
            hi = stp + 4.0 * (stp - stx);
        }
        stp = clampd(stp, p.step_min, p.step_max);
        if ((bracketed && (stp <= lo || stp >= hi)) || (bracketed && hi - lo <= 1e-15 * hi)) stp = stx;
        if (stp <= 0.0) stp = (hi > 0.0) ? 0.5 * hi : p.initial_step;
        return false;
    }

    // Safeguarded cubic/quadratic step (line_search.cpp:16-108).
    __host__ __device__ double cstep(double& sx, double& fxv, double& dx, double& sy, double& fyv, double& dy,
                                     double sp, double fp, double dp) {
        const double sgnd = dp * (dx >= 0.0 ? 1.0 : -1.0);
        double next = sp;
        if (fp > fxv) {
            const double theta = 3.0 * (fxv - fp) / (sp - sx) + dx + dp;
            const double s = dmax3(fabs(theta), fabs(dx), fabs(dp));
            double gam = s * sqrt((theta / s) * (theta / s) - (dx / s) * (dp / s));
            if (sp < sx) gam = -gam;
            const double pp = (gam - dx) + theta;
            const double q = ((gam - dx) + gam) + dp;
            const double stpc = sx + (pp / q) * (sp - sx);
            const double stpq = sx + ((dx / ((fxv - fp) / (sp - sx) + dx)) / 2.0) * (sp - sx);
            next = (fabs(stpc - sx) < fabs(stpq - sx)) ? stpc : stpc + (stpq - stpc) / 2.0;
            bracketed = 1;
        } else if (sgnd < 0.0) {
            const double theta = 3.0 * (fxv - fp) / (sp - sx) + dx + dp;
            const double s = dmax3(fabs(theta), fabs(dx), fabs(dp));
            double gam = s * sqrt((theta / s) * (theta / s) - (dx / s) * (dp / s));
            if (sp > sx) gam = -gam;
            const double pp = (gam - dp) + theta;
            const double q = ((gam - dp) + gam) + dx;
            const double stpc = sp + (pp / q) * (sx - sp);
            const double stpq = sp + (dp / (dp - dx)) * (sx - sp);
            next = (fabs(stpc - sp) > fabs(stpq - sp)) ? stpc : stpq;
            bracketed = 1;
        } else if (fabs(dp) < fabs(dx)) {
            const double theta = 3.0 * (fxv - fp) / (sp - sx) + dx + dp;
            const double s = dmax3(fabs(theta), fabs(dx), fabs(dp));
            double gam = s * sqrt(fmax(0.0, (theta / s) * (theta / s) - (dx / s) * (dp / s)));
            if (sp > sx) gam = -gam;
            const double pp = (gam - dp) + theta;
            const double q = (gam + (dx - dp)) + gam;
            const double r = pp / q;
            double stpc;
            if (r < 0.0 && gam != 0.0)
                stpc = sp + r * (sx - sp);
            else if (sp > sx)
                stpc = hi;
            else
                stpc = lo;
            const double stpq = sp + (dp / (dp - dx)) * (sx - sp);
            if (bracketed) {
                next = (fabs(stpc - sp) < fabs(stpq - sp)) ? stpc : stpq;
                next = (sp > sx) ? fmin(sp + 0.66 * (sy - sp), next) : fmax(sp + 0.66 * (sy - sp), next);
            } else {
                next = (fabs(stpc - sp) > fabs(stpq - sp)) ? stpc : stpq;
                next = clampd(next, lo, hi);
            }
        } else {
            if (bracketed) {
                const double theta = 3.0 * (fp - fyv) / (sy - sp) + dy + dp;
                const double s = dmax3(fabs(theta), fabs(dy), fabs(dp));
                double gam = s * sqrt((theta / s) * (theta / s) - (dy / s) * (dp / s));
                if (sp > sy) gam = -gam;
                const double pp = (gam - dp) + theta;
                const double q = ((gam - dp) + gam) + dy;
                next = sp + (pp / q) * (sy - sp);
            } else {
                next = (sp > sx) ? hi : lo;
            }
        }
        if (fp > fxv) {
            sy = sp;
            fyv = fp;
            dy = dp;
        } else {
            if (sgnd < 0.0) {
                sy = sx;
                fyv = fxv;
                dy = dx;
            }
            sx = sp;
            fxv = fp;
            dx = dp;
        }
        return next;
    }
};

}  // namespace cpfit_gpu
