// phi(a) = f(u_bar + a d) as a polynomial (poly.cu builds the coefficients); evaluation in
// double-double because phi is a small difference of terms of size ||T||^2.
#pragma once

#include "common.cuh"

namespace cpfit_gpu {

constexpr int kPolyDeg = 8;   // f is of degree 2N in a: 6 for order 3 (coefficients 7, 8 zero), 8 for order 4
constexpr int kPolyDeg3 = 6;

// phi(a) and phi'(a) by Horner on the double-double coefficients coef[0..kPolyDeg]
__device__ __forceinline__ void poly_eval(const dd* coef, double a, double& f, double& g) {
    dd v = coef[kPolyDeg];
    dd dv = dd_mul(dd{(double)kPolyDeg, 0.0}, coef[kPolyDeg]);
    for (int k = kPolyDeg - 1; k >= 0; --k) {
        v = dd_add(dd_mul(v, dd{a, 0.0}), coef[k]);
        if (k >= 1) dv = dd_add(dd_mul(dv, dd{a, 0.0}), dd_mul(dd{(double)k, 0.0}, coef[k]));
    }
    f = v.hi + v.lo;
    g = dv.hi + dv.lo;
}

}  // namespace cpfit_gpu
