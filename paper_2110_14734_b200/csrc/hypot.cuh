// hypot.cuh -- np.hypot as x86-64 numpy computes it: glibc 2.39's
// sysdeps/ieee754/dbl-64/e_hypot.c (2.35+), the non-FMA Borges kernel with its
// scaling branches, restated operation for operation;
// verified bit-exact against libm in tests/.  Used by the spanner arc costs
// (spanner.py:324), the dense oracle network (oracle.py:79) and WCD
// (lower_bound.py:92).
#pragma once

#include "common.cuh"

namespace w1g {

__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
    double t1, t2;
    double h = dsqrt(dadd(dmul(ax, ax), dmul(ay, ay)));
    if (h <= dmul(2.0, ay)) {
        const double delta = dsub(h, ay);
        t1 = dmul(ax, dsub(dmul(2.0, delta), ax));
        t2 = dmul(dsub(delta, dmul(2.0, dsub(ax, ay))), delta);
    } else {
        const double delta = dsub(h, ax);
        t1 = dmul(dmul(2.0, delta), dsub(ax, dmul(2.0, ay)));
        t2 = dadd(dmul(dsub(dmul(4.0, delta), ay), ay), dmul(delta, delta));
    }
    // an exact h (t1 + t2 == +-0: h - (+-0) / 2h is h) skips the division -- and its slow
    // path, which a zero quotient takes (lattice points give exact distances often)
    const double num = dadd(t1, t2);
    return num == 0.0 ? h : dsub(h, ddiv(num, dmul(2.0, h)));
}

__device__ __forceinline__ double glibc_hypot(double x, double y) {
    if (!isfinite(x) || !isfinite(y)) {
        if (isinf(x) || isinf(y)) return INFINITY;
        return dadd(x, y);
    }
    x = fabs(x);
    y = fabs(y);
    double ax = x < y ? y : x, ay = x < y ? x : y;
    if (ax > 0x1p+511) {
        if (ay <= dmul(ax, 0x1p-54)) return dadd(ax, ay);
        return ddiv(hypot_kernel(dmul(ax, 0x1p-600), dmul(ay, 0x1p-600)), 0x1p-600);
    }
    if (ay < 0x1p-511) {
        if (ax >= ddiv(ay, 0x1p-54)) return dadd(ax, ay);
        return dmul(hypot_kernel(ddiv(ax, 0x1p-600), ddiv(ay, 0x1p-600)), 0x1p-600);
    }
    if (ay <= dmul(ax, 0x1p-54)) return dadd(ax, ay);
    return hypot_kernel(ax, ay);
}

}  // namespace w1g
