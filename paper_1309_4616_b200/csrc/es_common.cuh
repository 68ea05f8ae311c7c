// Shared device/host definitions for the expstencil_b200 kernels.
//
// Arithmetic rule: every fp64 operation on the reference's expression trees
// uses the explicit round-to-nearest intrinsics (__dadd_rn, __dmul_rn, ...),
// which nvcc never contracts into DFMA, and the library is additionally
// compiled with -fmad=false.  That reproduces the reference's
// -ffp-contract=off Cython core bit for bit (reference setup.py:5-15).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/expstencil_b200.h"

#define ES_DEV __device__ __forceinline__

namespace es {

ES_DEV double add(double a, double b) { return __dadd_rn(a, b); }
ES_DEV double sub(double a, double b) { return __dsub_rn(a, b); }
ES_DEV double mul(double a, double b) { return __dmul_rn(a, b); }
ES_DEV double div(double a, double b) { return __ddiv_rn(a, b); }
ES_DEV double sqrt_rn(double a) { return __dsqrt_rn(a); }

// Per-point stencil value, expression tree of _core.pyx:116-122:
//   sx = (2c - xm - xp) wx; sy, sz alike; lap = (sx + sy) + sz;
//   lap = D lap (coefficient); [Rosenbrock: lap = lap - g' c];
//   out = alpha lap + beta c
ES_DEV double lap7(double c, double xm, double xp, double ym, double yp, double zm, double zp,
                   double wx, double wy, double wz) {
    const double c2 = mul(2.0, c);
    const double sx = mul(sub(sub(c2, xm), xp), wx);
    const double sy = mul(sub(sub(c2, ym), yp), wy);
    const double sz = mul(sub(sub(c2, zm), zp), wz);
    return add(add(sx, sy), sz);
}

// The compiled core's C99 `double complex` product under -ffp-contract=off
// (_core.pyx:263-278; real operands promoted to (v, 0)).
ES_DEV double2 cmul_c(double ar, double ai, double br, double bi) {
    return make_double2(sub(mul(ar, br), mul(ai, bi)), add(mul(ar, bi), mul(ai, br)));
}

// D(x, y) = 1/sqrt((1 + x*x) + y*y) with x = (ix+1)/(nx+1) (grid.py:80-83,
// bench.py:40-41): correctly rounded div/sqrt reproduce numpy's sampling.
ES_DEV double axis_coord(int64_t i, int64_t n) { return div((double)(i + 1), (double)(n + 1)); }
// __drcp_rn is the correctly rounded 1/s, i.e. bit-identical to
// __ddiv_rn(1.0, s), with a shorter refinement sequence.
ES_DEV double radial_from_sq(double one_plus_x2, double y) {
    return __drcp_rn(sqrt_rn(add(one_plus_x2, mul(y, y))));
}

// ordered-integer image of a double (monotone in the value) for atomic
// min/max; inverse: b = (o >> 63) ? (o & ~sign) : ~o
ES_DEV unsigned long long ord(double d) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

struct SeriesState {
    int k;            // last completed node (0 = none yet)
    int consecutive;  // consecutive passes of the term test
    int done;         // series finished (converged, tol == 0 exhausted, or failed)
    int converged;    // 1 unless the degree budget ran out with tol > 0
    double last_term;
    double last_pnorm;
    int pass;  // two-node series (stencil_tb.cuh): HBM passes completed (selects the w buffers / halo parity)
    int pad_;
};

// Outcome of the fused small-grid exponential-Euler step, written by the
// kernel into host-mapped pinned memory (series_small.cu, step.cu)
struct SmallStepRecord {
    SeriesState a, b;
    unsigned long long bad;
};

}  // namespace es
