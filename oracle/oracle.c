/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot path (arXiv 1309.4616 reference,
 * package `expstencil`).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference legs may load this library, and only as the
 * checker or the timed CPU baseline -- never as the product path.
 *
 * Pinning: tests/test_oracle_golden.py checks every function below against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py
 * imports the reference built by oracle/build_ref.sh).  Neumann boundaries and
 * the Rosenbrock operator M = A - diag(g') do not exist in the reference; they
 * are build-defined here and pinned only against the
 * dense-matrix oracles in the tests.
 *
 * Build flags: -O2 -ffp-contract=off, no -ffast-math (mirrors the reference
 * setup.py:5-15), so every per-point expression rounds exactly like the
 * reference's Cython core.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MODE_ZERO 0
#define ORC_MODE_PERIODIC 1
#define ORC_MODE_FACES 2
#define ORC_MODE_NEUMANN 3

#define ORC_COEFF_NONE 0
#define ORC_COEFF_RADIAL 1
#define ORC_COEFF_ARRAY 2

typedef struct {
    int64_t nx, ny, lz;     /* slab extents; x fastest (grid.py:96-102) */
    int64_t z0, nz_total;   /* global z offset of the slab, total planes */
    double wx, wy, wz;      /* host-computed 1/dx^2 (stencil.py:116-122) */
    int32_t mode;           /* ghost rule, ORC_MODE_* */
    int32_t coeff_kind;     /* ORC_COEFF_* */
    const double *coeff;    /* (lz, ny, nx) slab-local, ORC_COEFF_ARRAY */
    const double *faces[6]; /* fx_lo,fx_hi (nz_total,ny); fy_lo,fy_hi (nz_total,nx); fz_lo,fz_hi (ny,nx) */
    const double *halo_lo;  /* (ny, nx) plane below the slab or NULL */
    const double *halo_hi;  /* (ny, nx) plane above the slab or NULL */
    const double *gdiag;    /* Rosenbrock diag g'(u_n) (lz,ny,nx) or NULL */
} orc_slab;

/* Radial diffusion coefficient D(x,y) = 1/sqrt(1+x^2+y^2) sampled at the
 * interior point (ix,iy); coordinates as grid.py:80-83, expression tree as
 * bench.py:40-41 (numpy evaluates (1 + x*x) + y*y). */
static double radial_coeff(int64_t ix, int64_t iy, int64_t nx, int64_t ny) {
    double x = (double)(ix + 1) / (double)(nx + 1);
    double y = (double)(iy + 1) / (double)(ny + 1);
    return 1.0 / sqrt((1.0 + x * x) + y * y);
}

/* One output point; follows _core.pyx:42-122 (ghost precedence: interior,
 * halo (z only), periodic wrap, face value, Neumann mirror, zero). */
static double orc_point(const orc_slab *s, const double *u, double alpha, double beta,
                        int64_t iz, int64_t iy, int64_t ix) {
    const int64_t nx = s->nx, ny = s->ny, lz = s->lz;
    const int64_t plane = nx * ny;
    const int64_t idx = ix + nx * (iy + ny * iz);
    const double c = u[idx];
    const int mode = s->mode;
    const int at_z_lo = s->z0 == 0;
    const int at_z_hi = s->z0 + lz == s->nz_total;
    double xm, xp, ym, yp, zm, zp;

    if (ix > 0) xm = u[idx - 1];
    else if (mode == ORC_MODE_PERIODIC) xm = u[idx + nx - 1];
    else if (mode == ORC_MODE_FACES) xm = s->faces[0][(s->z0 + iz) * ny + iy];
    else if (mode == ORC_MODE_NEUMANN) xm = c;
    else xm = 0.0;
    if (ix < nx - 1) xp = u[idx + 1];
    else if (mode == ORC_MODE_PERIODIC) xp = u[idx - (nx - 1)];
    else if (mode == ORC_MODE_FACES) xp = s->faces[1][(s->z0 + iz) * ny + iy];
    else if (mode == ORC_MODE_NEUMANN) xp = c;
    else xp = 0.0;

    if (iy > 0) ym = u[idx - nx];
    else if (mode == ORC_MODE_PERIODIC) ym = u[idx + (ny - 1) * nx];
    else if (mode == ORC_MODE_FACES) ym = s->faces[2][(s->z0 + iz) * nx + ix];
    else if (mode == ORC_MODE_NEUMANN) ym = c;
    else ym = 0.0;
    if (iy < ny - 1) yp = u[idx + nx];
    else if (mode == ORC_MODE_PERIODIC) yp = u[idx - (ny - 1) * nx];
    else if (mode == ORC_MODE_FACES) yp = s->faces[3][(s->z0 + iz) * nx + ix];
    else if (mode == ORC_MODE_NEUMANN) yp = c;
    else yp = 0.0;

    if (iz > 0) zm = u[idx - plane];
    else if (s->halo_lo) zm = s->halo_lo[iy * nx + ix];
    else if (mode == ORC_MODE_PERIODIC) zm = u[idx + (lz - 1) * plane];
    else if (mode == ORC_MODE_FACES && at_z_lo) zm = s->faces[4][iy * nx + ix];
    else if (mode == ORC_MODE_NEUMANN && at_z_lo) zm = c;
    else zm = 0.0;
    if (iz < lz - 1) zp = u[idx + plane];
    else if (s->halo_hi) zp = s->halo_hi[iy * nx + ix];
    else if (mode == ORC_MODE_PERIODIC) zp = u[idx - (lz - 1) * plane];
    else if (mode == ORC_MODE_FACES && at_z_hi) zp = s->faces[5][iy * nx + ix];
    else if (mode == ORC_MODE_NEUMANN && at_z_hi) zp = c;
    else zp = 0.0;

    const double two = 2.0;
    double sx = (two * c - xm - xp) * s->wx;
    double sy = (two * c - ym - yp) * s->wy;
    double sz = (two * c - zm - zp) * s->wz;
    double lap = (sx + sy) + sz;
    if (s->coeff_kind == ORC_COEFF_ARRAY) lap = s->coeff[idx] * lap;
    else if (s->coeff_kind == ORC_COEFF_RADIAL) lap = radial_coeff(ix, iy, nx, ny) * lap;
    if (s->gdiag) lap = lap - s->gdiag[idx] * c; /* build-defined Rosenbrock row */
    return alpha * lap + beta * c;
}

/* out = alpha * (D A u) + beta * u over one slab (_core.pyx:176-226). */
void orc_stencil_fused_slab(const orc_slab *s, const double *u, double *out, double alpha,
                            double beta) {
    const int64_t nx = s->nx, ny = s->ny, lz = s->lz;
#pragma omp parallel for schedule(static)
    for (int64_t iz = 0; iz < lz; ++iz)
        for (int64_t iy = 0; iy < ny; ++iy)
            for (int64_t ix = 0; ix < nx; ++ix)
                out[ix + nx * (iy + ny * iz)] = orc_point(s, u, alpha, beta, iz, iy, ix);
}

/* Sum of squares with a fixed, thread-count-independent order: per z-plane
 * sequential partials, then planes in order. */
static double orc_sumsq_planes(const double *x, int64_t plane, int64_t nplanes, double *scratch) {
#pragma omp parallel for schedule(static)
    for (int64_t z = 0; z < nplanes; ++z) {
        const double *q = x + z * plane;
        double acc = 0.0;
        for (int64_t i = 0; i < plane; ++i) acc += q[i] * q[i];
        scratch[z] = acc;
    }
    double tot = 0.0;
    for (int64_t z = 0; z < nplanes; ++z) tot += scratch[z];
    return tot;
}

/*
 * Newton-Leja series on a stencil slab (restates matfunc.newton_apply,
 * matfunc.py:271-318) as ONE fused pass per node: w_k = (alpha A + beta_k I)
 * w_{k-1}, p_k = p_{k-1} + dd_k w_k, with p_0 = dd_0 v folded into node 1.
 * Returns 0 when the series stopped (converged, or tol == 0), 2 when the
 * degree budget ran out (ConvergenceError).  ws: 2*n doubles + nz doubles.
 */
int orc_newton_stencil(const orc_slab *s, const double *v, double *p, const double *dd,
                       const double *xi, int32_t ndd, double alpha, double shift, double tol,
                       double *ws, int32_t *matvecs, double *last_term, double *last_pnorm) {
    const int64_t nx = s->nx, ny = s->ny, lz = s->lz;
    const int64_t n = nx * ny * lz, plane = nx * ny;
    double *wa = ws, *wb = ws + n, *part = ws + 2 * n;
    *matvecs = 0;
    *last_term = INFINITY;
    *last_pnorm = 0.0;
    const double d0 = dd[0];
    for (int64_t i = 0; i < n; ++i) p[i] = d0 * v[i];
    if (ndd == 1) return 0;
    const double *wsrc = v;
    int consecutive = 0;
    for (int32_t k = 1; k < ndd; ++k) {
        double beta = -shift - xi[k - 1];
        double *wdst = (k & 1) ? wa : wb;
        orc_stencil_fused_slab(s, wsrc, wdst, alpha, beta);
        const double dk = dd[k];
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) p[i] = p[i] + dk * wdst[i];
        *matvecs = k;
        double term = fabs(dk) * sqrt(orc_sumsq_planes(wdst, plane, lz, part));
        double pn = sqrt(orc_sumsq_planes(p, plane, lz, part));
        *last_term = term;
        *last_pnorm = pn;
        if (tol > 0) {
            if (term <= tol * pn) {
                if (++consecutive >= 2) return 0;
            } else {
                consecutive = 0;
            }
        }
        wsrc = wdst;
    }
    return tol == 0 ? 0 : 2;
}

/* y[r] = alpha * sum_k vals[k] x[col[k]] (+ beta x[r]) accumulated strictly in
 * storage order (_core.pyx:245-260). */
void orc_csr_fused_rows(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr,
                        const int32_t *col, const double *vals, const double *x, double *y,
                        double alpha, double beta, int use_beta) {
#pragma omp parallel for schedule(static)
    for (int64_t r = row_lo; r < row_hi; ++r) {
        double acc = 0.0;
        for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) acc = acc + vals[k] * x[col[k]];
        y[r] = use_beta ? alpha * acc + beta * x[r] : alpha * acc;
    }
}

/* Newton-Leja series for a square CSR operator (same loop as above). ws: 2n. */
int orc_newton_csr(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *vals,
                   const double *v, double *p, const double *dd, const double *xi, int32_t ndd,
                   double alpha, double shift, double tol, double *ws, int32_t *matvecs,
                   double *last_term, double *last_pnorm) {
    double *wa = ws, *wb = ws + n;
    *matvecs = 0;
    *last_term = INFINITY;
    *last_pnorm = 0.0;
    for (int64_t i = 0; i < n; ++i) p[i] = dd[0] * v[i];
    if (ndd == 1) return 0;
    const double *wsrc = v;
    int consecutive = 0;
    for (int32_t k = 1; k < ndd; ++k) {
        double beta = -shift - xi[k - 1];
        double *wdst = (k & 1) ? wa : wb;
        orc_csr_fused_rows(0, n, row_ptr, col, vals, wsrc, wdst, alpha, beta, 1);
        const double dk = dd[k];
        double sw = 0.0, sp = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            p[i] = p[i] + dk * wdst[i];
            sw += wdst[i] * wdst[i];
            sp += p[i] * p[i];
        }
        *matvecs = k;
        double term = fabs(dk) * sqrt(sw);
        double pn = sqrt(sp);
        *last_term = term;
        *last_pnorm = pn;
        if (tol > 0) {
            if (term <= tol * pn) {
                if (++consecutive >= 2) return 0;
            } else {
                consecutive = 0;
            }
        }
        wsrc = wdst;
    }
    return tol == 0 ? 0 : 2;
}

/* ---- complex CSR (the propagate path, cli.py:304-357) -------------------
 * Vectors are interleaved (re, im) pairs.  Two complex products appear:
 *   cmul_c: the reference's compiled core, C99 `double complex` a*b under
 *           -ffp-contract=off (_core.pyx:263-278, GCC lowering):
 *           (a.r b.r - a.i b.i, a.r b.i + a.i b.r), a real vals[k] promoted
 *           to (v, 0) first (Cython __pyx_t_double_complex_from_parts);
 *   cmul_np: numpy's complex128 multiply as measured on this build
 *           (p += dd[k] * w, matfunc.py:300):
 *           (fma(a.r, b.r, -(a.i b.i)), fma(a.r, b.i, a.i b.r)). */
static inline void cmul_c(double ar, double ai, double br, double bi, double *cr, double *ci) {
    double ac = ar * br, bd = ai * bi, ad = ar * bi, bc = ai * br;
    *cr = ac - bd;
    *ci = ad + bc;
}
static inline void cmul_np(double ar, double ai, double br, double bi, double *cr, double *ci) {
    *cr = fma(ar, br, -(ai * bi));
    *ci = fma(ar, bi, ai * br);
}

/* y[r] = alpha (sum_k vals[k] x[col[k]]) (+ beta x[r]); vals real
 * (vals_complex = 0) or interleaved complex; alpha, beta complex. */
void orc_csr_fused_rows_z(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr, const int32_t *col,
                          const double *vals, int vals_complex, const double *x, double *y, double alpha_r,
                          double alpha_i, double beta_r, double beta_i, int use_beta) {
#pragma omp parallel for schedule(static)
    for (int64_t r = row_lo; r < row_hi; ++r) {
        double acc_r = 0.0, acc_i = 0.0;
        for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            const double vr = vals_complex ? vals[2 * k] : vals[k], vi = vals_complex ? vals[2 * k + 1] : 0.0;
            double pr, pi;
            cmul_c(vr, vi, x[2 * (int64_t)col[k]], x[2 * (int64_t)col[k] + 1], &pr, &pi);
            acc_r = acc_r + pr;
            acc_i = acc_i + pi;
        }
        double yr, yi;
        cmul_c(alpha_r, alpha_i, acc_r, acc_i, &yr, &yi);
        if (use_beta) {
            double br, bi;
            cmul_c(beta_r, beta_i, x[2 * r], x[2 * r + 1], &br, &bi);
            yr = yr + br;
            yi = yi + bi;
        }
        y[2 * r] = yr;
        y[2 * r + 1] = yi;
    }
}

/* Complex Newton-Leja series (matfunc.py:271-318 with complex dd / v):
 * w_k = (alpha A + beta_k) w_{k-1} through the complex core, p += dd_k w_k
 * with numpy's product, term = |dd_k| ||w_k|| (ddabs = numpy abs(dd)).
 * ws: 4n doubles. */
int orc_newton_csr_z(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *vals, int vals_complex,
                     const double *v, double *p, const double *dd, const double *ddabs, const double *xi,
                     int32_t ndd, double alpha_r, double alpha_i, double shift, double tol, double *ws,
                     int32_t *matvecs, double *last_term, double *last_pnorm) {
    double *wa = ws, *wb = ws + 2 * n;
    *matvecs = 0;
    *last_term = INFINITY;
    *last_pnorm = 0.0;
    for (int64_t i = 0; i < n; ++i) cmul_np(dd[0], dd[1], v[2 * i], v[2 * i + 1], &p[2 * i], &p[2 * i + 1]);
    if (ndd == 1) return 0;
    const double *wsrc = v;
    int consecutive = 0;
    for (int32_t k = 1; k < ndd; ++k) {
        double beta = -shift - xi[k - 1];
        double *wdst = (k & 1) ? wa : wb;
        orc_csr_fused_rows_z(0, n, row_ptr, col, vals, vals_complex, wsrc, wdst, alpha_r, alpha_i, beta, 0.0, 1);
        double sw = 0.0, sp = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double tr, ti;
            cmul_np(dd[2 * k], dd[2 * k + 1], wdst[2 * i], wdst[2 * i + 1], &tr, &ti);
            p[2 * i] = p[2 * i] + tr;
            p[2 * i + 1] = p[2 * i + 1] + ti;
            sw += wdst[2 * i] * wdst[2 * i] + wdst[2 * i + 1] * wdst[2 * i + 1];
            sp += p[2 * i] * p[2 * i] + p[2 * i + 1] * p[2 * i + 1];
        }
        *matvecs = k;
        double term = ddabs[k] * sqrt(sw);
        double pn = sqrt(sp);
        *last_term = term;
        *last_pnorm = pn;
        if (tol > 0) {
            if (term <= tol * pn) {
                if (++consecutive >= 2) return 0;
            } else {
                consecutive = 0;
            }
        }
        wsrc = wdst;
    }
    return tol == 0 ? 0 : 2;
}

/* out = (1/4 (2 - u)) exp(20 (1 - 1/u)) (_core.pyx:325-338); returns the first
 * index with u <= 0 (integrator.py:43-49) or -1. */
int64_t orc_combustion(const double *u, double *out, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (u[i] <= 0.0) return i;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double r = 1.0 / u[i];
        double t = 20.0 * (1.0 - r);
        out[i] = (0.25 * (2.0 - u[i])) * exp(t);
    }
    return -1;
}

/* Build-defined Jacobian diagonal of the combustion term:
 * g'(u) = e^{20(1-1/u)} (-1/4 + 5 (2-u)/u^2). */
void orc_combustion_jac(const double *u, double *out, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double r = 1.0 / u[i];
        double e = exp(20.0 * (1.0 - r));
        double q = (5.0 * (2.0 - u[i])) * (r * r);
        out[i] = e * (q - 0.25);
    }
}

/* out = y + h z (integrator.py:187, numpy rounding: y + fl(h*z)). */
void orc_axpy_step(const double *y, const double *z, double h, double *out, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = y[i] + h * z[i];
}

int orc_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
