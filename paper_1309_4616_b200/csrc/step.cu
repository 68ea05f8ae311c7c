// Fused integrator steps: one C call per step, one host synchronisation.
//
// Exponential Euler (integrator.py:177-189): y = exp(-hA) u and
// z = phi1(-hA) g_n are independent series over the same operator, so they
// run concurrently -- the exp series on the caller's stream, g_n = g(u) - b
// and the phi1 series on a side stream forked from it -- and join before
// u_out = y + h z.  At small grids (C1: 65,536 points, latency-bound nodes)
// the two series' node chains overlap almost completely; at HBM-bound sizes
// they share the bandwidth and the step costs what the two series cost.
//
// Exponential Rosenbrock-Euler (build-defined): the
// fused prologue (F = g(u) - A u, g' and its range in one stencil pass), the
// interval check against the interval the caller's divided differences were
// built for (Python's snap_interval, restated bit for bit), the series on
// M = A - diag(g'), and u_out = u + h z.
//
// The final combination is guarded on the device by the series states, so a
// series that ran out of nodes leaves y / F / g_n intact for the caller's
// halving rescue (matfunc.py:328-373).
#include <cmath>
#include <cstring>

#include "es_common.cuh"
#include "es_host.h"
#include "stencil.cuh"

namespace es {

namespace {

struct Fork {
    int device = -1;
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, t0 = nullptr, t1 = nullptr;
    unsigned long long *bad = nullptr, *bad_host = nullptr;
    SmallStepRecord *rec_host = nullptr, *rec_dev = nullptr;  // host-mapped outcome of the small-grid step
};
thread_local Fork t_fork;

int fork_resources(Fork *&f) {
    f = &t_fork;
    const int dev = current_device();
    if (f->device == dev) return ES_OK;
    if (cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f->join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreate(&f->t0) != cudaSuccess || cudaEventCreate(&f->t1) != cudaSuccess ||
        cudaMalloc(&f->bad, 2 * sizeof(unsigned long long)) != cudaSuccess ||  // k_fill_u64 writes two words
        cudaMallocHost(&f->bad_host, sizeof(unsigned long long)) != cudaSuccess ||
        cudaHostAlloc(&f->rec_host, sizeof(SmallStepRecord), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&f->rec_dev, f->rec_host, 0) != cudaSuccess)
        return check_launch("step resources");
    f->device = dev;
    return ES_OK;
}

// out = y + h z, only if every given series finished converged
__global__ void k_axpy_if(const double *__restrict__ y, const double *z, double h, double *out, int64_t n,
                          const SeriesState *a, const SeriesState *b) {
    if ((a && a->converged != 1) || (b && b->converged != 1)) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = add(y[i], mul(h, z[i]));
}

unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>(std::max<int64_t>((n + 255) / 256, 1), 148 * 32); }

int series_status(int rc, int32_t *status) {
    *status = rc == ES_ERR_NOT_CONVERGED ? ES_ERR_NOT_CONVERGED : ES_OK;
    return rc == ES_ERR_NOT_CONVERGED ? ES_OK : rc;
}

}  // namespace

int run_expeuler_step(const es_stencil_desc *d, const double *u, double *u_out, const double *dd_exp, int ndd_exp,
                      const double *dd_phi, int ndd_phi, const double *xi, double alpha, double shift, double tol,
                      double h, int nonlin, const double *source, double *scratch, void *ws_exp, void *ws_phi,
                      size_t ws_bytes, es_step_result *res, cudaStream_t s) {
    const int64_t n = d->nx * d->ny * d->lz;
    *res = es_step_result{};
    res->first_bad = -1;
    Fork *f;
    int rc = fork_resources(f);
    if (rc) return rc;
    const bool phi = nonlin == ES_NONLIN_COMBUSTION || source != nullptr;
    double *g = scratch, *z = scratch + n;
    // tiny grids: both series, g(u) - b and the combination in ONE persistent
    // launch (series_small.cu); otherwise two concurrent series graphs
    bool fused = false;
    if (phi) {
        SeriesParams ha, hb;
        SeriesParams *da = nullptr, *db = nullptr;
        StencilPlan pa, pb;
        bool oka = false, okb = false;
        rc = small_prepare(d, u, u_out, dd_exp, xi, ndd_exp, alpha, shift, tol, nullptr, ws_exp, ws_bytes, 2, &ha, &da,
                           &pa, &oka, s);
        if (!rc && oka)
            rc = small_prepare(d, g, z, dd_phi, xi, ndd_phi, alpha, shift, tol, nullptr, ws_phi, ws_bytes, 2, &hb, &db,
                               &pb, &okb, s);
        if (rc) return rc;
        if (oka && okb && pa.nchunks == pb.nchunks && pa.chunk == pb.chunk) {
            cudaEventRecord(f->t0, s);
            if ((rc = launch_expeuler_small_init(&ha, da, &hb, db, f->bad, n, s))) return rc;
            if ((rc = launch_expeuler_small(d, da, db, pa, u, g, source, nonlin, h, f->bad, f->rec_dev, s))) return rc;
            cudaEventRecord(f->t1, s);
            // both states and the domain word arrive in host-mapped memory: one sync, no copies
            if (cudaStreamSynchronize(s) != cudaSuccess) return check_launch("small-grid step sync");
            SmallStepRecord rec;
            std::memcpy(&rec, f->rec_host, sizeof(rec));  // written by the kernel, complete after the sync
            *f->bad_host = rec.bad;
            rc = series_status(series_result_of(rec.a, &res->exp_series), &res->status_exp);
            if (!rc) rc = series_status(series_result_of(rec.b, &res->phi1_series), &res->status_phi1);
            if (rc) return rc;
            fused = true;
        }
    }
    if (!fused) cudaEventRecord(f->t0, s);
    // ES_STEP_SERIAL=1: the phi1 series on the caller's stream after the exp
    // series (diagnostics; the default forks it onto a side stream)
    cudaStream_t side = env_int("ES_STEP_SERIAL", 0) ? s : f->side;
    if (phi && !fused) {
        cudaEventRecord(f->fork, s);
        cudaStreamWaitEvent(side, f->fork, 0);
    }
    if (!fused)
        rc = run_stencil_series(d, u, u_out, dd_exp, xi, ndd_exp, alpha, shift, tol, nullptr, ws_exp, ws_bytes, nullptr,
                                s);
    if (!rc && phi && !fused) {
        if (nonlin == ES_NONLIN_COMBUSTION) {
            rc = launch_combustion(u, g, n, f->bad, side);
            if (!rc && source) rc = launch_axpy(g, source, -1.0, g, n, side);  // g(u) - b (integrator.py:121)
        } else {
            rc = launch_scale(source, -1.0, g, n, side);
        }
        if (!rc)
            rc = run_stencil_series(d, g, z, dd_phi, xi, ndd_phi, alpha, shift, tol, nullptr, ws_phi, ws_bytes,
                                    nullptr, side);
        cudaMemcpyAsync(f->bad_host, f->bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, side);
        cudaEventRecord(f->join, side);
        cudaStreamWaitEvent(s, f->join, 0);
    }
    if (rc) return rc;
    if (!fused) cudaEventRecord(f->t1, s);
    if (phi && !fused) {
        k_axpy_if<<<grid_for(n), 256, 0, s>>>(u_out, z, h, u_out, n, series_state_ptr(ws_exp),
                                              series_state_ptr(ws_phi));
        if ((rc = check_launch("step combination"))) return rc;
    }
    if (!fused) {
        rc = series_status(read_series_state(series_state_ptr(ws_exp), &res->exp_series, s), &res->status_exp);
        if (!rc && phi)
            rc = series_status(read_series_state(series_state_ptr(ws_phi), &res->phi1_series, s), &res->status_phi1);
        if (rc) return rc;
    }
    cudaEventElapsedTime(&res->series_ms, f->t0, f->t1);
    if (phi && nonlin == ES_NONLIN_COMBUSTION && *f->bad_host < (unsigned long long)n) {
        res->first_bad = (int64_t)*f->bad_host;
        return set_error(ES_ERR_DOMAIN, "combustion nonlinearity undefined at index %lld", (long long)res->first_bad);
    }
    if (res->status_exp || res->status_phi1)
        return set_error(ES_ERR_NOT_CONVERGED, "Newton series did not converge (exp: %d nodes%s, phi1: %d nodes%s)",
                         res->exp_series.matvecs, res->status_exp ? " unconverged" : "", res->phi1_series.matvecs,
                         res->status_phi1 ? " unconverged" : "");
    return ES_OK;
}

int run_exprb_finish(const es_stencil_desc *d, const double *u, double *u_out, const double *dd, const double *xi,
                     int ndd, double alpha, double shift, double tol, double h, const double *scratch, void *ws,
                     size_t ws_bytes, es_step_result *res, cudaStream_t s) {
    const int64_t n = d->nx * d->ny * d->lz;
    const double *F = scratch, *gp = scratch + n;
    Fork *f;
    int rc = fork_resources(f);
    if (rc) return rc;
    cudaEventRecord(f->t0, s);
    rc = run_stencil_series(d, F, u_out, dd, xi, ndd, alpha, shift, tol, gp, ws, ws_bytes, nullptr, s);
    if (rc) return rc;
    cudaEventRecord(f->t1, s);
    k_axpy_if<<<grid_for(n), 256, 0, s>>>(u, u_out, h, u_out, n, series_state_ptr(ws), nullptr);
    if ((rc = check_launch("step combination"))) return rc;
    rc = series_status(read_series_state(series_state_ptr(ws), &res->phi1_series, s), &res->status_phi1);
    if (rc) return rc;
    cudaEventElapsedTime(&res->series_ms, f->t0, f->t1);
    if (res->status_phi1)
        return set_error(ES_ERR_NOT_CONVERGED, "Newton series did not converge within degree %d",
                         res->phi1_series.matvecs);
    return ES_OK;
}

int run_exprb_step(const es_stencil_desc *d, const double *u, double *u_out, const double *dd, const double *xi,
                   int ndd, double alpha, double shift, double tol, double h, double a, double b, double lo, double hi,
                   double *scratch, void *aux, void *ws, size_t ws_bytes, es_step_result *res, cudaStream_t s) {
    const int64_t n = d->nx * d->ny * d->lz;
    *res = es_step_result{};
    double mm[2] = {0.0, 0.0};
    int64_t bad = -1;
    int rc = run_rosenbrock_prologue(d, u, scratch, scratch + n, mm, &bad, aux, nullptr, nullptr, s);
    res->first_bad = bad;
    res->gprime_min = mm[0];
    res->gprime_max = mm[1];
    if (rc) return rc;
    // integrator.py (this package): snap_interval(a - max g', b - min g', [a, b])
    double l = a - mm[1], r = b - mm[0];
    const double q = (b - a) / 1024.0;
    if (q > 0) {
        l = std::floor(l / q) * q;
        r = std::ceil(r / q) * q;
    }
    res->lo = l;
    res->hi = r;
    if (l != lo || r != hi)
        return set_error(ES_ERR_RANGE, "interval of A - diag(g') is [%.17g, %.17g], divided differences were built "
                                       "for [%.17g, %.17g]", l, r, lo, hi);
    return run_exprb_finish(d, u, u_out, dd, xi, ndd, alpha, shift, tol, h, scratch, ws, ws_bytes, res, s);
}

}  // namespace es
