// extern "C" entry points of libexpstencil_b200 (include/expstencil_b200.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "es_common.cuh"
#include "es_host.h"

namespace es {

static thread_local char t_err[512] = "";

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(t_err, sizeof(t_err), fmt, ap);
    va_end(ap);
    return code;
}

int check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(ES_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return ES_OK;
}

int current_device() {
    int d = -1;
    cudaGetDevice(&d);
    return d;
}

struct Pinned {
    int device = -1;
    SeriesState *host = nullptr;  // [2]
    unsigned long long *word = nullptr;
};
static thread_local Pinned t_pinned;

static int pinned(Pinned *&p) {
    p = &t_pinned;
    if (p->device != current_device() || !p->host) {
        if (cudaMallocHost(&p->host, 2 * sizeof(SeriesState)) != cudaSuccess ||
            cudaMallocHost(&p->word, sizeof(unsigned long long)) != cudaSuccess)
            return check_launch("pinned state");
        p->device = current_device();
    }
    return ES_OK;
}

int series_result_of(const SeriesState &st, es_series_result *res) {
    res->matvecs = st.k;
    res->converged = st.converged;
    res->last_term = st.last_term;
    res->last_pnorm = st.last_pnorm;
    res->passes = st.pass > 0 ? st.pass : st.k;  // one-node series never count passes
    res->reserved = 0;
    if (!st.done) return set_error(ES_ERR_CUDA, "series did not finish (k=%d)", st.k);
    if (st.converged < 0)
        return set_error(ES_ERR_CUDA, "peer-memory series: a peer did not arrive within the timeout (node %d)", st.k);
    if (!st.converged)
        return set_error(ES_ERR_NOT_CONVERGED, "Newton series did not converge within degree %d", st.k);
    return ES_OK;
}

int read_series_state(const SeriesState *state_dev, es_series_result *res, cudaStream_t stream) {
    Pinned *p;
    int rc = pinned(p);
    if (rc) return rc;
    cudaMemcpyAsync(p->host, state_dev, sizeof(SeriesState), cudaMemcpyDeviceToHost, stream);
    if (cudaStreamSynchronize(stream) != cudaSuccess) return check_launch("series sync");
    return series_result_of(p->host[0], res);
}

int read_series_states2(const SeriesState *a, es_series_result *ra, int *rc_a, const SeriesState *b,
                        es_series_result *rb, int *rc_b, const unsigned long long *word_dev,
                        unsigned long long *word_host, cudaStream_t stream) {
    Pinned *p;
    int rc = pinned(p);
    if (rc) return rc;
    cudaMemcpyAsync(p->host, a, sizeof(SeriesState), cudaMemcpyDeviceToHost, stream);
    cudaMemcpyAsync(p->host + 1, b, sizeof(SeriesState), cudaMemcpyDeviceToHost, stream);
    if (word_dev) cudaMemcpyAsync(p->word, word_dev, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream);
    if (cudaStreamSynchronize(stream) != cudaSuccess) return check_launch("series sync");
    if (word_dev) *word_host = *p->word;
    *rc_a = series_result_of(p->host[0], ra);
    *rc_b = series_result_of(p->host[1], rb);
    return ES_OK;
}

// pointers = false: only extents / mode / kind are checked (the f32 entry
// passes its coefficient and faces separately from the descriptor)
static int check_desc(const es_stencil_desc *d, bool pointers = true) {
    if (!d) return set_error(ES_ERR_ARG, "null descriptor");
    if (d->nx < 1 || d->ny < 1 || d->lz < 0 || d->z0 < 0 || d->z0 + d->lz > d->nz_total)
        return set_error(ES_ERR_ARG, "bad slab extents nx=%lld ny=%lld lz=%lld z0=%lld nz=%lld",
                         (long long)d->nx, (long long)d->ny, (long long)d->lz, (long long)d->z0,
                         (long long)d->nz_total);
    if (d->mode < ES_MODE_ZERO || d->mode > ES_MODE_NEUMANN) return set_error(ES_ERR_ARG, "bad mode %d", d->mode);
    if (d->mode == ES_MODE_PERIODIC && (d->z0 != 0 || d->lz != d->nz_total))
        return set_error(ES_ERR_ARG, "periodic wraparound is not defined on a partitioned slab");
    if (d->mode == ES_MODE_FACES && pointers)
        for (int i = 0; i < 6; ++i)
            if (!d->faces[i]) return set_error(ES_ERR_ARG, "faces mode needs six face arrays");
    if (d->coeff_kind < ES_COEFF_NONE || d->coeff_kind > ES_COEFF_ARRAY)
        return set_error(ES_ERR_ARG, "bad coefficient kind %d", d->coeff_kind);
    if (d->coeff_kind == ES_COEFF_ARRAY && !d->coeff && pointers)
        return set_error(ES_ERR_ARG, "coefficient array missing");
    return ES_OK;
}

}  // namespace es

using namespace es;

extern "C" int es_abi_version(void) { return 2; }

extern "C" const char *es_last_error(void) { return t_err; }

extern "C" int es_device_available(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n > 0 ? 1 : 0;
}

extern "C" int es_stencil_fused_slab(const es_stencil_desc *d, const double *u, double *out, double alpha,
                                     double beta, const double *halo_lo, const double *halo_hi, void *stream) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (!u || !out) return set_error(ES_ERR_ARG, "null vector");
    return launch_stencil_apply(d, u, out, alpha, beta, halo_lo, halo_hi, nullptr, (cudaStream_t)stream);
}

extern "C" int es_csr_fused_rows(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr, const int32_t *col_idx,
                                 const double *vals, const double *x, double *y, double alpha, double beta,
                                 int32_t use_beta, void *stream) {
    if (row_lo < 0 || row_hi < row_lo) return set_error(ES_ERR_ARG, "bad row range");
    if (row_hi > row_lo && (!row_ptr || !col_idx || !vals || !x || !y)) return set_error(ES_ERR_ARG, "null pointer");
    return launch_csr_rows(row_lo, row_hi, row_ptr, col_idx, vals, x, y, alpha, beta, use_beta,
                           (cudaStream_t)stream);
}

extern "C" size_t es_leja_stencil_workspace_bytes(const es_stencil_desc *d) {
    if (check_desc(d)) return 0;
    return stencil_series_ws_bytes(d);
}

extern "C" int es_leja_stencil(const es_stencil_desc *d, const double *v, double *p_out, const double *dd,
                               const double *xi, int32_t ndd, double alpha, double shift, double tol,
                               const double *gdiag, void *workspace, size_t workspace_bytes,
                               es_series_result *result_host, void *stream) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (d->mode == ES_MODE_FACES)
        return set_error(ES_ERR_ARG, "fused apply needs a linear operator (faces mode)");
    if (!v || !p_out || !dd || !xi || !workspace) return set_error(ES_ERR_ARG, "null pointer");
    if (v == p_out) return set_error(ES_ERR_ARG, "p_out must not alias v");
    return run_stencil_series(d, v, p_out, dd, xi, ndd, alpha, shift, tol, gdiag, workspace, workspace_bytes,
                              result_host, (cudaStream_t)stream);
}

extern "C" int es_leja_stencil_async(const es_stencil_desc *d, const double *v, double *p_out, const double *dd,
                                     const double *xi, int32_t ndd, double alpha, double shift, double tol,
                                     const double *gdiag, void *workspace, size_t workspace_bytes, void *stream) {
    return es_leja_stencil(d, v, p_out, dd, xi, ndd, alpha, shift, tol, gdiag, workspace, workspace_bytes,
                           nullptr, stream);
}

extern "C" int es_leja_fetch(void *workspace, es_series_result *result_host, void *stream) {
    if (!workspace || !result_host) return set_error(ES_ERR_ARG, "null pointer");
    return read_series_state(series_state_ptr(workspace), result_host, (cudaStream_t)stream);
}

extern "C" size_t es_leja_csr_workspace_bytes(int64_t n) { return n < 0 ? 0 : csr_series_ws_bytes(n); }

extern "C" int es_leja_csr(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *vals,
                           const double *v, double *p_out, const double *dd, const double *xi, int32_t ndd,
                           double alpha, double shift, double tol, void *workspace, size_t workspace_bytes,
                           es_series_result *result_host, void *stream) {
    if (n < 0) return set_error(ES_ERR_ARG, "negative n");
    if (!v || !p_out || !dd || !xi || !workspace || (n > 0 && (!row_ptr || !col_idx || !vals)))
        return set_error(ES_ERR_ARG, "null pointer");
    if (v == p_out) return set_error(ES_ERR_ARG, "p_out must not alias v");
    return run_csr_series(n, row_ptr, col_idx, vals, v, p_out, dd, xi, ndd, alpha, shift, tol, workspace,
                          workspace_bytes, result_host, (cudaStream_t)stream);
}

extern "C" int es_leja_csr_async(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *vals,
                                 const double *v, double *p_out, const double *dd, const double *xi, int32_t ndd,
                                 double alpha, double shift, double tol, void *workspace, size_t workspace_bytes,
                                 void *stream) {
    return es_leja_csr(n, row_ptr, col_idx, vals, v, p_out, dd, xi, ndd, alpha, shift, tol, workspace,
                       workspace_bytes, nullptr, stream);
}

extern "C" int es_rosenbrock_prologue(const es_stencil_desc *d, const double *u, double *F, double *gdiag,
                                      double *minmax_host, int64_t *first_bad_host, void *aux_dev,
                                      const double *halo_lo, const double *halo_hi, void *stream) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (!u || !F || !gdiag || !minmax_host || !first_bad_host || !aux_dev) return set_error(ES_ERR_ARG, "null pointer");
    return run_rosenbrock_prologue(d, u, F, gdiag, minmax_host, first_bad_host, aux_dev, halo_lo, halo_hi,
                                   (cudaStream_t)stream);
}

extern "C" int es_leja_dist_begin(const es_stencil_desc *d, const double *v, double *p_out, const double *dd,
                                  const double *xi, int32_t ndd, double alpha, double shift, double tol,
                                  const double *gdiag, const double *halo_lo, const double *halo_hi, void *workspace,
                                  size_t workspace_bytes, void *stream) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (d->mode == ES_MODE_FACES || d->mode == ES_MODE_PERIODIC)
        return set_error(ES_ERR_ARG, "slab series need a linear, non-periodic boundary rule");
    if (!v || !p_out || !dd || !xi || !workspace) return set_error(ES_ERR_ARG, "null pointer");
    if (v == p_out) return set_error(ES_ERR_ARG, "p_out must not alias v");
    return dist_begin(d, v, p_out, dd, xi, ndd, alpha, shift, tol, gdiag, halo_lo, halo_hi, workspace,
                      workspace_bytes, (cudaStream_t)stream);
}

extern "C" int es_leja_dist_source(const void *workspace, int32_t k, const double **src_out) {
    if (!workspace || !src_out) return set_error(ES_ERR_ARG, "null pointer");
    return dist_source(workspace, k, src_out);
}

extern "C" int es_leja_dist_nslices(const void *workspace, int32_t *nslices_out) {
    if (!workspace || !nslices_out) return set_error(ES_ERR_ARG, "null pointer");
    int n = 0;
    const int rc = dist_nslices(workspace, &n);
    *nslices_out = n;
    return rc;
}

extern "C" int es_leja_dist_node(const void *workspace, double *slices_out, void *stream) {
    if (!workspace || !slices_out) return set_error(ES_ERR_ARG, "null pointer");
    return dist_node(workspace, slices_out, (cudaStream_t)stream);
}

extern "C" int es_leja_dist_decide(const void *workspace, const double *slices_all, int32_t nslices, void *stream) {
    if (!workspace || !slices_all || nslices < 1) return set_error(ES_ERR_ARG, "bad slices");
    return dist_decide(workspace, slices_all, nslices, (cudaStream_t)stream);
}

extern "C" int es_leja_dist_end(const void *workspace, void *stream) {
    if (!workspace) return set_error(ES_ERR_ARG, "null pointer");
    return dist_end(workspace, (cudaStream_t)stream);
}

extern "C" int es_leja_csr_dist_begin(int64_t n_local, const int64_t *row_ptr, const int32_t *col_idx,
                                      const double *vals, const double *x_gathered, int64_t n_gathered,
                                      const double *v, double *p_out,
                                      const double *dd, const double *xi, int32_t ndd, double alpha, double shift,
                                      double tol, void *workspace, size_t workspace_bytes, void *stream) {
    if (n_local < 0) return set_error(ES_ERR_ARG, "negative n_local");
    if (!v || !p_out || !dd || !xi || !workspace || !x_gathered || (n_local > 0 && (!row_ptr || !col_idx || !vals)))
        return set_error(ES_ERR_ARG, "null pointer");
    if (v == p_out) return set_error(ES_ERR_ARG, "p_out must not alias v");
    if (n_gathered < n_local) return set_error(ES_ERR_ARG, "the gathered vector is shorter than the local block");
    return csr_dist_begin(n_local, row_ptr, col_idx, vals, x_gathered, n_gathered, v, p_out, dd, xi, ndd, alpha, shift, tol,
                          workspace, workspace_bytes, (cudaStream_t)stream);
}

extern "C" int es_leja_csr_dist_source(const void *workspace, int32_t k, const double **src_out) {
    if (!workspace || !src_out) return set_error(ES_ERR_ARG, "null pointer");
    return csr_dist_source(workspace, k, src_out);
}

extern "C" int es_leja_csr_dist_nslices(const void *workspace, int32_t *nslices_out) {
    if (!workspace || !nslices_out) return set_error(ES_ERR_ARG, "null pointer");
    int n = 0;
    const int rc = csr_dist_nslices(workspace, &n);
    *nslices_out = n;
    return rc;
}

extern "C" int es_leja_csr_dist_node(const void *workspace, double *slices_out, void *stream) {
    if (!workspace || !slices_out) return set_error(ES_ERR_ARG, "null pointer");
    return csr_dist_node(workspace, slices_out, (cudaStream_t)stream);
}

extern "C" int es_leja_csr_dist_end(const void *workspace, void *stream) {
    if (!workspace) return set_error(ES_ERR_ARG, "null pointer");
    return csr_dist_end(workspace, (cudaStream_t)stream);
}

extern "C" int es_csr_fused_rows_z(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr, const int32_t *col_idx,
                                   const double *vals, int32_t vals_complex, const double *x, double *y,
                                   double alpha_re, double alpha_im, double beta_re, double beta_im,
                                   int32_t use_beta, void *stream) {
    if (row_lo < 0 || row_hi < row_lo) return set_error(ES_ERR_ARG, "bad row range");
    if (row_hi > row_lo && (!row_ptr || !col_idx || !vals || !x || !y)) return set_error(ES_ERR_ARG, "null pointer");
    return launch_csr_rows_z(row_lo, row_hi, row_ptr, col_idx, vals, vals_complex, x, y, alpha_re, alpha_im, beta_re,
                             beta_im, use_beta, (cudaStream_t)stream);
}

extern "C" size_t es_leja_csr_z_workspace_bytes(int64_t n) { return n < 0 ? 0 : csr_z_series_ws_bytes(n); }

extern "C" int es_leja_csr_z(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *vals,
                             int32_t vals_complex, const double *v, double *p_out, const double *dd,
                             const double *ddabs, const double *xi, int32_t ndd, double alpha_re, double alpha_im,
                             double shift, double tol, void *workspace, size_t workspace_bytes,
                             es_series_result *result_host, void *stream) {
    if (n < 0) return set_error(ES_ERR_ARG, "negative n");
    if (!v || !p_out || !dd || !ddabs || !xi || !workspace || (n > 0 && (!row_ptr || !col_idx || !vals)))
        return set_error(ES_ERR_ARG, "null pointer");
    if (v == p_out) return set_error(ES_ERR_ARG, "p_out must not alias v");
    return run_csr_series_z(n, row_ptr, col_idx, vals, vals_complex, v, p_out, dd, ddabs, xi, ndd, alpha_re,
                            alpha_im, shift, tol, workspace, workspace_bytes, result_host, (cudaStream_t)stream);
}

extern "C" int es_leja_csr_z_async(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *vals,
                                   int32_t vals_complex, const double *v, double *p_out, const double *dd,
                                   const double *ddabs, const double *xi, int32_t ndd, double alpha_re,
                                   double alpha_im, double shift, double tol, void *workspace,
                                   size_t workspace_bytes, void *stream) {
    return es_leja_csr_z(n, row_ptr, col_idx, vals, vals_complex, v, p_out, dd, ddabs, xi, ndd, alpha_re, alpha_im,
                         shift, tol, workspace, workspace_bytes, nullptr, stream);
}

extern "C" int es_leja_stencil_nslices(const es_stencil_desc *d, int32_t *nslices_out) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (!nslices_out) return set_error(ES_ERR_ARG, "null pointer");
    *nslices_out = stencil_nslices(d);
    return ES_OK;
}

extern "C" int es_leja_p2p(const es_stencil_desc *d, const es_p2p_desc *p2p, const double *v, double *p_out,
                           const double *dd, const double *xi, int32_t ndd, double alpha, double shift, double tol,
                           const double *gdiag, void *workspace, size_t workspace_bytes, void *stream) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (d->mode == ES_MODE_FACES || d->mode == ES_MODE_PERIODIC)
        return set_error(ES_ERR_ARG, "slab series need a linear, non-periodic boundary rule");
    if (!p2p || !v || !p_out || !dd || !xi || !workspace) return set_error(ES_ERR_ARG, "null pointer");
    if (v == p_out) return set_error(ES_ERR_ARG, "p_out must not alias v");
    return run_p2p_series(d, p2p, v, p_out, dd, xi, ndd, alpha, shift, tol, gdiag, workspace, workspace_bytes,
                          (cudaStream_t)stream);
}

// allocation base of a device pointer (torch's caching allocator hands out
// sub-allocations; IPC handles name whole allocations)
static int alloc_base(const void *p, void **base_out) {
    static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *q = nullptr;
        cudaDriverEntryPointQueryResult r;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &q, cudaEnableDefault, &r) == cudaSuccess &&
            r == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(q);
    });
    if (!fn) return set_error(ES_ERR_CUDA, "cuMemGetAddressRange is unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, (CUdeviceptr)(uintptr_t)p) != CUDA_SUCCESS)
        return set_error(ES_ERR_ARG, "not a device allocation");
    *base_out = (void *)(uintptr_t)base;
    return ES_OK;
}

extern "C" int es_leja_csr_nslices(int64_t n_local, int32_t *nslices_out) {
    if (n_local < 0 || !nslices_out) return set_error(ES_ERR_ARG, "bad argument");
    *nslices_out = csr_nslices(n_local);
    return ES_OK;
}

extern "C" int es_leja_csr_p2p(int64_t n_local, const int64_t *row_ptr, const int32_t *col_idx, const double *vals,
                               const es_p2p_rows_desc *p2p, const double *v, double *p_out, const double *dd,
                               const double *xi, int32_t ndd, double alpha, double shift, double tol, void *workspace,
                               size_t workspace_bytes, void *stream) {
    if (n_local < 1) return set_error(ES_ERR_ARG, "a row block needs at least one row");
    if (!p2p || !v || !p_out || !dd || !xi || !workspace || !row_ptr || !col_idx || !vals)
        return set_error(ES_ERR_ARG, "null pointer");
    if (v == p_out) return set_error(ES_ERR_ARG, "p_out must not alias v");
    return run_csr_p2p_series(n_local, row_ptr, col_idx, vals, p2p, v, p_out, dd, xi, ndd, alpha, shift, tol,
                              workspace, workspace_bytes, (cudaStream_t)stream);
}

extern "C" int es_ipc_handle(const void *dev_ptr, void *handle_out, int64_t *offset_out) {
    if (!dev_ptr || !handle_out || !offset_out) return set_error(ES_ERR_ARG, "null pointer");
    void *base = nullptr;
    int rc = alloc_base(dev_ptr, &base);
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, base) != cudaSuccess) return check_launch("cudaIpcGetMemHandle");
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    std::memcpy(handle_out, &h, sizeof(h));
    *offset_out = (int64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
    return ES_OK;
}

extern "C" int es_ipc_open(const void *handle, int64_t offset, void **dev_ptr_out) {
    if (!handle || !dev_ptr_out) return set_error(ES_ERR_ARG, "null pointer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void *p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return check_launch("cudaIpcOpenMemHandle");
    *dev_ptr_out = static_cast<char *>(p) + offset;
    return ES_OK;
}

extern "C" int es_ipc_close(void *dev_ptr) {
    if (!dev_ptr) return set_error(ES_ERR_ARG, "null pointer");
    void *base = nullptr;
    int rc = alloc_base(dev_ptr, &base);
    if (rc) return rc;
    if (cudaIpcCloseMemHandle(base) != cudaSuccess) return check_launch("cudaIpcCloseMemHandle");
    return ES_OK;
}

extern "C" int es_stencil_fused_slab_f32(const es_stencil_desc *d, const float *u, float *out, double alpha,
                                         double beta, const float *coeff, const float *const *faces,
                                         const float *halo_lo, const float *halo_hi, void *stream) {
    int rc = check_desc(d, false);
    if (rc) return rc;
    if (d->nx * d->ny * d->lz > 0 && (!u || !out)) return set_error(ES_ERR_ARG, "null pointer");
    return launch_stencil_f32(d, u, out, alpha, beta, coeff, faces, halo_lo, halo_hi, (cudaStream_t)stream);
}

extern "C" int es_combustion_pointwise_f32(const float *u, float *out, int64_t n, void *stream) {
    if (n < 0 || (n > 0 && (!u || !out))) return set_error(ES_ERR_ARG, "bad argument");
    return launch_combustion_f32(u, out, n, (cudaStream_t)stream);
}

extern "C" size_t es_leja_state_offset(void) { return series_state_offset(); }

// ----- fused integrator steps (step.cu) ---------------------------------------

static int check_step(const es_stencil_desc *d, const double *u, const double *u_out, const void *scratch,
                      const void *ws, const es_step_result *res) {
    int rc = check_desc(d);
    if (rc) return rc;
    if (d->mode == ES_MODE_FACES) return set_error(ES_ERR_ARG, "fused step needs a linear operator (faces mode)");
    if (!u || !u_out || !scratch || !ws || !res) return set_error(ES_ERR_ARG, "null pointer");
    if (u == u_out) return set_error(ES_ERR_ARG, "u_out must not alias u");
    return ES_OK;
}

extern "C" int es_expeuler_step(const es_stencil_desc *d, const double *u, double *u_out, const double *dd_exp,
                                int32_t ndd_exp, const double *dd_phi, int32_t ndd_phi, const double *xi,
                                double alpha, double shift, double tol, double h, int32_t nonlinearity,
                                const double *source, double *scratch, void *ws_exp, void *ws_phi, size_t ws_bytes,
                                es_step_result *result_host, void *stream) {
    int rc = check_step(d, u, u_out, scratch, ws_exp, result_host);
    if (rc) return rc;
    if (nonlinearity != ES_NONLIN_NONE && nonlinearity != ES_NONLIN_COMBUSTION)
        return set_error(ES_ERR_ARG, "unknown nonlinearity %d", nonlinearity);
    const bool phi = nonlinearity == ES_NONLIN_COMBUSTION || source;
    if (!dd_exp || !xi || (phi && (!dd_phi || !ws_phi))) return set_error(ES_ERR_ARG, "null pointer");
    if (phi && ws_phi == ws_exp) return set_error(ES_ERR_ARG, "the two series need separate workspaces");
    return run_expeuler_step(d, u, u_out, dd_exp, ndd_exp, dd_phi, ndd_phi, xi, alpha, shift, tol, h, nonlinearity,
                             source, scratch, ws_exp, ws_phi, ws_bytes, result_host, (cudaStream_t)stream);
}

extern "C" int es_exprb_step(const es_stencil_desc *d, const double *u, double *u_out, const double *dd,
                             const double *xi, int32_t ndd, double alpha, double shift, double tol, double h,
                             double a, double b, double lo, double hi, double *scratch, void *aux_dev,
                             void *workspace, size_t workspace_bytes, es_step_result *result_host, void *stream) {
    int rc = check_step(d, u, u_out, scratch, workspace, result_host);
    if (rc) return rc;
    if (!dd || !xi || !aux_dev) return set_error(ES_ERR_ARG, "null pointer");
    return run_exprb_step(d, u, u_out, dd, xi, ndd, alpha, shift, tol, h, a, b, lo, hi, scratch, aux_dev, workspace,
                          workspace_bytes, result_host, (cudaStream_t)stream);
}

extern "C" int es_exprb_finish(const es_stencil_desc *d, const double *u, double *u_out, const double *dd,
                               const double *xi, int32_t ndd, double alpha, double shift, double tol, double h,
                               const double *scratch, void *workspace, size_t workspace_bytes,
                               es_step_result *result_host, void *stream) {
    int rc = check_step(d, u, u_out, scratch, workspace, result_host);
    if (rc) return rc;
    if (!dd || !xi) return set_error(ES_ERR_ARG, "null pointer");
    return run_exprb_finish(d, u, u_out, dd, xi, ndd, alpha, shift, tol, h, scratch, workspace, workspace_bytes,
                            result_host, (cudaStream_t)stream);
}
