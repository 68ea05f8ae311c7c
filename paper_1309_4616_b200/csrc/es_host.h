// Host-side internals shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>

#include <initializer_list>

#include "../../include/expstencil_b200.h"

namespace es {

int set_error(int code, const char *fmt, ...);
int check_launch(const char *what);
int current_device();
int env_int(const char *name, int dflt);

// One kernel node of a series loop body; every kernel takes the device
// SeriesParams pointer as its only argument.
struct GraphKernel {
    const void *fn;
    dim3 grid, block;
    size_t smem;
};
// Cached CUDA graph running `ks` in order inside a conditional WHILE node
// (graph.cu); nullptr when graphs are disabled (ES_NO_GRAPH=1) or
// unavailable, in which case the caller launches the nodes itself.
cudaGraphExec_t series_graph(const GraphKernel *ks, int nk, const void *dparams, unsigned long long *handle);

struct SeriesState;
SeriesState *series_state_ptr(void *ws);
size_t series_state_offset();
void launch_state_trivial(void *ws, cudaStream_t stream);
int read_series_state(const SeriesState *state_dev, es_series_result *res, cudaStream_t stream);
// two series' states (and optionally one device word) with ONE stream sync;
// returns each series' own read_series_state status in rc_a / rc_b
int read_series_states2(const SeriesState *a, es_series_result *ra, int *rc_a, const SeriesState *b,
                        es_series_result *rb, int *rc_b, const unsigned long long *word_dev,
                        unsigned long long *word_host, cudaStream_t stream);

struct StencilPlan {
    bool tma;  // v2 TMA-pipelined kernel (else the register-queue v1 kernel)
    bool dim2;
    int vec;
    int chunk;
    dim3 grid, block;
    size_t smem;
    int nslices, ntiles, nchunks;
    int64_t items;  // TMA: (chunk, tile) work items
};

StencilPlan plan_stencil(const es_stencil_desc *d, std::initializer_list<const void *> ptrs, bool tma_ok);
int launch_stencil_apply(const es_stencil_desc *d, const double *u, double *out, double alpha,
                         double beta, const double *halo_lo, const double *halo_hi,
                         const double *gdiag, cudaStream_t stream);
size_t stencil_series_ws_bytes(const es_stencil_desc *d);
int run_rosenbrock_prologue(const es_stencil_desc *d, const double *u, double *F, double *gdiag, double *minmax_host,
                            int64_t *first_bad_host, void *aux_dev, const double *halo_lo, const double *halo_hi,
                            cudaStream_t stream);
int dist_begin(const es_stencil_desc *d, const double *v, double *p_out, const double *dd, const double *xi, int ndd,
               double alpha, double shift, double tol, const double *gdiag, const double *halo_lo,
               const double *halo_hi, void *ws, size_t ws_bytes, cudaStream_t stream);
int dist_source(const void *ws, int k, const double **src);
int dist_nslices(const void *ws, int *nslices);
int dist_node(const void *ws, double *slices_out, cudaStream_t stream);
int dist_decide(const void *ws, const double *slices_all, int nslices, cudaStream_t stream);
int dist_end(const void *ws, cudaStream_t stream);
int run_stencil_series(const es_stencil_desc *d, const double *v, double *p_out, const double *dd,
                       const double *xi, int ndd, double alpha, double shift, double tol,
                       const double *gdiag, void *ws, size_t ws_bytes, es_series_result *res,
                       cudaStream_t stream);

int launch_csr_rows(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr, const int32_t *col,
                    const double *vals, const double *x, double *y, double alpha, double beta,
                    int use_beta, cudaStream_t stream);
size_t csr_series_ws_bytes(int64_t n);
int run_csr_series(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *vals,
                   const double *v, double *p_out, const double *dd, const double *xi, int ndd,
                   double alpha, double shift, double tol, void *ws, size_t ws_bytes,
                   es_series_result *res, cudaStream_t stream);

size_t csr_z_series_ws_bytes(int64_t n);
int launch_csr_rows_z(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr, const int32_t *col, const double *vals,
                      int vals_complex, const double *x, double *y, double ar, double ai, double br, double bi,
                      int use_beta, cudaStream_t stream);
int run_csr_series_z(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *vals, int vals_complex,
                     const double *v, double *p_out, const double *dd, const double *ddabs, const double *xi, int ndd,
                     double alpha_re, double alpha_im, double shift, double tol, void *ws, size_t ws_bytes,
                     es_series_result *res, cudaStream_t stream);
int stencil_nslices(const es_stencil_desc *d);
int launch_stencil_f32(const es_stencil_desc *d, const float *u, float *out, double alpha, double beta,
                       const float *coeff, const float *const *faces, const float *halo_lo, const float *halo_hi,
                       cudaStream_t stream);
int run_expeuler_step(const es_stencil_desc *d, const double *u, double *u_out, const double *dd_exp, int ndd_exp,
                      const double *dd_phi, int ndd_phi, const double *xi, double alpha, double shift, double tol,
                      double h, int nonlin, const double *source, double *scratch, void *ws_exp, void *ws_phi,
                      size_t ws_bytes, es_step_result *res, cudaStream_t s);
int run_exprb_step(const es_stencil_desc *d, const double *u, double *u_out, const double *dd, const double *xi,
                   int ndd, double alpha, double shift, double tol, double h, double a, double b, double lo, double hi,
                   double *scratch, void *aux, void *ws, size_t ws_bytes, es_step_result *res, cudaStream_t s);
int run_exprb_finish(const es_stencil_desc *d, const double *u, double *u_out, const double *dd, const double *xi,
                     int ndd, double alpha, double shift, double tol, double h, const double *scratch, void *ws,
                     size_t ws_bytes, es_step_result *res, cudaStream_t s);
int launch_combustion(const double *u, double *out, int64_t n, unsigned long long *bad_dev, cudaStream_t st);
int launch_fill_u64(unsigned long long *p, unsigned long long a, unsigned long long b, cudaStream_t st);

// persistent small-grid series (series_small.cu)
struct SeriesParams;
bool small_series_ok(const es_stencil_desc *d, const StencilPlan &pl, bool gd, int nseries);
int small_prepare(const es_stencil_desc *d, const double *v, double *p_out, const double *dd, const double *xi,
                  int ndd, double alpha, double shift, double tol, const double *gdiag, void *ws, size_t ws_bytes,
                  int nseries, SeriesParams *hp, SeriesParams **dparams, StencilPlan *plan, bool *ok,
                  cudaStream_t stream);
int launch_series_init(const SeriesParams *hp, SeriesParams *dparams, cudaStream_t stream);
int launch_expeuler_small_init(const SeriesParams *ha, SeriesParams *da, const SeriesParams *hb, SeriesParams *db,
                               unsigned long long *bad, int64_t n, cudaStream_t stream);
int launch_series_small(const es_stencil_desc *d, const SeriesParams *dparams, const StencilPlan &pl, bool gd,
                        cudaStream_t stream);
struct SmallStepRecord;
int launch_expeuler_small(const es_stencil_desc *d, const SeriesParams *pa, const SeriesParams *pb,
                          const StencilPlan &pl, const double *u, double *gn, const double *source, int nonlin,
                          double h, unsigned long long *bad, SmallStepRecord *rec, cudaStream_t stream);
int series_result_of(const SeriesState &st, es_series_result *res);
int launch_axpy(const double *y, const double *z, double h, double *out, int64_t n, cudaStream_t st);
int launch_scale(const double *x, double s, double *out, int64_t n, cudaStream_t st);
int launch_combustion_f32(const float *u, float *out, int64_t n, cudaStream_t stream);
int run_p2p_series(const es_stencil_desc *d, const es_p2p_desc *x, const double *v, double *p_out, const double *dd,
                   const double *xi, int ndd, double alpha, double shift, double tol, const double *gdiag, void *ws,
                   size_t ws_bytes, cudaStream_t stream);
int csr_nslices(int64_t n);
int run_csr_p2p_series(int64_t n, const int64_t *row_ptr, const int32_t *col, const double *vals,
                       const es_p2p_rows_desc *x, const double *v, double *p_out, const double *dd, const double *xi,
                       int ndd, double alpha, double shift, double tol, void *ws, size_t ws_bytes,
                       cudaStream_t stream);
int csr_dist_begin(int64_t n_local, const int64_t *row_ptr, const int32_t *col, const double *vals, const double *xg,
                   int64_t n_xg, const double *v, double *p_out, const double *dd, const double *xi, int ndd, double alpha,
                   double shift, double tol, void *ws, size_t ws_bytes, cudaStream_t stream);
int csr_dist_source(const void *ws, int k, const double **src);
int csr_dist_nslices(const void *ws, int *nslices);
int csr_dist_node(const void *ws, double *slices_out, cudaStream_t stream);
int csr_dist_end(const void *ws, cudaStream_t stream);

}  // namespace es
