/*
 * expstencil_b200 -- C ABI of the B200-native Leja-stencil hot path.
 *
 * Drop-in boundary for the reference's kernel-module protocol
 * (reference pkg/src/expstencil/_kernels.py:43-53 resolves a module exposing
 * stencil_fused_slab / csr_fused / csr_fused_rows / combustion_pointwise,
 * implemented by _core.pyx:176-348) plus the series-level fusion boundary
 * matfunc.newton_apply (matfunc.py:271-318).
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes; every array pointer is DEVICE memory
 *     (cudaMalloc'd, e.g. owned by a torch CUDA tensor) unless the name
 *     ends in _host;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *     work is stream-ordered; nothing allocates or frees caller memory;
 *   - return an ES_* status; on failure es_last_error() describes it
 *     (thread-local).  Python maps ES_ERR_NOT_CONVERGED to ConvergenceError,
 *     ES_ERR_DOMAIN to DomainError, ES_ERR_ARG to ValueError/TypeError;
 *   - fp64 throughout (the reference's hot path is always f64,
 *     matfunc.py:284/:292 upcasts).
 */
#ifndef EXPSTENCIL_B200_H
#define EXPSTENCIL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ES_OK 0
#define ES_ERR_ARG 1
#define ES_ERR_NOT_CONVERGED 2
#define ES_ERR_DOMAIN 3
#define ES_ERR_CUDA 4

/* ghost-value rules; 0..2 are the reference's MODE_ZERO/PERIODIC/FACES
 * (_pykernels.py:27-29), 3 is the build-defined homogeneous Neumann rule */
#define ES_MODE_ZERO 0
#define ES_MODE_PERIODIC 1
#define ES_MODE_FACES 2
#define ES_MODE_NEUMANN 3

/* position-dependent coefficient D at the output point (stencil.py:124-136) */
#define ES_COEFF_NONE 0
#define ES_COEFF_RADIAL 1 /* D = 1/sqrt(1+x^2+y^2) evaluated in-kernel (bench.py:40-41) */
#define ES_COEFF_ARRAY 2  /* D sampled on the grid, (lz, ny, nx) slab-local */

/* One z-slab of the x-fastest grid (grid.py:96-102); replaces the argument
 * list of _core.stencil_fused_slab (_core.pyx:176-191). */
typedef struct es_stencil_desc {
    int64_t nx, ny, lz;     /* slab extents (lz planes) */
    int64_t z0, nz_total;   /* global index of the slab's first plane, total planes */
    double wx, wy, wz;      /* host-computed per-axis 1/dx^2, 0 for 1-point axes */
    int32_t mode;           /* ES_MODE_* */
    int32_t coeff_kind;     /* ES_COEFF_* */
    const double *coeff;    /* ES_COEFF_ARRAY only */
    const double *faces[6]; /* ES_MODE_FACES only: fx_lo, fx_hi (nz_total, ny);
                               fy_lo, fy_hi (nz_total, nx); fz_lo, fz_hi (ny, nx) */
} es_stencil_desc;

/* Outcome of one Newton-Leja series (matfunc.py:297-318). */
typedef struct es_series_result {
    int32_t matvecs;   /* operator products performed */
    int32_t converged; /* 1: stopped by the twice-in-a-row test, or tol == 0 */
    double last_term;  /* |dd_k| ||w_k||_2 of the last node */
    double last_pnorm; /* ||p_k||_2 of the last node */
    int32_t passes;    /* sweeps over the operand: == matvecs, except where two nodes share one pass */
    int32_t reserved;
} es_series_result;

int es_abi_version(void);
const char *es_last_error(void);
/* 1 when a CUDA device is usable, 0 otherwise (never errors) */
int es_device_available(void);

/* out = alpha * (D A u) + beta * u on one slab; halo_lo/halo_hi are the
 * (ny, nx) planes below/above the slab or NULL (_core.pyx:176-226). */
int es_stencil_fused_slab(const es_stencil_desc *d, const double *u, double *out, double alpha,
                          double beta, const double *halo_lo, const double *halo_hi,
                          void *stream);

/* y[r] = alpha * sum_k vals[k] x[col[k]] (+ beta x[r] if use_beta) for
 * r in [row_lo, row_hi), summed in storage order (_core.pyx:245-319). */
int es_csr_fused_rows(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr,
                      const int32_t *col_idx, const double *vals, const double *x, double *y,
                      double alpha, double beta, int32_t use_beta, void *stream);

/* Single-precision twins of the two plain applies (_core.pyx instantiates
 * its stencil and combustion kernels for float too): weights, alpha, beta
 * are cast to float and every operation rounds in float.  d->coeff_kind /
 * d->coeff / d->faces are ignored: the float coefficient (slab-local,
 * nullable) and the six float face arrays (ES_MODE_FACES) come separately.
 * The combustion twin does NOT check the domain (callers do, as the
 * reference's integrator.py:43-49) and uses CUDA expf (<= 2 ulp from libm). */
int es_stencil_fused_slab_f32(const es_stencil_desc *d, const float *u, float *out, double alpha,
                              double beta, const float *coeff, const float *const *faces,
                              const float *halo_lo, const float *halo_hi, void *stream);
int es_combustion_pointwise_f32(const float *u, float *out, int64_t n, void *stream);

/* out = (2 - u)/4 * exp(20 (1 - 1/u)); if any u <= 0 returns ES_ERR_DOMAIN
 * with the first offending index in *first_bad_host (integrator.py:35-54,
 * _core.pyx:341-348).  Synchronises the stream. */
int es_combustion_pointwise(const double *u, double *out, int64_t n, int64_t *first_bad_host,
                            void *stream);

/* Fused Newton-Leja series on a stencil slab: p_out = sum_k dd_k w_k with
 * w_k = (alpha A + beta_k I) w_{k-1}, beta_k = -shift - xi[k-1], w_0 = v,
 * one pass over HBM per node -- per TWO nodes on 3D Dirichlet / Neumann
 * grids (ES_TB, default on) -- and the stopping test on the device
 * (matfunc.py:271-318); results and matvec counts do not depend on the
 * pass structure.  gdiag (nullable) turns A into the build-defined
 * Rosenbrock operator A - diag(gdiag).  dd, xi are device arrays of ndd
 * values.  Blocks until the series finished (one host read-back);
 * returns ES_ERR_NOT_CONVERGED when tol > 0 and the nodes ran out. */
size_t es_leja_stencil_workspace_bytes(const es_stencil_desc *d);
int es_leja_stencil(const es_stencil_desc *d, const double *v, double *p_out,
                    const double *dd, const double *xi, int32_t ndd, double alpha, double shift,
                    double tol, const double *gdiag, void *workspace, size_t workspace_bytes,
                    es_series_result *result_host, void *stream);

/* Asynchronous form: enqueue the whole series (no host sync); the outcome
 * stays in the workspace until es_leja_fetch synchronises the stream and
 * reads it (ES_ERR_NOT_CONVERGED as above).  Lets a caller bracket the
 * series with CUDA events or queue several series back to back. */
int es_leja_stencil_async(const es_stencil_desc *d, const double *v, double *p_out,
                          const double *dd, const double *xi, int32_t ndd, double alpha,
                          double shift, double tol, const double *gdiag, void *workspace,
                          size_t workspace_bytes, void *stream);
int es_leja_fetch(void *workspace, es_series_result *result_host, void *stream);

/* Same series for a square CSR operator (sparse.py:150-151 protocol). */
size_t es_leja_csr_workspace_bytes(int64_t n);
int es_leja_csr(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *vals,
                const double *v, double *p_out, const double *dd, const double *xi,
                int32_t ndd, double alpha, double shift, double tol, void *workspace,
                size_t workspace_bytes, es_series_result *result_host, void *stream);
int es_leja_csr_async(int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                      const double *vals, const double *v, double *p_out, const double *dd,
                      const double *xi, int32_t ndd, double alpha, double shift, double tol,
                      void *workspace, size_t workspace_bytes, void *stream);

/* Complex CSR (the reference's propagate path, cli.py:304-357; its compiled
 * core _core.pyx:263-278).  Complex arrays are interleaved (re, im) doubles
 * (C99 double complex / numpy complex128 layout); vals are real
 * (vals_complex = 0) or interleaved complex.  alpha / beta are complex
 * scalars given as (re, im) parts. */
int es_csr_fused_rows_z(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr,
                        const int32_t *col_idx, const double *vals, int32_t vals_complex,
                        const double *x, double *y, double alpha_re, double alpha_im,
                        double beta_re, double beta_im, int32_t use_beta, void *stream);

/* Every dtype combination of the kernel module's csr_fused_rows
 * (_core.pyx:281-315): col_bytes 4 (int32) or 8 (int64 -- the reference
 * widens columns past 2^31-1, sparse.py:37-39); (vals_kind, x_kind) one of
 * (F64, F64), (F32, F32), (F64, C128), (C128, C128); anything else returns
 * ES_ERR_TYPE (the core's TypeError).  Sums in storage order in the data's
 * precision; alpha / beta complex for C128 x (imaginary parts ignored for
 * real x, rounded to float for F32).  int32 f64 / complex route to the same
 * kernels as es_csr_fused_rows / es_csr_fused_rows_z. */
#define ES_ERR_TYPE 6
#define ES_KIND_F32 0
#define ES_KIND_F64 1
#define ES_KIND_C128 2
int es_csr_fused_rows_ex(int64_t row_lo, int64_t row_hi, const int64_t *row_ptr, const void *col_idx,
                         int32_t col_bytes, const void *vals, int32_t vals_kind, const void *x, void *y,
                         int32_t x_kind, double alpha_re, double alpha_im, double beta_re, double beta_im,
                         int32_t use_beta, void *stream);

/* Complex Newton-Leja series: p = sum_k dd_k w_k with complex dd (ndd
 * interleaved values), w_k = (alpha A + beta_k) w_{k-1}, complex alpha (the
 * reference's op_alpha: 1/gamma, or -1j/gamma on an imaginary-axis interval),
 * real beta_k = -shift - xi[k-1]; ddabs[k] = |dd_k| as the host computed it
 * (numpy abs) drives the stopping test.  Same semantics as es_leja_csr. */
size_t es_leja_csr_z_workspace_bytes(int64_t n);
int es_leja_csr_z(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *vals,
                  int32_t vals_complex, const double *v, double *p_out, const double *dd,
                  const double *ddabs, const double *xi, int32_t ndd, double alpha_re,
                  double alpha_im, double shift, double tol, void *workspace,
                  size_t workspace_bytes, es_series_result *result_host, void *stream);
int es_leja_csr_z_async(int64_t n, const int64_t *row_ptr, const int32_t *col_idx,
                        const double *vals, int32_t vals_complex, const double *v, double *p_out,
                        const double *dd, const double *ddabs, const double *xi, int32_t ndd,
                        double alpha_re, double alpha_im, double shift, double tol,
                        void *workspace, size_t workspace_bytes, void *stream);

/* Multi-GPU slab series (decomp.py:146-266 / :368-382 on one rank per GPU).
 * The series state lives on every rank; per node k = 1, 2, ... the caller
 *   1. sends the first/last plane of *es_leja_dist_source(ws, k) to the
 *      neighbouring ranks and receives theirs into halo_lo / halo_hi (the
 *      buffers passed to begin; NULL at the physical boundary),
 *   2. es_leja_dist_node: one fused pass over the slab plus this slab's
 *      per-z-chunk partial sums (nslices x 2 doubles) into slices_out,
 *   3. all-gathers the slices of all ranks in rank order and calls
 *      es_leja_dist_decide, which runs the stopping test identically on
 *      every rank (chunks aligned to global z make the sums bitwise equal to
 *      a single-GPU run),
 * and finally es_leja_dist_end + es_leja_fetch.  Nodes after the decision
 * return immediately, so the caller may enqueue ahead and poll. */
int es_leja_dist_begin(const es_stencil_desc *d, const double *v, double *p_out,
                       const double *dd, const double *xi, int32_t ndd, double alpha,
                       double shift, double tol, const double *gdiag, const double *halo_lo,
                       const double *halo_hi, void *workspace, size_t workspace_bytes, void *stream);
int es_leja_dist_source(const void *workspace, int32_t k, const double **src_out);
int es_leja_dist_nslices(const void *workspace, int32_t *nslices_out);
int es_leja_dist_node(const void *workspace, double *slices_out, void *stream);
int es_leja_dist_decide(const void *workspace, const double *slices_all, int32_t nslices, void *stream);
int es_leja_dist_end(const void *workspace, void *stream);

/* Peer-memory (NVLink P2P) slab series: the fused compute + exchange form of
 * the slab series above.  One call enqueues the whole series as one CUDA
 * graph on this rank's stream; no host involvement per node:
 *   - after node k the slice kernel stores the first / last plane of w_k
 *     straight into the lower / upper neighbour's halo buffer of parity
 *     (k + 1) & 1 (peer stores over NVLink), writes this slab's per-chunk
 *     sums into every rank's slice table at slice_offset and adds 1 to
 *     every rank's arrival counter
 *     (system-scope), then waits until its own counter reaches
 *     base + nranks * (k + 1) and runs the stopping test on the full table;
 *   - round 0 (before node 1) exchanges v's boundary planes the same way.
 * Every pointer below is a device address valid in THIS process: peers'
 * buffers are mapped with es_ipc_open (or are local buffers of other
 * in-process ranks).  Slice tables hold 2 x total_slices x 2 doubles, halo
 * buffers one (ny, nx) plane each; counters are u64, zero-initialised once
 * and never reset (pass base = nranks x rounds completed so far, where a
 * series of K nodes completes K + 1 rounds).  A peer that does not arrive
 * within timeout_ns ends the series with ES_ERR_CUDA at es_leja_fetch.
 * Completion / result: es_leja_fetch.
 *
 * halo_planes = 2 selects two Leja nodes per pass (the single-GPU default,
 * stencil_tb.cuh) where the operator allows it (Dirichlet / Neumann, no
 * sampled coefficient array, lz >= 2): halo buffers then hold TWO planes
 * each (halo_lo: planes -2, -1; halo_hi: lz, lz + 1), one round per pass
 * (pass p reads halo parity p & 1, round 0 fills parity 0; a series of K
 * nodes completes ceil(K / 2) + 1 rounds), slice tables hold
 * 2 x 2 x total_slices x 2 doubles, and with a g' diagonal gdiag_lo /
 * gdiag_hi are the neighbours' boundary planes of g' (filled by the caller
 * before the call; NULL without a neighbour).  halo_planes = 2 on an
 * operator that does not allow it (or with ES_TB=0) is ES_ERR_ARG: ranks must
 * agree on the round count.  0 or 1: one node per pass, one-plane halos. */
typedef struct es_p2p_desc {
    int32_t nranks, rank;
    int64_t slice_offset, total_slices;
    double *halo_lo[2], *halo_hi[2];  /* this rank's receive buffers by parity (NULL: no neighbour) */
    double *peer_lo[2], *peer_hi[2];  /* lower neighbour's halo_hi[2] / upper neighbour's halo_lo[2] */
    double *const *rank_slices;       /* device array [nranks] of slice-table pointers */
    unsigned long long *const *rank_arrive; /* device array [nranks] of counter pointers */
    unsigned long long *arrive_local; /* this rank's counter */
    unsigned long long base;
    int64_t timeout_ns;               /* <= 0: 10 s */
    int32_t halo_planes;              /* 0 / 1: one node per pass; 2: two (see above) */
    const double *gdiag_lo, *gdiag_hi; /* neighbours' g' boundary planes (halo_planes = 2) */
} es_p2p_desc;

int es_leja_stencil_nslices(const es_stencil_desc *d, int32_t *nslices_out);
int es_leja_p2p(const es_stencil_desc *d, const es_p2p_desc *p2p, const double *v, double *p_out,
                const double *dd, const double *xi, int32_t ndd, double alpha, double shift,
                double tol, const double *gdiag, void *workspace, size_t workspace_bytes,
                void *stream);

/* Peer-memory row-block CSR series: the fused compute + all-gather form of
 * es_leja_csr_dist_*.  Every rank keeps its gathered vector twice
 * (xg_local[0..1], npad doubles each; rank_xg[q] is rank q's buffer base,
 * parity 1 at + npad): node k gathers from parity k & 1 and stores each of
 * its rows' w_k at row_offset + r of EVERY rank's parity (k + 1) & 1
 * buffer; slices, arrival counters, base and timeout as in es_p2p_desc.
 * Column indices address the padded gathered layout (rank q's rows at
 * q * width, like the NCCL form).  Completion / result: es_leja_fetch. */
typedef struct es_p2p_rows_desc {
    int32_t nranks, rank;
    int64_t slice_offset, total_slices;
    int64_t row_offset, npad;
    double *xg_local[2];
    double *const *rank_xg;
    double *const *rank_slices;
    unsigned long long *const *rank_arrive;
    unsigned long long *arrive_local;
    unsigned long long base;
    int64_t timeout_ns;
} es_p2p_rows_desc;

int es_leja_csr_nslices(int64_t n_local, int32_t *nslices_out);
int es_leja_csr_p2p(int64_t n_local, const int64_t *row_ptr, const int32_t *col_idx,
                    const double *vals, const es_p2p_rows_desc *p2p, const double *v,
                    double *p_out, const double *dd, const double *xi, int32_t ndd, double alpha,
                    double shift, double tol, void *workspace, size_t workspace_bytes, void *stream);

/* CUDA IPC for the peer mappings: a 64-byte handle of a device allocation
 * (cudaIpcGetMemHandle; offset_out = dev_ptr - allocation base) and its
 * mapping in another process (peer access over NVLink). */
int es_ipc_handle(const void *dev_ptr, void *handle_out, int64_t *offset_out);
int es_ipc_open(const void *handle, int64_t offset, void **dev_ptr_out);
int es_ipc_close(void *dev_ptr);

/* Multi-GPU row-block CSR series (decomp.py:285-345, PartitionedCsr._run
 * :304-333, on one rank per GPU).  Each rank owns rows [r_lo, r_hi) as a
 * local CSR block (row_ptr rebased to 0, n_local + 1 entries) whose column
 * indices address x_gathered, the caller-owned buffer of n_gathered doubles
 * into which every node's source vectors of all ranks are all-gathered
 * (rank order).
 * The workspace is es_leja_csr_workspace_bytes(n_local).  Per node k the
 * caller
 *   1. all-gathers *es_leja_csr_dist_source(ws, k) (n_local doubles) of every
 *      rank into x_gathered,
 *   2. es_leja_csr_dist_node: the local rows' fused pass plus per-chunk
 *      (16384-row) partial sums (nslices x 2 doubles) into slices_out,
 *   3. all-gathers the slices of all ranks in rank order and calls
 *      es_leja_dist_decide (shared with the slab series),
 * and finally es_leja_csr_dist_end + es_leja_fetch. */
int es_leja_csr_dist_begin(int64_t n_local, const int64_t *row_ptr, const int32_t *col_idx,
                           const double *vals, const double *x_gathered, int64_t n_gathered,
                           const double *v,
                           double *p_out, const double *dd, const double *xi, int32_t ndd,
                           double alpha, double shift, double tol, void *workspace,
                           size_t workspace_bytes, void *stream);
int es_leja_csr_dist_source(const void *workspace, int32_t k, const double **src_out);
int es_leja_csr_dist_nslices(const void *workspace, int32_t *nslices_out);
int es_leja_csr_dist_node(const void *workspace, double *slices_out, void *stream);
int es_leja_csr_dist_end(const void *workspace, void *stream);
/* Byte offset of the series state {int k, consecutive, done, converged;
 * double last_term, last_pnorm} inside a series workspace (for asynchronous
 * polling of `done` with a plain device-to-host copy). */
size_t es_leja_state_offset(void);

/* Integrator-stage element-wise kernels (integrator.py:177-189,
 * matfunc.py:366-371); all stream-ordered, no sync. */
int es_axpy(const double *y, const double *z, double h, double *out, int64_t n, void *stream);
int es_scale(const double *x, double s, double *out, int64_t n, void *stream);
int es_half_sum(const double *a, const double *b, double *out, int64_t n, void *stream);
/* g'(u) of the combustion term (build-defined Rosenbrock Jacobian) and its
 * min/max written to minmax_dev[0..1]. */
int es_combustion_jacobian(const double *u, double *out, double *minmax_dev, int64_t n,
                           void *stream);
/* Fused prologue of the build-defined exponential Rosenbrock step for the
 * combustion term: one stencil pass over u writes F = g(u) - A u and
 * gdiag = g'(u), and returns min/max g' (minmax_host[0..1]) and the first
 * index with u <= 0 (ES_ERR_DOMAIN, *first_bad_host).  aux_dev: 3 x u64 of
 * device scratch.  Needs the TMA path (even nx, 16-byte aligned vectors, no
 * Dirichlet-function faces).  Synchronises the stream. */
int es_rosenbrock_prologue(const es_stencil_desc *d, const double *u, double *F, double *gdiag,
                           double *minmax_host, int64_t *first_bad_host, void *aux_dev,
                           const double *halo_lo, const double *halo_hi, void *stream);

/* max |x| (integrator.py:236 observer) into *out_dev. */
int es_max_abs(const double *x, int64_t n, double *out_dev, void *stream);

/* ---- fused integrator steps (the stage helpers) ----
 * One C call per step, stream-ordered, one host synchronisation at the end.
 * They replace the Python orchestration of integrator.py:177-189
 * (_StepWorkspace.step: exp series, g(u) - b, phi1 series, y + h z) and of the
 * build-defined exponential Rosenbrock step. */
#define ES_ERR_RANGE 5 /* es_exprb_step: the interval of M = A - diag(g') differs */

#define ES_NONLIN_NONE 0       /* g = 0 (g_n = -source, or no phi1 series) */
#define ES_NONLIN_COMBUSTION 1 /* g(u) = (2 - u)/4 exp(20 (1 - 1/u)) */

typedef struct es_step_result {
    es_series_result exp_series;  /* y = exp(-h A) u (exp-Euler only) */
    es_series_result phi1_series; /* z = phi1(-h A) g_n  /  phi1(-h M) F */
    int32_t status_exp, status_phi1; /* ES_OK / ES_ERR_NOT_CONVERGED per series */
    int64_t first_bad;            /* first index with u <= 0, else -1 */
    double gprime_min, gprime_max; /* Rosenbrock: range of g'(u) */
    double lo, hi;                /* Rosenbrock: snapped interval the step needs */
    float series_ms;              /* device time of the series (fork to join) */
} es_step_result;

/* Exponential Euler step u_out = exp(-hA) u + h phi1(-hA) g_n with
 * g_n = g(u) - source (integrator.py:177-189).  The exp and phi1 series share
 * the nodes xi, alpha and shift (one interval, one h) and run CONCURRENTLY
 * (the phi1 series on an internal stream forked from `stream`).
 * scratch: 2 n doubles (g_n, z); ws_exp / ws_phi: two series workspaces of
 * es_leja_stencil_workspace_bytes each.  u_out must not alias u.
 * Returns ES_ERR_DOMAIN (first_bad) if any u <= 0 with combustion, or
 * ES_ERR_NOT_CONVERGED with status_exp / status_phi1 telling which series
 * ran out of nodes: u_out then holds y (when the exp series converged) and
 * scratch holds g_n and z, so the caller can run the halving rescue
 * (matfunc.py:328-373) for that series only. */
int es_expeuler_step(const es_stencil_desc *d, const double *u, double *u_out, const double *dd_exp,
                     int32_t ndd_exp, const double *dd_phi, int32_t ndd_phi, const double *xi, double alpha,
                     double shift, double tol, double h, int32_t nonlinearity, const double *source,
                     double *scratch, void *ws_exp, void *ws_phi, size_t ws_bytes, es_step_result *result_host,
                     void *stream);

/* Exponential Rosenbrock-Euler step (build-defined) for the combustion term:
 * fused prologue F = g(u) - A u, g' = g'(u); the interval of M = A - diag(g')
 * is [a - max g', b - min g'] snapped outward to multiples of (b - a)/1024
 * ([a, b]: A's Gershgorin interval).  If it equals [lo, hi] (the interval dd
 * was built for), runs z = phi1(-hM) F and u_out = u + h z; otherwise returns
 * ES_ERR_RANGE with the snapped interval in result->lo/hi and F, g' kept in
 * scratch (2 n doubles) for es_exprb_finish with the right dd.
 * aux_dev: 4 x u64 device scratch. */
int es_exprb_step(const es_stencil_desc *d, const double *u, double *u_out, const double *dd, const double *xi,
                  int32_t ndd, double alpha, double shift, double tol, double h, double a, double b, double lo,
                  double hi, double *scratch, void *aux_dev, void *workspace, size_t workspace_bytes,
                  es_step_result *result_host, void *stream);
int es_exprb_finish(const es_stencil_desc *d, const double *u, double *u_out, const double *dd, const double *xi,
                    int32_t ndd, double alpha, double shift, double tol, double h, const double *scratch,
                    void *workspace, size_t workspace_bytes, es_step_result *result_host, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* EXPSTENCIL_B200_H */
